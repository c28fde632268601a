mkdir -p gpurun_out
: > gpurun_out/exp68.log
for v in nopush lbtick cur; do for c in c4 c1; do
L=build_variants/libunigpu_$v.so; [ $v = cur ] && L=paper_2111_08692_b200/libunigpu.so
UG_LIB_OVERRIDE=$L OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp68.log
done; done
