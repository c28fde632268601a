mkdir -p gpurun_out
: > gpurun_out/exp66.log
for v in lpl4 lpl3 lpl2 lpl1; do for c in c4 c1 c3; do
L=build_variants/libunigpu_$v.so
UG_LIB_OVERRIDE=$L OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp66.log
done; done
