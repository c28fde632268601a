mkdir -p gpurun_out
: > gpurun_out/exp81.log
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1 >> gpurun_out/exp81.log
for v in r1j cur; do for c in "c2a 256" "c2b 256" "c4 1024" "c1 1024" "c3 512"; do set -- $c
L=build_variants/libunigpu_$v.so; [ $v = cur ] && L=paper_2111_08692_b200/libunigpu.so
UG_LIB_OVERRIDE=$L OPS=utf16le_to_utf8,utf16be_to_utf8 timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp81.log
done; done
