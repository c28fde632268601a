mkdir -p gpurun_out
: > gpurun_out/exp63.log
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/exp63.log
for v in r16r5 cur; do for c in c4 c1 c3 c2b c2a; do
L=build_variants/libunigpu_$v.so; [ $v = cur ] && L=paper_2111_08692_b200/libunigpu.so
UG_LIB_OVERRIDE=$L OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 512 10 2>&1 | tail -1 >> gpurun_out/exp63.log
done; done
