mkdir -p gpurun_out
: > gpurun_out/exp35.log
for v in r1 r2; do UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp35.log; done
for v in base r1 r2; do for c in c4 c1 c3; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp35.log
done; done
