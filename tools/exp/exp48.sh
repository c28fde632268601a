mkdir -p gpurun_out
: > gpurun_out/exp48.log
for v in v2 v3 v3r3; do for c in c4 c3; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_validate,utf16le_validate timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp48.log
done; done
UG_LIB_OVERRIDE=build_variants/libunigpu_v3.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp48.log
