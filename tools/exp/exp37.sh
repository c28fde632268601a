mkdir -p gpurun_out
: > gpurun_out/exp37.log
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 >> gpurun_out/exp37.log
echo "pytest rc=$?" >> gpurun_out/exp37.log
for c in c4 c1 c3; do
UG_LIB_OVERRIDE=build_variants/libunigpu_oldrev.so OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp37.log
OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp37.log
done
