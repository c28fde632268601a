mkdir -p gpurun_out
: > gpurun_out/exp36.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp36.log
for c in c4 c3; do
UG_LIB_OVERRIDE=build_variants/libunigpu_base.so OPS=utf8_length_from_utf16le,utf16_length_from_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp36.log
OPS=utf8_length_from_utf16le,utf16_length_from_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp36.log
done
