mkdir -p gpurun_out
: > gpurun_out/exp45.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 >> gpurun_out/exp45.log
for c in c4 c1; do
OPS=utf8_to_utf16le,utf8_to_utf16be,utf16le_to_utf8,utf16be_to_utf8,utf16le_validate,utf16be_validate timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp45.log
done
