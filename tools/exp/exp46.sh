mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "utf16be_configs" 2>&1 | tail -40 > gpurun_out/exp46_t.log
: > gpurun_out/exp46.log
for c in c4 c1 c3; do
OPS=utf16le_to_utf8,utf16be_to_utf8,utf16le_validate,utf16be_validate timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp46.log
done
