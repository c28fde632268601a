mkdir -p gpurun_out
: > gpurun_out/exp50.log
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp50.log
for c in c4 c1 c3; do
OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp50.log
done
