mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_e5.log 2>&1; echo "pytest=$?" > gpurun_out/exp5.log; tail -2 gpurun_out/pytest_e5.log >> gpurun_out/exp5.log
timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp5.log 2>&1
OPS=utf8_to_utf16le timeout 300 python tools/opbench.py c4 256 2 > /dev/null 2>&1 && OPS=utf8_to_utf16le,utf16le_to_utf8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_transcode -s 2 -c 2 -o gpurun_out/prof_e5 python tools/opbench.py c4 256 2 > gpurun_out/ncu_e5.log 2>&1; echo "ncu=$?" >> gpurun_out/exp5.log
