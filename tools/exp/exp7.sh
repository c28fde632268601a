mkdir -p gpurun_out
./tools/ubench2 > gpurun_out/exp7.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_e7.log 2>&1; echo "pytest=$?" >> gpurun_out/exp7.log; tail -1 gpurun_out/pytest_e7.log >> gpurun_out/exp7.log
timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp7.log 2>&1
