mkdir -p gpurun_out
timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 > gpurun_out/exp29.log
timeout -s KILL 120 python tools/opbench.py c4 1024 10 >> gpurun_out/exp29.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_susp0.so timeout -s KILL 120 python tools/opbench.py c4 1024 10 >> gpurun_out/exp29.log 2>&1
