mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_mid.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_e11.log 2>&1; echo "pytest=$?" > gpurun_out/exp11.log; tail -1 gpurun_out/pytest_e11.log >> gpurun_out/exp11.log
UG_LIB_OVERRIDE=build_variants/libunigpu_midtrace.so timeout 300 python tools/trace_lb.py 1024 >> gpurun_out/exp11.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_mid.so timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp11.log 2>&1
