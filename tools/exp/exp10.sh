mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_late.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_e10.log 2>&1; echo "pytest=$?" > gpurun_out/exp10.log; tail -1 gpurun_out/pytest_e10.log >> gpurun_out/exp10.log
UG_LIB_OVERRIDE=build_variants/libunigpu_latetrace.so timeout 300 python tools/trace_lb.py 1024 >> gpurun_out/exp10.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_late.so timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp10.log 2>&1
