mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_e12.log 2>&1; echo "pytest=$?" > gpurun_out/exp12.log; tail -1 gpurun_out/pytest_e12.log >> gpurun_out/exp12.log
UG_LIB_OVERRIDE=build_variants/libunigpu_trace.so timeout 300 python tools/trace_lb.py 1024 >> gpurun_out/exp12.log 2>&1
timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp12.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_late.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp12.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_lb2.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp12.log 2>&1
