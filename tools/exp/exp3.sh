mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_trace.so timeout 300 python tools/trace_lb.py 1024 > gpurun_out/exp3.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_main.so timeout 300 python tools/opbench.py c4 1024 10 >> gpurun_out/exp3.log 2>&1
