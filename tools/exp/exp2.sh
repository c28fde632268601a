mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_trace.so timeout 300 python tools/trace_lb.py 1024 > gpurun_out/exp2.log 2>&1
