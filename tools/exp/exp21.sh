mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_nt512trace.so timeout 300 python tools/trace2.py c4 1024 > gpurun_out/exp21.log 2>&1
UG_LIB_OVERRIDE=build_variants/libunigpu_nt512trace.so timeout 300 python tools/trace2.py c1 1024 >> gpurun_out/exp21.log 2>&1
