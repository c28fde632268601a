mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_trace.so timeout 300 python tools/dbg_flags.py > gpurun_out/exp14.log 2>&1
