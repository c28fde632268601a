mkdir -p gpurun_out
: > gpurun_out/exp30.log
for v in vr6 vr3; do UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_validate,utf16le_validate timeout -s KILL 120 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp30.log; done
