mkdir -p gpurun_out
: > gpurun_out/exp23.log
for v in bothnolb nolb; do UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le timeout 300 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp23.log; done
