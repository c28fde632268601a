mkdir -p gpurun_out
for v in lb8 lb16 lb32; do
  UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le,utf16le_to_utf8,utf8_validate timeout 300 python tools/opbench.py c4 1024 10
done > gpurun_out/exp1.log 2>&1
