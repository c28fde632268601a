mkdir -p gpurun_out
: > gpurun_out/exp26.log
OPS=utf16le_to_utf8 timeout 300 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp26.log
for v in nodec noval both bothnolb; do UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf16le_to_utf8 timeout 300 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp26.log; done
