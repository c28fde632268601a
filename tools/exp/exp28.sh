mkdir -p gpurun_out
: > gpurun_out/exp28.log
for v in slong sshort slongfull; do UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le timeout -s KILL 90 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp28.log; done
