mkdir -p gpurun_out
: > gpurun_out/exp31.log
for c in "c1 1024" "c4 1024"; do set -- $c; UG_LIB_OVERRIDE=build_variants/libunigpu_nt256p.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp31.log; done
