mkdir -p gpurun_out
: > gpurun_out/exp34.log
for v in base nolb; do for c in c4 c1; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp34.log
done; done
