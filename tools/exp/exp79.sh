mkdir -p gpurun_out
: > gpurun_out/exp79.log
for v in nt256c4c r1j; do for c in "c4 1024" "c1 1024" "c3 512" "c2b 256"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp79.log
done; done
