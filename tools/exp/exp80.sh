mkdir -p gpurun_out
: > gpurun_out/exp80.log
for v in v6a4 v4a3 r1j; do for c in "c4 1024" "c3 512" "c1 1024"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_validate,utf16le_validate timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp80.log
done; done
