mkdir -p gpurun_out
: > gpurun_out/exp88.log
for v in fnoconf r1l; do for c in "c4 1024" "c2b 256"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp88.log
done; done
