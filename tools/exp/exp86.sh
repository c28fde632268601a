mkdir -p gpurun_out
: > gpurun_out/exp86.log
for v in noconf r1l; do for c in "c4 1024" "c2b 256"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp86.log
done; done
