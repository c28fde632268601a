mkdir -p gpurun_out
: > gpurun_out/exp39.log
for v in cf51 cf52 cf42 cf41; do for c in c4 c1; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp39.log
done; done
