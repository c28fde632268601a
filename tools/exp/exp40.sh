mkdir -p gpurun_out
: > gpurun_out/exp40.log
for v in r52 r51 r42; do for c in c4 c1 c3; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp40.log
done; done
