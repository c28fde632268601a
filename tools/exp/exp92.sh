mkdir -p gpurun_out
: > gpurun_out/exp92.log
UG_LIB_OVERRIDE=build_variants/libunigpu_rpst2.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp92.log
for v in rpst2 r1m; do for c in "c4 1024" "c2b 256" "c1 1024" "c3 512"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp92.log
done; done
