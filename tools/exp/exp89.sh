mkdir -p gpurun_out
: > gpurun_out/exp89.log
UG_LIB_OVERRIDE=build_variants/libunigpu_pst.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp89.log
for v in pst r1l; do for c in "c4 1024" "c2b 256" "c1 1024" "c3 512"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp89.log
done; done
