mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_nt384.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 > gpurun_out/exp25.log
for c in "c1 1024" "c4 1024"; do set -- $c; UG_LIB_OVERRIDE=build_variants/libunigpu_nt384.so timeout 300 python tools/opbench.py $1 $2 10 >> gpurun_out/exp25.log 2>&1; done
