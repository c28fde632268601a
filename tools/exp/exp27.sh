mkdir -p gpurun_out
UG_LIB_OVERRIDE=build_variants/libunigpu_nlb2.so timeout -s KILL 120 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 > gpurun_out/exp27.log
for c in "c1 1024" "c4 1024"; do set -- $c; UG_LIB_OVERRIDE=build_variants/libunigpu_nlb2.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 90 python tools/opbench.py $1 $2 10 >> gpurun_out/exp27.log 2>&1; done
UG_LIB_OVERRIDE=build_variants/libunigpu_nlb2both.so OPS=utf8_to_utf16le timeout -s KILL 90 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp27.log
