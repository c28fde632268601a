mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 > gpurun_out/exp24.log
for c in "c1 1024" "c4 1024"; do set -- $c; OPS=utf8_to_utf16le,utf16le_to_utf8 timeout 300 python tools/opbench.py $1 $2 10 >> gpurun_out/exp24.log 2>&1; done
UG_LIB_OVERRIDE=build_variants/libunigpu_bothp.so OPS=utf8_to_utf16le timeout 300 python tools/opbench.py c4 1024 10 2>&1 | tail -1 >> gpurun_out/exp24.log
UG_LIB_OVERRIDE=build_variants/libunigpu_trace.so timeout 300 python tools/trace2.py c4 1024 2>&1 | grep -v cta0 >> gpurun_out/exp24.log
