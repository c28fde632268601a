mkdir -p gpurun_out
: > gpurun_out/exp53.log
for v in nt384 nt256c4; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp53.log
for c in c4 c1 c3; do
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp53.log
done; done
for c in c1 c3; do OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp53.log; done
