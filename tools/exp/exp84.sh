mkdir -p gpurun_out
: > gpurun_out/exp84.log
UG_LIB_OVERRIDE=build_variants/libunigpu_smb.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp84.log
for v in smb r1k; do for c in "c4 1024" "c1 1024" "c3 512"; do set -- $c
UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp84.log
done; done
