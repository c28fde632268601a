mkdir -p gpurun_out
: > gpurun_out/exp85.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp85.log
for v in r1k cur; do for c in "c4 1024" "c1 1024" "c3 512" "c2b 256"; do set -- $c
L=build_variants/libunigpu_$v.so; [ $v = cur ] && L=paper_2111_08692_b200/libunigpu.so
UG_LIB_OVERRIDE=$L OPS=utf16le_to_utf8,utf16le_validate,utf8_length_from_utf16le timeout -s KILL 120 python tools/opbench.py $1 $2 10 2>&1 | tail -1 >> gpurun_out/exp85.log
done; done
