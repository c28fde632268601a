mkdir -p gpurun_out
: > gpurun_out/exp42.log
UG_LIB_OVERRIDE=build_variants/libunigpu_d3.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/exp42.log
for v in base d3; do for c in c4 c1 c3; do
L=build_variants/libunigpu_$v.so; [ $v = base ] && L=paper_2111_08692_b200/libunigpu.so
UG_LIB_OVERRIDE=$L OPS=utf8_to_utf16le timeout -s KILL 120 python tools/opbench.py $c 1024 10 2>&1 | tail -1 >> gpurun_out/exp42.log
done; done
