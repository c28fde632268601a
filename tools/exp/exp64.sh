mkdir -p gpurun_out
: > gpurun_out/exp64.log
for c in c4 c1 c3; do UG_LIB_OVERRIDE=build_variants/libunigpu_pfx.so timeout -s KILL 200 python tools/exp/prefix_expt.py $c 2>&1 | tail -1 >> gpurun_out/exp64.log; done
