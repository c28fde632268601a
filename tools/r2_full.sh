#!/bin/bash
# Round-2 full measurement (under gpurun): default bench line (planned path), the single-pass
# path for comparison, the reference arm, the ncu launch list of the bench command, DRAM traffic
# of the planned transcoders AT THE BENCH SIZE, one full-set capture at 1 GiB.
cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
timeout -s KILL 1200 python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo "bench=$?"
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref=$?"
timeout -s KILL 900 python bench.py --path chained --no-e2e --no-cpu-baseline --no-per-config > gpurun_out/bench_chained_$TAG.log 2>&1; echo "chained=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-per-op --no-per-config"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launches=$?"
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --kernel-name-base mangled -k regex:'k_transcode_plannedINS_(6U8PolTILb0EEELb0|7U16PolTILb0)' -c 2 --csv --log-file gpurun_out/traffic8g_$TAG.csv $CMD > gpurun_out/ncu_traffic_$TAG.log 2>&1; echo "traffic=$?"
# (mangled names: the forward's running form on config 4 - NOF = false, the input has >= F0
# bytes; its other form returns at once - and the reverse)
OPS=pfwd,prev timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'k_transcode_plannedINS_(6U8PolTILb0EEELb0|7U16PolTILb0)' -c 2 -o gpurun_out/full_$TAG python tools/ncu_one.py c4 1024 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full=$?"
cp paper_2111_08692_b200/libunigpu.so gpurun_out/lib_$TAG.so
