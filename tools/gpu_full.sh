#!/bin/bash
# Full measurement round (under gpurun): default bench line, reference arm, ncu launch list of
# the same bench command, and one full-set capture of the dominant kernel for DRAM traffic.
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
timeout -s KILL 900 python bench.py > gpurun_out/bench_full_$TAG.log 2> gpurun_out/bench_full_$TAG.err; echo "bench=$?"
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout -s KILL 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 60 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launches=$?"
CMD2="python bench.py --size-mib 1024 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout -s KILL 600 $CMD2 > gpurun_out/plain2_$TAG.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_transcode -s 2 -c 2 -o gpurun_out/full_$TAG $CMD2 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "full=$?"
cp paper_2111_08692_b200/libunigpu.so gpurun_out/lib_$TAG.so
