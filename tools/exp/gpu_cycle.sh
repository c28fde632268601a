#!/bin/bash
# One GPU round: parity tests, a 1 GiB bench, and an ncu capture of the transcoders (256 MiB).
# Usage (under gpurun): bash tools/gpu_cycle.sh [tag] [ncu-kernel-regex]
TAG=${1:-cycle}
KRE=${2:-k_transcode}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_$TAG.log
timeout -s KILL 600 python bench.py --size-mib 1024 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo "bench=$?"
timeout -s KILL 300 python bench.py --size-mib 256 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b256_$TAG.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 2 -o gpurun_out/prof_$TAG python bench.py --size-mib 256 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
