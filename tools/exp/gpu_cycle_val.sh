#!/bin/bash
# Parity + ncu capture of the validators and length kernels (256 MiB bench config).
TAG=${1:-val}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"; tail -1 gpurun_out/pytest_$TAG.log
timeout -s KILL 600 python bench.py --size-mib 1024 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo "bench=$?"
CMD="python bench.py --size-mib 256 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD > gpurun_out/b256_$TAG.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_validate|k_len" -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
