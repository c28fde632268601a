#!/bin/bash
# Quick GPU check: parity tests + per-op timings on config 4 (1 GiB).  usage: tools/quick.sh tag
TAG=${1:-q}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout -s KILL 300 python tools/opbench.py c4 1024 10 > gpurun_out/op_$TAG.log 2>&1; echo "op=$?"; cat gpurun_out/op_$TAG.log
