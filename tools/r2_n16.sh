#!/bin/bash
# The all-ASCII narrowing copy of the planned reverse: parity, then A/B (tools/opbench.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-n16}
timeout -s KILL 900 python -m pytest tests/test_gpu_planned.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/${TAG}_pytest.log
OPS=${OPS:-utf16le_to_utf8_planned} CFGS=${CFGS:-"c1:1024 c4:1024 c3:512"} REPS=30 bash tools/r2_ab.sh $TAG
