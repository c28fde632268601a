#!/bin/bash
# UTF-8 validator with VH chunks per thread per tile: parity, then A/B (tools/opbench.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-vh}
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "utf8 or phase or straddl or valid or config or shard or spec" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/${TAG}_pytest.log
OPS=utf8_validate CFGS="c4:1024 c1:1024 c2a:256 c2b:256 c3:512" REPS=30 bash tools/r2_ab.sh $TAG
