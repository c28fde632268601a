#!/bin/bash
# Streaming UTF-16 validator: parity, then A/B against the TMA-ring build (tools/opbench.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v16}
timeout -s KILL 900 python -m pytest tests/test_gpu_validate16.py tests/test_gpu_parity.py -m gpu -x -q -k "validate16 or utf16 or be or shard or Validate or valid" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/${TAG}_pytest.log
OPS=utf16le_validate,utf16be_validate CFGS="c4:1024 c1:1024 c3:512 c2a:256 c2b:256" REPS=30 bash tools/r2_ab.sh $TAG
