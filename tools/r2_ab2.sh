#!/bin/bash
# A/B of variants on chosen ops (tools/opbench.py), plus the planned GPU tests on the default lib
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
if [ -n "$TESTS" ]; then timeout -s KILL 900 python -m pytest $TESTS -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/${TAG}_pytest.log; fi
bash tools/r2_ab.sh $TAG
