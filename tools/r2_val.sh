#!/bin/bash
# round-2 validator A/B: tests on the default build, then per-op timings of the validators for
# the default (streaming) build and the ring build on every config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v}
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/${TAG}_pytest.log
for lib in paper_2111_08692_b200/libunigpu.so ${EXTRA_LIBS}; do
  for c in "c4 1024" "c1 1024" "c2a 256" "c2b 256" "c3 512"; do
    set -- $c
    UG_LIB_OVERRIDE=$PWD/$lib OPS=${OPS:-utf8_validate,utf16le_validate,utf16_length_from_utf8,utf8_length_from_utf16le} timeout 300 python tools/opbench.py $1 $2 20 2>&1 | tail -1
  done
done > gpurun_out/${TAG}_ops.log
cat gpurun_out/${TAG}_ops.log
