#!/bin/bash
# A/B per-op timings of library variants (tools/opbench.py), transcoders by default:
#   LIBS="variants/a.so variants/b.so" CFGS="c4:1024 c1:1024" bash tools/r2_ab.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
OPS=${OPS:-utf8_to_utf16le,utf16le_to_utf8}
CFGS=${CFGS:-"c4:1024 c1:1024 c3:512 c2b:256"}
for rep in 1 2; do
for c in $CFGS; do
  for lib in $LIBS; do
    UG_LIB_OVERRIDE=$PWD/$lib OPS=$OPS timeout 300 python tools/opbench.py ${c%:*} ${c#*:} ${REPS:-20} 2>&1 | tail -1
  done
done
done > gpurun_out/${TAG}_ab.log
python tools/ab_table.py gpurun_out/${TAG}_ab.log
