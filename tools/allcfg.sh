#!/bin/bash
# per-op timings on every BASELINE config (sizes as in BASELINE.json): tools/allcfg.sh tag
TAG=${1:-x}
mkdir -p gpurun_out
for c in "c1 1024" "c2a 256" "c2b 256" "c3 512" "c4 1024"; do
  set -- $c
  timeout 300 python tools/opbench.py $1 $2 10 2>&1 | tail -1
done > gpurun_out/allcfg_$TAG.log
