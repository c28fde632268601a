#!/bin/bash
# ncu full capture of the transcoders on 256 MiB of config 4: tools/prof.sh tag [kernel-regex] [ops]
TAG=${1:-p}; KRE=${2:-k_transcode}; OPS=${3:-utf8_to_utf16le,utf16le_to_utf8}
mkdir -p gpurun_out
OPS=$OPS timeout 300 python tools/opbench.py c4 256 2 > /dev/null 2>&1 && \
OPS=$OPS timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 2 -c 2 -o gpurun_out/prof_$TAG python tools/opbench.py c4 256 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
