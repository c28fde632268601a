#!/bin/bash
# ncu full capture of utf8_to_utf16le with a chosen library: tools/prof2.sh tag lib
TAG=$1; LIB=$2
mkdir -p gpurun_out
UG_LIB_OVERRIDE=$LIB OPS=utf8_to_utf16le timeout 300 python tools/opbench.py c4 256 2 > /dev/null 2>&1 && \
UG_LIB_OVERRIDE=$LIB OPS=utf8_to_utf16le timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transcode -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/opbench.py c4 256 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
