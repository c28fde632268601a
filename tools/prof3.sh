#!/bin/bash
# ncu full capture of one op: tools/prof3.sh tag op kernel-regex [lib]
# The library used is copied next to the report (line mapping needs the exact build).
TAG=$1; OP=$2; KRE=$3; LIB=${4:-paper_2111_08692_b200/libunigpu.so}
mkdir -p gpurun_out
cp $LIB gpurun_out/lib_$TAG.so
UG_LIB_OVERRIDE=$LIB OPS=$OP timeout 300 python tools/opbench.py ${CFG:-c4} 256 2 > /dev/null 2>&1 && \
UG_LIB_OVERRIDE=$LIB OPS=$OP timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/opbench.py ${CFG:-c4} 256 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
