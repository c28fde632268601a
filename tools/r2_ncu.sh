#!/bin/bash
# one full ncu capture (source-correlated) of the transcoders on 1 GiB of a config:
#   LIB=variants/x.so bash tools/r2_ncu.sh TAG [cfg] [mib]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-n}; CFG=${2:-c4}; MIB=${3:-1024}
LIB=${LIB:-paper_2111_08692_b200/libunigpu.so}
UG_LIB_OVERRIDE=$PWD/$LIB timeout 300 python tools/ncu_one.py $CFG $MIB > gpurun_out/${TAG}_plain.log 2>&1; echo "plain=$?"
UG_LIB_OVERRIDE=$PWD/$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_transcode}" -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/${TAG} python tools/ncu_one.py $CFG $MIB > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu=$?"
cp $LIB gpurun_out/${TAG}_lib.so
