#!/bin/bash
# Build libunigpu variants with extra -D flags: tools/variants.sh tag "-DFOO=1" [tag2 "-D..."] ...
cd "$(dirname "$0")/../paper_2111_08692_b200/csrc"
while [ $# -gt 1 ]; do
  tag=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
    -o ../../build_variants/libunigpu_$tag.so kernels.cu api.cu &
done
wait
