#!/bin/bash
# Build libunigpu.so as of a commit (for A/B): tools/build_at.sh COMMIT OUT.so [extra nvcc flags]
set -e
C=$1; OUT=$(realpath -m $2); shift 2
D=$(mktemp -d)
git -C "$(dirname "$0")/.." archive "$C" paper_2111_08692_b200/csrc include | tar -x -C "$D"
cd "$D/paper_2111_08692_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o "$OUT" kernels.cu api.cu
rm -rf "$D"
