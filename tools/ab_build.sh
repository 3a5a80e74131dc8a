#!/bin/bash
# Build the committed HEAD (or REV) of the CUDA sources into paper_2010_03817_b200/libspecwalk_A.so
# for A/B timing against the working tree's libspecwalk.so (same gpurun call, same GPU).
REV=${1:-HEAD}
T=$(mktemp -d)
git archive $REV paper_2010_03817_b200/csrc include | tar -x -C $T
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -o paper_2010_03817_b200/libspecwalk_A.so $T/paper_2010_03817_b200/csrc/specwalk.cu && echo "built A from $REV"
rm -rf $T
