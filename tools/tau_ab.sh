#!/bin/bash
# Build variants of libspecwalk with different Lanczos / PRO tolerances (m > 112 global variant)
# usage (here): bash tools/tau_ab.sh ; then on the box: SPECWALK_LIB=... pytest / probe
set -e
cd $(dirname $0)/..
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC"
for v in "tau13:-DSW_PRO_TAU=1e-13" "tau14:-DSW_PRO_TAU=1e-14" "tol14:-DSW_LANCZOS_TOL=1e-14" "both:-DSW_PRO_TAU=1e-13 -DSW_LANCZOS_TOL=1e-14"; do
  name=${v%%:*}; defs=${v#*:}
  $B $defs -o paper_2010_03817_b200/libspecwalk_$name.so paper_2010_03817_b200/csrc/specwalk.cu &
done
wait
ls -la paper_2010_03817_b200/libspecwalk_*.so
