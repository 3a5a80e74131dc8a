#!/bin/bash
# lanczos2 PRO-threshold variants (here): bash tools/tau2_ab.sh
cd $(dirname $0)/..
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC"
for v in "t10:-DSW_PRO_TAU2=1e-10" "t11:-DSW_PRO_TAU2=1e-11" "t12:-DSW_PRO_TAU2=1e-12"; do
  name=${v%%:*}; defs=${v#*:}
  $B $defs -o paper_2010_03817_b200/libspecwalk_$name.so paper_2010_03817_b200/csrc/specwalk.cu &
done
$B -o paper_2010_03817_b200/libspecwalk.so paper_2010_03817_b200/csrc/specwalk.cu &
wait
