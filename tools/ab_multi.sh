#!/bin/bash
# On the box: time several prebuilt libspecwalk_*.so variants in rotation (same GPU):
#   bash tools/ab_multi.sh TAG "v1 v2 ..." probe-args      (variant v -> paper_2010_03817_b200/libspecwalk_v.so)
TAG=$1; shift; VARS=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for i in 1 2; do
  for v in $VARS; do
    SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_$v.so python tools/prof_probe.py "$@" 2>/dev/null | sed "s/^/$v /" >> $O/ab.txt
  done
done
echo done > $O/DONE
