#!/bin/bash
# On the box: HMC-r probe (tools/probe_hmc.py) of several prebuilt libspecwalk_*.so variants in rotation:
#   bash tools/hmc_multi.sh TAG "v1 v2 ..." probe-args      (variant v -> paper_2010_03817_b200/libspecwalk_v.so)
TAG=$1; shift; VARS=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for i in 1 2; do
  for v in $VARS; do
    SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_$v.so python tools/probe_hmc.py "$@" 2>/dev/null | sed "s/^/$v /" >> $O/hmc.txt
  done
done
