#!/bin/bash
# one K2 launch under ncu with source-level sampling: bash tools/gpu_ncu_src.sh TAG n:m:chains:rounds
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:chord_kernel -s 4 -c 1 -o $O/k2src \
   python tools/prof_probe.py "$@" > $O/ncu.log 2>&1
echo done > $O/DONE
