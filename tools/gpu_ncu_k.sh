#!/bin/bash
# one launch of a named kernel under ncu (full set + source): bash tools/gpu_ncu_k.sh TAG KERNEL_REGEX SKIP probe-args
TAG=$1; shift; K=$1; shift; SKIP=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$K -s $SKIP -c 1 -o $O/rep \
   python tools/prof_probe.py "$@" > $O/ncu.log 2>&1
echo done > $O/DONE
