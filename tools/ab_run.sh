#!/bin/bash
# On the box: alternate A (libspecwalk_A.so) and B (libspecwalk.so) probes: bash tools/ab_run.sh TAG probe-args
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for i in 1 2; do
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_A.so python tools/prof_probe.py "$@" 2>/dev/null | sed 's/^/A /' >> $O/ab.txt
  python tools/prof_probe.py "$@" 2>/dev/null | sed 's/^/B /' >> $O/ab.txt
done
echo done > $O/DONE
