#!/bin/bash
# lanczos2 first-check position (30% of md default) A/B at m = 100 / 72
T=${1:-r2p}; O=gpurun_out/$T; mkdir -p $O
for i in 1 2; do
  for v in base fc26 fc34 fc38; do
    if [ $v = base ]; then L=$PWD/paper_2010_03817_b200/libspecwalk.so; else L=$PWD/paper_2010_03817_b200/libspecwalk_$v.so; fi
    SPECWALK_LIB=$L timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/${v}_$i.json 2>&1
  done
done
echo done > $O/DONE
