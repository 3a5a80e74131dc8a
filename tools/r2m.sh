#!/bin/bash
# fused small-m chord kernels compiled for more resident CTAs (register cap 80, some spills) vs default
T=${1:-r2m}; O=gpurun_out/$T; mkdir -p $O
for i in 1 2; do
  timeout 300 python tools/prof_probe.py 40:40:65536:12 60:60:65536:12 30:30:65536:12 20:20:65536:12 > $O/base_$i.json 2>&1
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_minb.so timeout 300 python tools/prof_probe.py 40:40:65536:12 60:60:65536:12 30:30:65536:12 20:20:65536:12 > $O/minb_$i.json 2>&1
done
timeout 300 python tools/vol_time.py 1 2 3 4 > $O/vol_base.jsonl 2>&1
SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_minb.so timeout 300 python tools/vol_time.py 1 2 3 4 > $O/vol_minb.jsonl 2>&1
echo done > $O/DONE
