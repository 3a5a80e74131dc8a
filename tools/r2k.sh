#!/bin/bash
T=${1:-r2k}; O=gpurun_out/$T; mkdir -p $O
for i in 1 2; do
  SPECWALK_G_FUSED=1 timeout 300 python tools/prof_probe.py 200:200:65536:3 136:136:65536:4 > $O/fused_$i.json 2>&1
  timeout 300 python tools/prof_probe.py 200:200:65536:3 136:136:65536:4 > $O/split_$i.json 2>&1
done
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 > $O/bench_m200.json 2>&1
echo done > $O/DONE
