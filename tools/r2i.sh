#!/bin/bash
# m = 200 (configs[4]) global-scratch K2: 1 vs 2 CTAs per SM, and the per-phase cycle breakdown
T=${1:-r2i}; O=gpurun_out/$T; mkdir -p $O
for i in 1 2; do
  SPECWALK_G_CTAS=1 timeout 300 python tools/prof_probe.py 200:200:65536:3 > $O/g1_$i.json 2>&1
  timeout 300 python tools/prof_probe.py 200:200:65536:3 > $O/g2_$i.json 2>&1
done
SPECWALK_PROF=1 timeout 300 python tools/prof_probe.py 200:200:16384:3 > $O/prof_m200.json 2> $O/prof_m200.err
SPECWALK_PROF=1 timeout 300 python tools/prof_probe.py 100:100:16384:6 > $O/prof_m100.json 2> $O/prof_m100.err
echo done > $O/DONE
# HMC-r: lanczos2 (full Gram-Schmidt per iteration) vs the register-resident kernel
timeout 900 python -m pytest tests/test_gpu_hmc.py tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -s -k "hmc" > $O/hmc_tests.log 2>&1; echo "exit $?" >> $O/hmc_tests.log
for i in 1 2; do
  SPECWALK_HMC_LZ_OLD=1 timeout 600 python bench.py --steps 2 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --m200-rounds 0 > $O/hmc_old_$i.json 2>&1
  timeout 600 python bench.py --steps 2 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --m200-rounds 0 > $O/hmc_new_$i.json 2>&1
done
echo done2 > $O/DONE2
