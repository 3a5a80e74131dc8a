#!/bin/bash
# lanczos_t_kernel: first convergence check at 12 / 15 (committed) / 17 / 20 % of md, configs[4] shape and m = 136, same GPU
T=${1:-lt4}; O=gpurun_out/$T; mkdir -p $O
D=$PWD/paper_2010_03817_b200
for i in 1 2; do
  timeout 600 python tools/prof_probe.py 200:200:65536:3 136:136:65536:3 > $O/C15_$i.json 2>> $O/ab.err
  for p in 12 17 20; do
    SPECWALK_LIB=$D/libspecwalk_C$p.so timeout 600 python tools/prof_probe.py 200:200:65536:3 136:136:65536:3 > $O/C${p}_$i.json 2>> $O/ab.err
  done
done
for p in 12 17 20; do
SPECWALK_LIB=$D/libspecwalk_C$p.so timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle_C$p.log 2>&1; echo "exit $?" >> $O/tests_oracle_C$p.log
done
echo done > $O/DONE
