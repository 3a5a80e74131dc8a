#!/bin/bash
# factor2_kernel (two chains per SM) A/B against factor_kernel<512> + the M100/billiard parity tests
T=${1:-f2}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
SPECWALK_FACTOR2=1 python -c "import sys; sys.path.insert(0,'.'); import paper_2010_03817_b200 as sw, specgen; S=sw.Spectrahedron.from_instance(specgen.config_instance(3)); print(S.k2_config())" > $O/k2cfg.txt 2>&1
Q="--steps 12 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
for i in 1 2; do
  timeout 600 python bench.py $Q > $O/bench_f1_$i.json 2> $O/bench_f1_$i.err
  SPECWALK_FACTOR2=1 timeout 600 python bench.py $Q > $O/bench_f2_$i.json 2> $O/bench_f2_$i.err
done
SPECWALK_FACTOR2=1 timeout 1500 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_walk.py tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py tests/test_gpu_hnr.py -m gpu -q -p no:cacheprovider -s -x > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
B="python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 2"
S=/tmp/ncu_$T; mkdir -p $S
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"chmc_chord_kernel|chmc_poly_kernel" -s 6 -c 2 -o $S/chmc_full $B > $O/ncu_chmc_full.log 2>&1
python tools/summarize_ncu.py full $S/chmc_full.ncu-rep $O/chmc_full.txt "configs[2] collocation HMC-r: K7a poly, K7b chord (one timed round)" >> $O/summ.log 2>&1
SPECWALK_FACTOR2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"factor2_kernel" -s 3 -c 1 -o $S/f2_full python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0 > $O/ncu_f2_full.log 2>&1
python tools/summarize_ncu.py full $S/f2_full.ncu-rep $O/f2_full.txt "M100 round 4: factor2_kernel" >> $O/summ.log 2>&1
echo done > $O/DONE
