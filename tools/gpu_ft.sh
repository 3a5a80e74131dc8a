#!/bin/bash
# factor_t_kernel (lower-tile storage, two chains per SM) vs factor_kernel<512>: A/B on the M100
# bench, then the billiard parity tests with factor_t
T=${1:-ft}; O=gpurun_out/$T; mkdir -p $O
SPECWALK_FACTOR_T=1 python -c "import sys; sys.path.insert(0,'.'); import paper_2010_03817_b200 as sw, specgen; S=sw.Spectrahedron.from_instance(specgen.config_instance(3)); print(S.k2_config())" > $O/k2cfg.txt 2>&1
export SPECWALK_PARITY_REPORT=$O/parity
SPECWALK_FACTOR_T=1 timeout 900 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_parity_configs.py -m gpu -q -p no:cacheprovider -s -x -k "m100 or oracle" > $O/tests_quick.log 2>&1; echo "exit $?" >> $O/tests_quick.log
Q="--steps 12 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
for i in 1 2; do
  timeout 600 python bench.py $Q > $O/bench_A_$i.json 2> $O/bench_A_$i.err
  SPECWALK_FACTOR_T=1 timeout 600 python bench.py $Q > $O/bench_B_$i.json 2> $O/bench_B_$i.err
done
echo done > $O/DONE
