#!/bin/bash
# A = HEAD build with SPECWALK_FACTOR_T=1, B = working tree (factor_t default), C = working tree with
# factor_kernel<512> (SPECWALK_FACTOR_T=0); M100 bench rounds; then billiard parity tests on B
T=${1:-ab3}; O=gpurun_out/$T; mkdir -p $O
Q="--steps 12 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
for i in 1 2; do
  SPECWALK_FACTOR_T=1 SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_A.so timeout 600 python bench.py $Q > $O/bench_A_$i.json 2> $O/bench_A_$i.err
  timeout 600 python bench.py $Q > $O/bench_B_$i.json 2> $O/bench_B_$i.err
  SPECWALK_FACTOR_T=0 timeout 600 python bench.py $Q > $O/bench_C_$i.json 2> $O/bench_C_$i.err
done
SPECWALK_PROF=1 timeout 300 python tools/prof_probe.py > $O/prof.txt 2>&1
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_walk.py tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py tests/test_gpu_hnr.py -m gpu -q -p no:cacheprovider -s > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
