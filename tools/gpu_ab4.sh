#!/bin/bash
# A = HEAD build, B = working tree: M100 bench rounds (+ per-call / trajectory parity on B)
T=${1:-ab4}; O=gpurun_out/$T; mkdir -p $O
Q="--steps 12 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
for i in 1 2; do
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_A.so timeout 600 python bench.py $Q > $O/bench_A_$i.json 2> $O/bench_A_$i.err
  timeout 600 python bench.py $Q > $O/bench_B_$i.json 2> $O/bench_B_$i.err
done
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -s > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
