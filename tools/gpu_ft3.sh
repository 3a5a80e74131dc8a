#!/bin/bash
T=${1:-ft3}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
Q="--steps 12 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
timeout 600 python bench.py $Q > $O/bench_B.json 2> $O/bench_B.err
SPECWALK_PROF=1 timeout 300 python tools/prof_probe.py > $O/prof.txt 2>&1
echo done > $O/DONE
