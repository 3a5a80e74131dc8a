#!/bin/bash
# One GPU pass: gpu tests, bench, ncu launch list, one full ncu capture of K2.
# usage (on the box via gpurun): bash tools/gpu_round.sh TAG [skip_tests]
TAG=${1:-x}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
if [ "$2" != "skip_tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"lanczos_kernel|chord_kernel" -s 3 -c 1 -o $O/k2_full \
  python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 > $O/ncu_full.log 2>&1
echo done > $O/DONE
