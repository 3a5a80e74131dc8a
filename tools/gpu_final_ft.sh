#!/bin/bash
# the final factor_t_kernel: ncu --set full + source counters, and the new edge-size parity cases
T=${1:-ftz}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 900 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -s -k "v1_" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
S=/tmp/ncu_$T; mkdir -p $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"factor_t_kernel" -s 3 -c 1 -o $S/ft_full python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0 > $O/ncu.log 2>&1
ncu -i $S/ft_full.ncu-rep --page source --csv --print-source sass > $S/ft_sass.csv 2> $O/src.err
gzip -c $S/ft_sass.csv > $O/factor_t_sass.csv.gz
python tools/summarize_ncu.py full $S/ft_full.ncu-rep $O/ft_full.txt "M100 round 4: factor_t_kernel (final)" > $O/summ.log 2>&1
echo done > $O/DONE
