#!/bin/bash
# factor_kernel source-level capture (stalls + shared-memory excessive wavefronts per SASS line)
T=${1:-fsrc}; O=gpurun_out/$T; mkdir -p $O
S=/tmp/ncu_$T; mkdir -p $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"factor_kernel" -s 3 -c 1 -o $S/f_full python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0 > $O/ncu.log 2>&1
ncu -i $S/f_full.ncu-rep --page source --csv --print-source sass > $S/f_sass.csv 2> $O/src.err
gzip -c $S/f_sass.csv > $O/factor_sass.csv.gz
python tools/summarize_ncu.py full $S/f_full.ncu-rep $O/f_full.txt "M100 round 4: factor_kernel" > $O/summ.log 2>&1
echo done > $O/DONE
