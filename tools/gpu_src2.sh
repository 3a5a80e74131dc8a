#!/bin/bash
# source-level capture (stalls + shared-memory excess wavefronts) of lanczos2_kernel and tail_kernel
T=${1:-src2}; O=gpurun_out/$T; mkdir -p $O
S=/tmp/ncu_$T; mkdir -p $S
B="python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lanczos2_kernel|tail_kernel" -s 6 -c 2 -o $S/lt_full $B > $O/ncu.log 2>&1
ncu -i $S/lt_full.ncu-rep --page source --csv --print-source sass -k regex:lanczos2_kernel > $S/lz2.csv 2> $O/src.err
ncu -i $S/lt_full.ncu-rep --page source --csv --print-source sass -k regex:tail_kernel > $S/tail.csv 2>> $O/src.err
gzip -c $S/lz2.csv > $O/lanczos2_sass.csv.gz; gzip -c $S/tail.csv > $O/tail_sass.csv.gz
python tools/summarize_ncu.py full $S/lt_full.ncu-rep $O/lt_full.txt "M100 round 4: lanczos2_kernel, tail_kernel" > $O/summ.log 2>&1
echo done > $O/DONE
