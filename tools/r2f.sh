#!/bin/bash
T=${1:-r2f}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
F="ncu --set full --clock-control none --import-source on"
S=/tmp/ncu_$T; mkdir -p $S
python tools/prof_target.py m100 3 1 > $O/pt_m100.log 2>&1 && timeout 1200 $F -k regex:"lanczos2_kernel" -s 3 -c 1 -o $S/lz2 python tools/prof_target.py m100 3 1 > $O/ncu_lz2.log 2>&1
python tools/summarize_ncu.py full $S/lz2.ncu-rep $O/lz2_full.txt "M100 round 4: lanczos2_kernel (two chains per SM)" >> $O/summ.log 2>&1
ncu -i $S/lz2.ncu-rep --page source --csv --print-source sass > $S/lz2_sass.csv 2>> $O/summ.log; gzip -c $S/lz2_sass.csv > $O/lz2_sass.csv.gz
du -sh $O >> $O/summ.log
echo done > $O/DONE
