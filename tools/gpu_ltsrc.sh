#!/bin/bash
# lanczos_t_kernel: A/B vs the fused m = 200 kernel and a source-level ncu capture
T=${1:-ltsrc}; O=gpurun_out/$T; mkdir -p $O
S=/tmp/ncu_$T; mkdir -p $S
for i in 1 2; do
  SPECWALK_G_SPLIT=0 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/fused_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/lt_$i.json 2>> $O/ab.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lanczos_t_kernel" -s 2 -c 1 -o $S/lt_full python tools/prof_target.py m200 2 1 > $O/ncu.log 2>&1
ncu -i $S/lt_full.ncu-rep --page source --csv --print-source sass > $S/lt_sass.csv 2> $O/src.err
gzip -c $S/lt_sass.csv > $O/lt_sass.csv.gz
python tools/summarize_ncu.py full $S/lt_full.ncu-rep $O/lt_full.txt "m200 round: lanczos_t_kernel" > $O/summ.log 2>&1
echo done > $O/DONE
