#!/bin/bash
# factor_g_kernel with batched branch-free B loads: parity, then K2 phases at m = 200 / 136 (KCH 7 = libspecwalk.so, KCH 9 = _k9)
T=${1:-fg2}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/k7_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_k9.so timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/k9_$i.json 2>> $O/ab.err
done
SPECWALK_PROF=1 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/prof_k7.json 2> $O/prof_k7.err
timeout 600 python tools/prof_probe.py 136:136:65536:3 > $O/m136_k7.json 2>> $O/ab.err
S=/tmp/ncu_$T; mkdir -p $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"factor_g_kernel" -s 2 -c 1 -o $S/fg_full python tools/prof_target.py m200 2 1 > $O/ncu.log 2>&1
python tools/summarize_ncu.py full $S/fg_full.ncu-rep $O/fg_full.txt "configs[4] round 3: factor_g_kernel<384>" > $O/summ.log 2>&1
ncu -i $S/fg_full.ncu-rep --page source --csv --print-source sass > $S/fg_sass.csv 2>> $O/summ.log; gzip -c $S/fg_sass.csv > $O/fg_sass.csv.gz
echo done > $O/DONE
