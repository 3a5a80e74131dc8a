#!/bin/bash
# final evidence at HEAD: every -m gpu test (parity report), smoke, the default bench, the launch list over the
# bench's timed rounds, and ncu --set full of the hot kernels at M100 and configs[4]
T=${1:-r2z}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
B="python bench.py --steps 5 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
$B > $O/bench_short.json 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
python tools/summarize_launches.py $O/launches.csv 3 > $O/launches_timed.txt 2>&1
F="ncu --set full --clock-control none --import-source on"
S=/tmp/ncu_$T; mkdir -p $S
python tools/prof_target.py m100 3 1 > $O/pt_m100.log 2>&1 && timeout 1200 $F -k regex:"gemm_f64_dmma|factor_t_kernel|factor_kernel|lanczos2_kernel|tail_kernel" -s 16 -c 5 -o $S/m100_full python tools/prof_target.py m100 3 1 > $O/ncu_m100.log 2>&1
python tools/summarize_ncu.py full $S/m100_full.ncu-rep $O/m100_full.txt "M100 round 4: K1, factor_t, lanczos2, tail, K3" >> $O/summ.log 2>&1
python tools/prof_target.py m200 2 1 > $O/pt_m200.log 2>&1 && timeout 1500 $F -k regex:"factor_g_kernel|lanczos_t_kernel|tail_kernel" -s 6 -c 3 -o $S/m200_full python tools/prof_target.py m200 2 1 > $O/ncu_m200.log 2>&1
python tools/summarize_ncu.py full $S/m200_full.ncu-rep $O/m200_full.txt "configs[4] round 3: factor_g_kernel<384>, lanczos_t_kernel, tail_kernel" >> $O/summ.log 2>&1
ncu -i $S/m200_full.ncu-rep --page source --csv --print-source sass -k regex:factor_g_kernel > $S/ck2_sass.csv 2>> $O/summ.log; gzip -c $S/ck2_sass.csv > $O/m200_factor_sass.csv.gz
du -sh $O >> $O/summ.log
echo done > $O/DONE
