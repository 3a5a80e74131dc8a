#!/bin/bash
# final evidence: launch list over the bench's timed rounds + ncu --set full of every hot kernel
T=${1:-r2o}; O=gpurun_out/$T; mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0"
$B > $O/bench_short.json 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
python tools/summarize_launches.py $O/launches.csv 3 > $O/launches_timed.txt 2>&1
F="ncu --set full --clock-control none --import-source on"
S=/tmp/ncu_$T; mkdir -p $S
python tools/prof_target.py m100 3 1 > $O/pt_m100.log 2>&1 && timeout 1200 $F -k regex:"gemm_f64_dmma|factor_t_kernel|factor_kernel|lanczos2_kernel|tail_kernel" -s 16 -c 5 -o $S/m100_full python tools/prof_target.py m100 3 1 > $O/ncu_m100.log 2>&1
python tools/summarize_ncu.py full $S/m100_full.ncu-rep $O/m100_full.txt "M100 round 4: K1, factor, lanczos2, tail, K3" >> $O/summ.log 2>&1
ncu -i $S/m100_full.ncu-rep --page source --csv --print-source sass -k regex:lanczos2_kernel > $S/lz2_sass.csv 2>> $O/summ.log; gzip -c $S/lz2_sass.csv > $O/lanczos2_sass.csv.gz
ncu -i $S/m100_full.ncu-rep --page source --csv --print-source sass -k regex:factor_kernel > $S/factor_sass.csv 2>> $O/summ.log; gzip -c $S/factor_sass.csv > $O/factor_sass.csv.gz
python tools/prof_target.py hmc 2 1 > $O/pt_hmc.log 2>&1 && timeout 1500 $F -k regex:"hmc_factor_kernel|lanczos2_kernel|hmc_weyl_kernel|hmc_tail_kernel|hmc_setup_kernel" -s 30 -c 5 -o $S/hmc_full python tools/prof_target.py hmc 2 1 > $O/ncu_hmc.log 2>&1
python tools/summarize_ncu.py full $S/hmc_full.ncu-rep $O/hmc_full.txt "configs[3] HMC-r round 2: setup/factor/lanczos2/weyl/tail" >> $O/summ.log 2>&1
python tools/prof_target.py m200 2 1 > $O/pt_m200.log 2>&1 && timeout 1200 $F -k regex:"chord_kernel2" -s 2 -c 1 -o $S/m200_full python tools/prof_target.py m200 2 1 > $O/ncu_m200.log 2>&1
python tools/summarize_ncu.py full $S/m200_full.ncu-rep $O/m200_full.txt "configs[4] round 3: chord_kernel2<512,false,16>" >> $O/summ.log 2>&1
C="python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 2"
timeout 1200 $F -k regex:"chmc_chord_kernel|chmc_poly_kernel" -s 6 -c 2 -o $S/chmc_full $C > $O/ncu_chmc.log 2>&1
python tools/summarize_ncu.py full $S/chmc_full.ncu-rep $O/chmc_full.txt "configs[2] collocation HMC-r round 4: K7a poly, K7b chord" >> $O/summ.log 2>&1
du -sh $O >> $O/summ.log
echo done > $O/DONE
