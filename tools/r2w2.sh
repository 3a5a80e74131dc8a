#!/bin/bash
# full GPU tests + bench + smoke + CHMC ncu (launch list and a full capture of K7a/K7b)
T=${1:-r2w2}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
B="python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/chmc_launches.csv -k regex:"chmc|gemm|normal" $B > $O/ncu_chmc_launch.log 2>&1
S=/tmp/ncu_$T; mkdir -p $S
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"chmc_chord_kernel|chmc_poly_kernel" -s 6 -c 2 -o $S/chmc_full $B > $O/ncu_chmc_full.log 2>&1
python tools/summarize_ncu.py full $S/chmc_full.ncu-rep $O/chmc_full.txt "configs[2] collocation HMC-r: K7a poly, K7b chord" >> $O/summ.log 2>&1
echo done > $O/DONE
