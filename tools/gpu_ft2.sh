#!/bin/bash
# factor_t_kernel default: all GPU tests, then its ncu capture with source counters
T=${1:-ft2}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
python -c "import sys; sys.path.insert(0,'.'); import paper_2010_03817_b200 as sw, specgen; S=sw.Spectrahedron.from_instance(specgen.config_instance(3)); print(S.k2_config())" > $O/k2cfg.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
S=/tmp/ncu_$T; mkdir -p $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"factor_t_kernel" -s 3 -c 1 -o $S/ft_full python bench.py --steps 1 --warmup 3 --cpu-seconds 0 --volume-seeds 0 --e2e-chains 0 --hmc-rounds 0 --m200-rounds 0 --chmc-rounds 0 > $O/ncu.log 2>&1
ncu -i $S/ft_full.ncu-rep --page source --csv --print-source sass > $S/ft_sass.csv 2> $O/src.err
gzip -c $S/ft_sass.csv > $O/factor_t_sass.csv.gz
python tools/summarize_ncu.py full $S/ft_full.ncu-rep $O/ft_full.txt "M100 round 4: factor_t_kernel" > $O/summ.log 2>&1
SPECWALK_PROF=1 timeout 300 python tools/prof_probe.py > $O/prof.txt 2>&1
echo done > $O/DONE
