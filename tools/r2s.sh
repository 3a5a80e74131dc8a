#!/bin/bash
T=${1:-r2s}; O=gpurun_out/$T; mkdir -p $O
for i in 1 2; do
  for v in base ub ubns; do
    if [ $v = base ]; then L=$PWD/paper_2010_03817_b200/libspecwalk.so; else L=$PWD/paper_2010_03817_b200/libspecwalk_$v.so; fi
    SPECWALK_LIB=$L timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/${v}_$i.json 2>&1
  done
done
SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_ubns.so SPECWALK_PARITY_REPORT=$O/parity timeout 900 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_oracle.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "m100 or rand_100 or v1_ or bench_configuration" > $O/tests_ubns.log 2>&1
echo done > $O/DONE
