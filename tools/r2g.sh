#!/bin/bash
T=${1:-r2g}; O=gpurun_out/$T; mkdir -p $O
for v in base t10 t11 t12; do
  if [ $v = base ]; then L=$PWD/paper_2010_03817_b200/libspecwalk.so; else L=$PWD/paper_2010_03817_b200/libspecwalk_$v.so; fi
  SPECWALK_LIB=$L SPECWALK_PARITY_REPORT=$O/$v timeout 900 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_oracle.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "m100 or v1_ or rand_100 or rand_20_72 or bench_configuration" > $O/tests_$v.log 2>&1
  SPECWALK_LIB=$L timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/probe_$v.json 2>&1
done
SPECWALK_LZ_OLD=1 timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/probe_old.json 2>&1
echo done > $O/DONE
