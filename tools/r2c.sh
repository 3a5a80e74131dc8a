#!/bin/bash
O=gpurun_out/r2c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hnr.py tests/test_gpu_parity_configs.py -m gpu -q -p no:cacheprovider -k "hnr or per_call" -s > $O/tests_new.log 2>&1; echo "exit $?" >> $O/tests_new.log
for v in base tau13 tau14 tol14 both; do
  if [ $v = base ]; then L=$PWD/paper_2010_03817_b200/libspecwalk.so; else L=$PWD/paper_2010_03817_b200/libspecwalk_$v.so; fi
  SPECWALK_LIB=$L SPECWALK_PARITY_REPORT=$O/$v timeout 600 python -m pytest tests/test_gpu_parity_configs.py -m gpu -q -p no:cacheprovider -k "cfg4 or m100" > $O/traj_$v.log 2>&1
  SPECWALK_LIB=$L timeout 300 python tools/prof_probe.py 200:200:16384:6 100:100:16384:20 > $O/probe_$v.json 2>&1
done
