#!/bin/bash
# A = libspecwalk_A.so (M as full rows), B = libspecwalk.so (M as lower tiles from the factor phase)
T=${1:-lt3}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_A.so timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/A_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/B_$i.json 2>> $O/ab.err
done
echo done > $O/DONE
