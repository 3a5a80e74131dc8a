#!/bin/bash
# factor_g_kernel: W = L^-1 with four DMMA chains per tile and the Cholesky's trailing update two tiles per warp step
# (libspecwalk_B.so) against the committed build (libspecwalk.so): parity with B, then same-GPU A/B
T=${1:-fg3}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
B=$PWD/paper_2010_03817_b200/libspecwalk_B.so
SPECWALK_LIB=$B timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
SPECWALK_LIB=$B timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/A_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$B timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/B_$i.json 2>> $O/ab.err
done
SPECWALK_LIB=$B SPECWALK_PROF=1 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/prof_B.json 2> $O/prof_B.err
SPECWALK_LIB=$B timeout 600 python tools/prof_probe.py 136:136:65536:3 > $O/m136_B.json 2>> $O/ab.err
echo done > $O/DONE
