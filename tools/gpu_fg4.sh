#!/bin/bash
# A = libspecwalk.so (committed); P5 = factor_g congruence stage 1 software-pipelined (batches of 5, two register buffers);
# T4 = tail_kernel with 4 CTAs/SM (64 registers).  Parity with P5 at m > 112, then same-GPU A/B.
T=${1:-fg4}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
D=$PWD/paper_2010_03817_b200
SPECWALK_LIB=$D/libspecwalk_P5.so timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
SPECWALK_LIB=$D/libspecwalk_P5.so timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/A200_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$D/libspecwalk_P5.so timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/P5_200_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$D/libspecwalk_T4.so timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/T4_200_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 100:100:65536:12 > $O/A100_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$D/libspecwalk_T4.so timeout 600 python tools/prof_probe.py 100:100:65536:12 > $O/T4_100_$i.json 2>> $O/ab.err
done
SPECWALK_LIB=$D/libspecwalk_P5.so SPECWALK_PROF=1 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/prof_P5.json 2> $O/prof_P5.err
echo done > $O/DONE
