#!/bin/bash
# A = libspecwalk.so (pipelined batches of 5, stage 2 two tiles at a time); S4 = stage 2 four tiles at a time;
# P7 = pipelined batches of 7; A256 = A with 256 threads.  Parity with S4 and P7 at m > 112, then same-GPU A/B.
T=${1:-fg5}; O=gpurun_out/$T; mkdir -p $O
D=$PWD/paper_2010_03817_b200
for v in S4 P7; do
SPECWALK_LIB=$D/libspecwalk_$v.so timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle_$v.log 2>&1; echo "exit $?" >> $O/tests_oracle_$v.log
done
SPECWALK_LIB=$D/libspecwalk_S4.so timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4_S4.log 2>&1; echo "exit $?" >> $O/tests_cfg4_S4.log
for i in 1 2; do
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/A_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$D/libspecwalk_S4.so timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/S4_$i.json 2>> $O/ab.err
  SPECWALK_LIB=$D/libspecwalk_P7.so timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/P7_$i.json 2>> $O/ab.err
  SPECWALK_G_FACTOR=256 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/A256_$i.json 2>> $O/ab.err
done
echo done > $O/DONE
