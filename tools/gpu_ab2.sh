#!/bin/bash
# A (HEAD build) vs B (working tree) at small m (fused chord kernel, m = 40, 20), collocation HMC-r,
# HMC-r fused (m = 136); then the GPU tests that exercise the changed tile code
T=${1:-ab2}; O=gpurun_out/$T; mkdir -p $O
for i in 1 2; do
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_A.so timeout 300 python tools/probe.py 40:40:65536:2 20:20:65536:3 > $O/probe_A_$i.txt 2>&1
  timeout 300 python tools/probe.py 40:40:65536:2 20:20:65536:3 > $O/probe_B_$i.txt 2>&1
  SPECWALK_LIB=$PWD/paper_2010_03817_b200/libspecwalk_A.so timeout 300 python tools/probe_chmc.py > $O/chmc_A_$i.txt 2>&1
  timeout 300 python tools/probe_chmc.py > $O/chmc_B_$i.txt 2>&1
done
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_walk.py tests/test_gpu_hmc.py tests/test_gpu_chmc.py tests/test_gpu_estimators.py tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -s > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
