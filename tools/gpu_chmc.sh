#!/bin/bash
# collocation HMC-r GPU tests (+ the existing HMC ones as a regression check)
T=${1:-chmc}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_chmc.py -m gpu -q -p no:cacheprovider -s -x > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
