#!/bin/bash
T=${1:-r2z}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_hmc.py tests/test_gpu_estimators.py -m gpu -q -p no:cacheprovider -s -k "trajectory or m161" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
