#!/bin/bash
T=${1:-traj}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1800 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_walk.py tests/test_gpu_chmc.py tests/test_gpu_hmc.py -m gpu -q -p no:cacheprovider -s > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
