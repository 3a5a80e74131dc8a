#!/bin/bash
T=${1:-r2u}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_hmc.py tests/test_gpu_parity_configs.py tests/test_gpu_estimators.py -m gpu -q -p no:cacheprovider -s -k "trajectory or m161 or elliptope" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
timeout 1800 python tools/elliptope_volume.py 20:1:2048:0.15 > $O/elliptope20.jsonl 2>&1
echo done > $O/DONE
