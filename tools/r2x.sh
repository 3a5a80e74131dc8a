#!/bin/bash
T=${1:-r2x}; O=gpurun_out/$T; mkdir -p $O
timeout 600 python tools/dbg_ball2.py 100 > $O/ball100_lz2.log 2>&1
for n in 100 160; do timeout 600 python tools/dbg_ball.py $n > $O/ball_$n.log 2>&1; done
timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/probe.json 2>&1
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_hmc.py tests/test_gpu_parity_configs.py tests/test_gpu_oracle.py tests/test_gpu_estimators.py -m gpu -q -p no:cacheprovider -s > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
echo done > $O/DONE
