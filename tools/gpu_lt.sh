#!/bin/bash
# m > 112 split with lanczos_t_kernel: parity at m = 120..200 and an A/B of the K2 phases at m = 200
T=${1:-lt1}; O=gpurun_out/$T; mkdir -p $O
timeout 300 python tools/prof_probe.py 200:200:8192:2 > $O/smoke_probe.json 2> $O/smoke_probe.err
echo "probe exit $?" >> $O/smoke_probe.err
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  SPECWALK_G_SPLIT=0 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/fused_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/lt_$i.json 2>> $O/ab.err
done
echo done > $O/DONE
