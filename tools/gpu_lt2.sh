#!/bin/bash
# lanczos_t_kernel: parity at m = 120..200, A/B vs the fused kernel, factor phase with 1 CTA/SM
T=${1:-lt2}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  SPECWALK_G_SPLIT=0 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/fused_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/lt_$i.json 2>> $O/ab.err
  SPECWALK_G_CTAS=1 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/lt_g1_$i.json 2>> $O/ab.err
done
SPECWALK_PROF=1 timeout 600 python tools/prof_probe.py 200:200:16384:3 > $O/prof.json 2> $O/prof.err
echo done > $O/DONE
