#!/bin/bash
# factor_g_kernel (m > 112 factor phase, G/L/W tiles in shared memory): parity at m = 120/136/200 and configs[4],
# then same-GPU A/B against the global-scratch factor phase (SPECWALK_G_FACTOR=0) and the 256-thread variant
T=${1:-fg}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  SPECWALK_G_FACTOR=0 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/old_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/fg384_$i.json 2>> $O/ab.err
  SPECWALK_G_FACTOR=256 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/fg256_$i.json 2>> $O/ab.err
done
SPECWALK_PROF=1 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/prof384.json 2> $O/prof384.err
timeout 600 python tools/prof_probe.py 136:136:65536:3 > $O/m136_fg.json 2>> $O/ab.err
SPECWALK_G_FACTOR=0 timeout 600 python tools/prof_probe.py 136:136:65536:3 > $O/m136_old.json 2>> $O/ab.err
echo done > $O/DONE
