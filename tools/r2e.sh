#!/bin/bash
# lanczos2 (two chains per SM) vs the register-resident lanczos_kernel: parity tests + A/B probes
T=${1:-r2e}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1500 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_parity_configs.py tests/test_gpu_walk.py tests/test_gpu_fullsize.py tests/test_gpu_hnr.py -m gpu -q -p no:cacheprovider -s -k "not configs2_instance and not vs_oracle_rand_cube_10 and not m200 and not cfg4" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
for i in 1 2; do
  SPECWALK_LZ_OLD=1 timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/probe_old_$i.json 2>&1
  timeout 300 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 > $O/probe_new_$i.json 2>&1
done
echo done > $O/DONE
