#!/bin/bash
# m > 152 split: tail_kernel<512> (one CTA per SM) against tail_kernel<256> (SPECWALK_T512=0), same library, same GPU
T=${1:-t512}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 1200 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "200 or 136 or 120 or 113 or 201 or 208" > $O/tests_oracle.log 2>&1; echo "exit $?" >> $O/tests_oracle.log
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "cfg4 or (m200 and billiard) or m200_configs4" > $O/tests_cfg4.log 2>&1; echo "exit $?" >> $O/tests_cfg4.log
for i in 1 2; do
  SPECWALK_T512=0 timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/t256_$i.json 2>> $O/ab.err
  timeout 600 python tools/prof_probe.py 200:200:65536:3 > $O/t512_$i.json 2>> $O/ab.err
done
echo done > $O/DONE
