#!/bin/bash
# m > 112 split (factor phase, lanczos_cl_kernel 2-CTA cluster, tail; opt-in SPECWALK_G_SPLIT=1) vs the fused kernel
T=${1:-r2j}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
python -c "
import paper_2010_03817_b200 as sw, specgen
for k in (4,):
    S = sw.Spectrahedron.from_instance(specgen.config_instance(k)); print(S.k2_config())
S = sw.Spectrahedron.from_instance(specgen.rand_cube(10, 136, 16)); print(S.k2_config())
" > $O/config.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_oracle.py tests/test_gpu_parity_configs.py tests/test_gpu_fullsize.py tests/test_gpu_hnr.py -m gpu -q -p no:cacheprovider -s -k "200 or cfg4 or v2_ or v3_ or m200" > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
for i in 1 2; do
  SPECWALK_G_FUSED=1 timeout 300 python tools/prof_probe.py 200:200:65536:3 136:136:65536:4 > $O/fused_$i.json 2>&1
  timeout 300 python tools/prof_probe.py 200:200:65536:3 136:136:65536:4 > $O/split_$i.json 2>&1
done
echo done > $O/DONE
