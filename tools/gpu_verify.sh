#!/bin/bash
# Full GPU verification: every -m gpu test (parity report), the default bench, smoke.
T=${1:-verify}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
echo done > $O/DONE
