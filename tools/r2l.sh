#!/bin/bash
T=${1:-r2l}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python tools/e2e_probe.py 16384:1 65536:1 16384:4 32768:2 > $O/e2e_probe.jsonl 2>&1
echo done > $O/DONE
