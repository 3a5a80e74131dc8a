#!/bin/bash
T=${1:-r2n}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1500 python tools/paper_context.py --seeds 2 > $O/paper_context.jsonl 2>&1
echo done > $O/DONE
