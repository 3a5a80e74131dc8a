#!/bin/bash
T=${1:-r2h}; O=gpurun_out/$T; mkdir -p $O
export SPECWALK_PARITY_REPORT=$O/parity
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python tools/elliptope_volume.py 5:3 8:2 12:2 20:2 > $O/elliptope_volume.jsonl 2>&1
timeout 600 python tools/prof_probe.py 100:100:65536:12 72:72:65536:12 60:60:65536:12 40:40:65536:12 > $O/probe.json 2>&1
echo done > $O/DONE
