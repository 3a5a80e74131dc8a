#!/bin/bash
# quick loop on the box: gpu tests (optional filter) + K2 phase probe
# usage: bash tools/gpu_quick.sh TAG "pytest -k expr or ALL or NONE" probe-args...
TAG=$1; shift; K=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
if [ "$K" != "NONE" ]; then
  if [ "$K" == "ALL" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1
  else timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > $O/gpu_tests.log 2>&1; fi
  echo "exit $?" >> $O/gpu_tests.log
fi
if [ $# -gt 0 ]; then
  SPECWALK_PROF=1 timeout 900 python tools/prof_probe.py "$@" > $O/prof.json 2> $O/prof.err
  timeout 600 python tools/prof_probe.py "$@" > $O/noprof.json 2> $O/noprof.err
fi
echo done > $O/DONE
