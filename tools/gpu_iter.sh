#!/bin/bash
# build-test-measure loop on the box: bash tools/gpu_iter.sh TAG TESTS(ALL|NONE|-k expr) probe-args...
TAG=$1; shift; K=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
if [ "$K" != "NONE" ]; then
  if [ "$K" == "ALL" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1
  else timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > $O/gpu_tests.log 2>&1; fi
  echo "exit $?" >> $O/gpu_tests.log
fi
if [ $# -gt 0 ]; then
  timeout 600 python tools/prof_probe.py "$@" > $O/noprof.json 2> $O/noprof.err
  cp paper_2010_03817_b200/libspecwalk.so /tmp/libspecwalk.keep.so
  SPECWALK_DEFS=-DSW_PROF_LANCZOS=1 python -c "from paper_2010_03817_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
  SPECWALK_PROF=1 timeout 900 python tools/prof_probe.py "$@" > $O/prof.json 2> $O/prof.err
  cp /tmp/libspecwalk.keep.so paper_2010_03817_b200/libspecwalk.so
fi
echo done > $O/DONE
