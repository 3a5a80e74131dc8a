#!/bin/bash
T=${1:-c5}; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chmc.py -m gpu -q -p no:cacheprovider -s -x > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
timeout 600 python tools/probe_chmc.py > $O/probe.txt 2>&1; echo "exit $?" >> $O/probe.txt
SPECWALK_CHMC_512=1 timeout 600 python tools/probe_chmc.py > $O/probe_512.txt 2>&1; echo "exit $?" >> $O/probe_512.txt
echo done > $O/DONE
