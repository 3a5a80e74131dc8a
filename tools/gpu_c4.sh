#!/bin/bash
# collocation HMC-r tests + probe, then the elliptope k = 20 volume pin (n = 190)
T=${1:-c4}; O=gpurun_out/$T; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chmc.py -m gpu -q -p no:cacheprovider -s -x > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
timeout 600 python tools/probe_chmc.py > $O/probe.txt 2>&1; echo "exit $?" >> $O/probe.txt
timeout 1500 python tools/elliptope_volume.py 20:1:1024:0.2 > $O/elliptope20.jsonl 2> $O/elliptope20.err; echo "exit $?" >> $O/elliptope20.err
echo done > $O/DONE
