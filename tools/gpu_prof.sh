#!/bin/bash
# K2 phase breakdown on the box: bash tools/gpu_prof.sh TAG [probe args]
TAG=${1:-p}; shift
O=gpurun_out/$TAG; mkdir -p $O
SPECWALK_PROF=1 timeout 900 python tools/prof_probe.py "$@" > $O/prof.json 2> $O/prof.err
timeout 600 python tools/prof_probe.py "$@" > $O/noprof.json 2> $O/noprof.err
echo done > $O/DONE
