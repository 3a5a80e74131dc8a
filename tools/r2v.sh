#!/bin/bash
T=${1:-r2v}; O=gpurun_out/$T; mkdir -p $O
for n in 160 120 100 60; do timeout 600 python tools/dbg_ball.py $n > $O/ball_$n.log 2>&1; done
echo done > $O/DONE
