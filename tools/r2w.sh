#!/bin/bash
T=${1:-r2w}; O=gpurun_out/$T; mkdir -p $O
timeout 600 python tools/dbg_ball2.py 100 > $O/ball100_lz2.log 2>&1
SPECWALK_LZ_OLD=1 timeout 600 python tools/dbg_ball2.py 100 > $O/ball100_old.log 2>&1
SPECWALK_K2_FUSED=1 timeout 600 python tools/dbg_ball2.py 100 > $O/ball100_fused.log 2>&1
SPECWALK_LZ_OLD=1 timeout 600 python tools/dbg_ball.py 100 > $O/ball100_old_walk.log 2>&1
echo done > $O/DONE
