#!/bin/bash
# round 2 (session 3): phase-instrumented implicit kernel (clock64 sums per warp, CTA 0), config 2 T=500
cd $GRAFT_REPO_ROOT
O=gpurun_out
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_phase.so timeout 300 python scripts/prof_one.py --config 2 --variant implicit --T 500 --reps 1 > $O/s17_phase.log 2>&1
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_phase.so AB_N=1048576 timeout 300 python scripts/prof_one.py --config 5 --variant implicit --T 10 --n 1048576 --reps 1 > $O/s17_phase5.log 2>&1
cat $O/s17_phase.log; cat $O/s17_phase5.log
