#!/bin/bash
# round 2 (session 3): phase-instrumented implicit kernel with the ping-pong (CTA 0), config 2 T=500
cd $GRAFT_REPO_ROOT
O=gpurun_out
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_phase2.so timeout 300 python scripts/prof_one.py --config 2 --variant implicit --T 500 --reps 1 > $O/s23_phase.log 2>&1
cat $O/s23_phase.log
