#!/bin/bash
# round 2, call g: A/B pure vs hybrid with the bench protocol; compute-sanitizer racecheck
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python -u scripts/ab_hybrid.py 2 -1 0.25 0.2 0.15 > $O/r02g_ab.log 2>&1; cat $O/r02g_ab.log
bash scripts/gpu_runs/r02_san.sh racecheck
