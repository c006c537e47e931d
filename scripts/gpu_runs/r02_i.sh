#!/bin/bash
# round 2, call i: one full capture of the tensor-core exponent kernel (phase-split version)
cd $GRAFT_REPO_ROOT
O=gpurun_out
CMD="python scripts/prof_one.py --config 2 --variant implicit --T 20 --reps 2"
timeout 300 $CMD > $O/r02i_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:itc_kernel -s 1 -c 1 -o $O/r02i_itc -f $CMD > $O/r02i_ncu.log 2>&1
echo "ncu rc=$?"; tail -1 $O/r02i_ncu.log
