#!/bin/bash
# round 2, call h: A/B of the tensor-core exponent kernel, then one full capture of it
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python scripts/ab_tc.py 2 200 > $O/r02h_ab.log 2>&1; tail -6 $O/r02h_ab.log
CMD="python scripts/prof_one.py --config 2 --variant implicit --T 20 --reps 2"
timeout 300 $CMD > $O/r02h_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:itc_kernel -s 1 -c 1 -o $O/r02h_itc -f $CMD > $O/r02h_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 $O/r02h_ncu.log
