#!/bin/bash
# round 2 (session 3): Alg. 2 factor passes with an L2 prefetch LSK_ACCEL_PF row batches ahead
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in tuning pf1 pf2 pf4 tuning; do
  echo "== $lib" >> $O/s15_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 600 python scripts/ab_accel.py 2 100 2>&1 | grep graph | head -1 >> $O/s15_ab.log
done
cat $O/s15_ab.log
