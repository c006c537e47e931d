#!/bin/bash
# round 2 (session 3): Alg. 2 factor passes with a per-warp cp.async double buffer (cpa)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in tuning cpa tuning cpa; do
  echo "== $lib" >> $O/s16_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 600 python scripts/ab_accel.py 2 100 2>&1 | grep 'graph ' | head -1 >> $O/s16_ab.log
done
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_cpa.so timeout 600 python scripts/ab_accel.py 1 200 2>&1 | grep 'graph ' >> $O/s16_ab.log
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so timeout 600 python scripts/ab_accel.py 1 200 2>&1 | grep 'graph ' >> $O/s16_ab.log
cat $O/s16_ab.log
