#!/bin/bash
# round 2 (session 3): HEAD implicit kernel vs the smem-stash boundary-overlap kernel (LSK_PRE 0/1/2)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in old stash2; do
  echo "== $lib" >> $O/s5_ab.log
  export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so
  timeout 300 python scripts/ab_env.py 2 0 off=LSK_PRE:0 after=LSK_PRE:1 inside=LSK_PRE:2 >> $O/s5_ab.log 2>&1
  AB_N=1048576 timeout 300 python scripts/ab_env.py 5 20 off=LSK_PRE:0 inside=LSK_PRE:2 >> $O/s5_ab.log 2>&1
  timeout 300 python scripts/ab_env.py 1 0 off=LSK_PRE:0 inside=LSK_PRE:2 >> $O/s5_ab.log 2>&1
done
cat $O/s5_ab.log | grep -v vs
