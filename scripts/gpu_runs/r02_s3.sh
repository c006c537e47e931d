#!/bin/bash
# round 2 (session 3): HEAD implicit kernel vs the peeled boundary-overlap kernel (LSK_PRE 0/2)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in old new; do
  echo "== $lib" >> $O/s3_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 2 0 off=LSK_PRE:0 after=LSK_PRE:1 inside=LSK_PRE:2 >> $O/s3_ab.log 2>&1
done
cat $O/s3_ab.log
