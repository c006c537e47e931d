#!/bin/bash
# round 2 (session 3): polling back-off A/B (group barrier LSK_BAR_NS, svec LSK_SV_NS)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in tuning b32 s32 b32s32 tuning b32 s32 b32s32; do
  echo "== $lib" >> $O/s22_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 2 0 pp=LSK_PP:1 2>&1 | grep 'config' >> $O/s22_ab.log
done
cat $O/s22_ab.log
