#!/bin/bash
# round 2 (session 3): team 0's second pre-generated tile (stash B; XS = 2 slot layout) A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_sb.so
timeout 600 python scripts/ab_env.py 2 0 base=LSK_STASHB:0 sb=LSK_STASHB:1 > $O/s26_ab.log 2>&1
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so timeout 600 python scripts/ab_env.py 2 0 tuning=LSK_PP:1 >> $O/s26_ab.log 2>&1
AB_N=4099 timeout 300 python scripts/ab_env.py 2 60 base=LSK_STASHB:0 sb=LSK_STASHB:1 >> $O/s26_ab.log 2>&1
cat $O/s26_ab.log
