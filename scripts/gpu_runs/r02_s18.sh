#!/bin/bash
# round 2 (session 3): ping-pong team scheduling (alternating feature generations) A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so
timeout 600 python scripts/ab_env.py 2 0 base=LSK_PP:0 pp=LSK_PP:1 pp_nopre=LSK_PP:1+LSK_PRE:0 > $O/s18_ab.log 2>&1
AB_N=6151 timeout 300 python scripts/ab_env.py 2 61 base=LSK_PP:0 pp=LSK_PP:1 >> $O/s18_ab.log 2>&1
AB_N=4099 timeout 300 python scripts/ab_env.py 2 60 base=LSK_PP:0 pp=LSK_PP:1 >> $O/s18_ab.log 2>&1
cat $O/s18_ab.log
