#!/bin/bash
# round 2 (session 3): two-generation tile loop (GEN2) A/B on config 2 and config 5 (reduced)
cd $GRAFT_REPO_ROOT
O=gpurun_out
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_g2.so
timeout 600 python scripts/ab_env.py 2 0 base=LSK_PRE:2 g1=LSK_ICFG:128,4,2,16,0,1 g2=LSK_ICFG:128,4,2,16,0,2 g3=LSK_ICFG:128,4,2,16,0,3 g4=LSK_ICFG:128,4,2,16,0,4 t3g2=LSK_ICFG:128,3,2,16,0,2 r32g2=LSK_ICFG:128,4,2,32,0,2 r32g3=LSK_ICFG:128,4,2,32,0,3 > $O/s13_ab.log 2>&1
cat $O/s13_ab.log
