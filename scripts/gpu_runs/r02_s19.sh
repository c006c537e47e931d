#!/bin/bash
# round 2 (session 3): ping-pong hand-over row (LSK_PP 1 = after the tile, 2 = after 3/4, 3 = after 1/2)
cd $GRAFT_REPO_ROOT
O=gpurun_out
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_pp.so
timeout 600 python scripts/ab_env.py 2 0 base=LSK_PP:0 pp1=LSK_PP:1 pp2=LSK_PP:2 pp3=LSK_PP:3 > $O/s19_ab.log 2>&1
cat $O/s19_ab.log
