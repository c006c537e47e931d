#!/bin/bash
# round 2 (session 3): resident kernel, DSMEM loads pipelined (resnew) vs serialised (resold)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in resold resnew; do
  echo "== $lib" >> $O/s8_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 1 0 g4=LSK_RESG:4 g8=LSK_RESG:8 >> $O/s8_ab.log 2>&1
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so AB_N=1100 timeout 300 python scripts/ab_env.py 1 0 g8=LSK_RESG:8 >> $O/s8_ab.log 2>&1
done
grep -v ' vs ' $O/s8_ab.log
