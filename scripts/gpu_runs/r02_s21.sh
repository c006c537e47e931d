#!/bin/bash
# round 2 (session 3): s staged before the stopping-test barrier (stage) vs after it (tuning)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in tuning stage tuning stage; do
  echo "== $lib" >> $O/s21_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 2 0 pp=LSK_PP:1 >> $O/s21_ab.log 2>&1
done
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_stage.so AB_N=6151 timeout 300 python scripts/ab_env.py 5 60 d=LSK_PP:1 >> $O/s21_ab.log 2>&1
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so AB_N=6151 timeout 300 python scripts/ab_env.py 5 60 d=LSK_PP:1 >> $O/s21_ab.log 2>&1
cat $O/s21_ab.log
