#!/bin/bash
# round 2 (session 3): point rows loaded one row ahead in the feature generation (xpf) vs not
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in tuning xpf tuning xpf; do
  echo "== $lib" >> $O/s24_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 2 0 pp=LSK_PP:1 2>&1 | grep 'config' >> $O/s24_ab.log
done
cat $O/s24_ab.log
