#!/bin/bash
# round 2 (session 3): boundary-overlap A/B (LSK_PRE 0/1/2) on config 2, implicit parity tests
cd $GRAFT_REPO_ROOT
O=gpurun_out
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so
timeout 300 python scripts/ab_env.py 2 0 off=LSK_PRE:0 after=LSK_PRE:1 inside=LSK_PRE:2 > $O/s2_ab.log 2>&1
AB_N=6151 timeout 300 python scripts/ab_env.py 5 60 off=LSK_PRE:0 after=LSK_PRE:1 inside=LSK_PRE:2 >> $O/s2_ab.log 2>&1
AB_N=500 timeout 300 python scripts/ab_env.py 1 0 off=LSK_PRE:0 after=LSK_PRE:1 inside=LSK_PRE:2 >> $O/s2_ab.log 2>&1
for m in 1 2; do LSK_PRE=$m timeout 900 python -m pytest tests -q -m gpu -x -k "implicit or smoke or determin" > $O/s2_pytest_$m.log 2>&1; echo "pytest pre=$m rc=$?" >> $O/s2_pytest_$m.log; done
cat $O/s2_ab.log; tail -n 2 $O/s2_pytest_*.log
