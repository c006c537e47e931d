#!/bin/bash
# round 2 (session 3): staggered team start A/B on config 2, implicit parity tests
cd $GRAFT_REPO_ROOT
O=gpurun_out
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so
timeout 300 python scripts/ab_env.py 2 0 off=LSK_STAGGER:0 on=LSK_STAGGER:1 > $O/s1_ab.log 2>&1
cat $O/s1_ab.log
AB_N=200000 timeout 300 python scripts/ab_env.py 2 100 off=LSK_STAGGER:0 on=LSK_STAGGER:1 >> $O/s1_ab.log 2>&1
unset LSK_LIB_PATH
timeout 900 python -m pytest tests -q -m gpu -x -k "implicit or smoke" > $O/s1_pytest.log 2>&1
echo "pytest rc=$?" >> $O/s1_pytest.log
tail -n 5 $O/s1_ab.log; tail -n 3 $O/s1_pytest.log
