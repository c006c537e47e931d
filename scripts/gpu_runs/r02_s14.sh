#!/bin/bash
# round 2 (session 3): graph-driven accelerated solve (device line search) vs the host loop;
# the Alg. 2 GPU tests on the product build
cd $GRAFT_REPO_ROOT
O=gpurun_out
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so timeout 600 python scripts/ab_accel.py 2 100 > $O/s14_ab.log 2>&1
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so timeout 600 python scripts/ab_accel.py 1 200 >> $O/s14_ab.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "accel" > $O/s14_pytest.log 2>&1
echo "pytest rc=$?" >> $O/s14_pytest.log
cat $O/s14_ab.log; tail -n 15 $O/s14_pytest.log
