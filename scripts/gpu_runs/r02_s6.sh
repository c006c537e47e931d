#!/bin/bash
# round 2 (session 3): resident small-problem kernel — parity tests, cluster-size A/B on config 1
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py tests/test_gpu_boundary.py -q -x > $O/s6_pytest.log 2>&1
echo "pytest rc=$?" >> $O/s6_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config1 or tolerance or tiny or determin or smoke or marginal or largest" >> $O/s6_pytest.log 2>&1
echo "pytest2 rc=$?" >> $O/s6_pytest.log
export LSK_LIB_PATH=$PWD/scripts/variants/liblsk_tuning.so
timeout 300 python scripts/ab_env.py 1 0 grid=LSK_RESG:0 g2=LSK_RESG:2 g4=LSK_RESG:4 g8=LSK_RESG:8 > $O/s6_ab.log 2>&1
timeout 300 python scripts/ab_env.py 2 0 pre0=LSK_PRE:0 pre2=LSK_PRE:2 >> $O/s6_ab.log 2>&1
tail -n 15 $O/s6_pytest.log; grep -v ' vs ' $O/s6_ab.log; grep ' vs ' $O/s6_ab.log | head -4
