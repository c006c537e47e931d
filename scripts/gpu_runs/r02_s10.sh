#!/bin/bash
# round 2 (session 3): resident kernel, st.async push boundary (push) vs cluster barrier + DSMEM loads (tuning)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in tuning push; do
  echo "== $lib" >> $O/s10_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 1 0 g4=LSK_RESG:4 g8=LSK_RESG:8 >> $O/s10_ab.log 2>&1
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so AB_N=1100 timeout 300 python scripts/ab_env.py 1 0 g8=LSK_RESG:8 >> $O/s10_ab.log 2>&1
done
LSK_LIB_PATH=$PWD/scripts/variants/liblsk_push.so timeout 600 python -m pytest tests/test_gpu_resident.py -q -x > $O/s10_pytest.log 2>&1
echo "pytest rc=$?" >> $O/s10_pytest.log
grep -v ' vs ' $O/s10_ab.log; tail -n 3 $O/s10_pytest.log
