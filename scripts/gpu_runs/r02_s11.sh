#!/bin/bash
# round 2 (session 3): A/B — scalings broadcast through shared memory (wt1) vs shuffles (wt0);
# early pre-generation by the short team (LSK_PRE=3); then the GPU suite on the product build
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in wt0 wt1; do
  echo "== $lib" >> $O/s11_ab.log
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so timeout 300 python scripts/ab_env.py 2 0 pre2=LSK_PRE:2 pre3=LSK_PRE:3 >> $O/s11_ab.log 2>&1
  LSK_LIB_PATH=$PWD/scripts/variants/liblsk_$lib.so AB_N=1048576 timeout 300 python scripts/ab_env.py 5 20 pre2=LSK_PRE:2 >> $O/s11_ab.log 2>&1
done
grep -v ' vs ' $O/s11_ab.log; grep ' vs ' $O/s11_ab.log | head -3
timeout 1500 python -m pytest tests -q -m gpu > $O/s11_pytest_gpu.log 2>&1
echo "suite rc=$?" >> $O/s11_pytest_gpu.log
tail -n 4 $O/s11_pytest_gpu.log
