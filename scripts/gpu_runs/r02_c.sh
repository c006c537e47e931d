#!/bin/bash
# round 2, call c: debug the emulated-rank exchange and the cluster mode (short timeouts)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for c in "cluster implicit 500 3" "cluster stream 500 3" "cluster implicit 500 200" "cluster stream 500 200" \
         "emul stream 2 4000 2" "emul implicit 2 4000 2"; do
  echo "== $c" >> $O/r02c.log
  timeout 90 python -u scripts/debug_emul.py $c >> $O/r02c.log 2>&1
  echo "rc=$?" >> $O/r02c.log
done
timeout 900 python -m pytest tests/test_gpu_boundary.py -x -q -m gpu -k "cluster" > $O/r02c_cluster_tests.log 2>&1
echo "rc=$?" >> $O/r02c_cluster_tests.log
cat $O/r02c.log; tail -5 $O/r02c_cluster_tests.log
