#!/bin/bash
# round 2, call d: emulated ranks (xrs fix) and cluster mode, then the whole GPU suite
cd $GRAFT_REPO_ROOT
O=gpurun_out
for c in "emul stream 2 4000 2" "emul implicit 2 4000 2" "emul stream 8 8000 41" "emul implicit 4 8000 40" "cluster implicit 500 200" "cluster stream 500 200"; do
  echo "== $c" >> $O/r02d.log
  timeout 120 python -u scripts/debug_emul.py $c >> $O/r02d.log 2>&1
  echo "rc=$?" >> $O/r02d.log
done
cat $O/r02d.log
if grep -q "rc=124" $O/r02d.log; then echo "emulation still hangs; skipping the suite"; exit 1; fi
timeout 2400 python -m pytest tests -q -m gpu -x > $O/r02d_gpu.log 2>&1
echo "suite rc=$?" >> $O/r02d_gpu.log
tail -15 $O/r02d_gpu.log
