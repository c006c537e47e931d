#!/bin/bash
# round 2, call e: the warp-specialised hybrid — phi sweep on config 2, parity, then the suite
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python -u scripts/hybrid_sweep.py 2 -1 0 0.0528 0.07 0.2 0.25 > $O/r02e_sweep.log 2>&1
echo "sweep rc=$?" >> $O/r02e_sweep.log
cat $O/r02e_sweep.log
if grep -q "rc=124" $O/r02e_sweep.log; then exit 1; fi
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "config2 or config5 or implicit or smoke or p2p or nccl" > $O/r02e_parity.log 2>&1
echo "parity rc=$?" >> $O/r02e_parity.log
tail -5 $O/r02e_parity.log
