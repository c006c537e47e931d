#!/bin/bash
# round 2 (session 3): two-team ping-pong tile-count tests
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_resident.py -q -x -k pingpong > $O/s25_pytest.log 2>&1
echo "pytest rc=$?" >> $O/s25_pytest.log
tail -n 15 $O/s25_pytest.log
