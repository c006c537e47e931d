#!/bin/bash
# round 2, final session: the measured parity errors of the five configurations at full size and
# full T (pytest -s prints them), for BASELINE.md §5
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1800 python -m pytest -m gpu -s -q tests/test_gpu_full.py "tests/test_gpu_parity.py::test_config1_full_streaming" "tests/test_gpu_parity.py::test_config1_full_implicit" "tests/test_gpu_parity.py::test_config2_full_size" > $O/r02x_parity_errors.log 2>&1
echo "rc=$?" >> $O/r02x_parity_errors.log
grep -n "parity:\|full\|passed\|failed\|rc=" $O/r02x_parity_errors.log
