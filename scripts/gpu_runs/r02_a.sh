#!/bin/bash
# round 2, call a: boundary tests first (short timeout: the multi-launch fix), then the GPU suite
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_boundary.py -x -q -m gpu > gpurun_out/r02a_boundary.log 2>&1
echo "boundary rc=$?" >> gpurun_out/r02a_boundary.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02a_gpu.log 2>&1
echo "suite rc=$?" >> gpurun_out/r02a_gpu.log
tail -3 gpurun_out/r02a_boundary.log gpurun_out/r02a_gpu.log
