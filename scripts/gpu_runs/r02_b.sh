#!/bin/bash
# round 2, call b: emulated-rank + full-size parity tests, the default bench line, and the
# dram traffic of the config-3 stream kernel and the config-4 batched kernel (ncu --set full)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_emulated_ranks.py tests/test_gpu_full.py -q -m gpu -s > $O/r02b_tests.log 2>&1
echo "tests rc=$?" >> $O/r02b_tests.log
timeout 900 python bench.py > $O/r02b_bench.json 2> $O/r02b_bench.err
echo "bench rc=$?" >> $O/r02b_bench.err
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
C4="python bench.py --config 4 --steps 1 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 600 $C3 > $O/r02b_c3.json 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:sinkhorn_kernel -s 3 -c 1 -o $O/r02b_c3 -f $C3 > $O/r02b_ncu_c3.log 2>&1
timeout 600 $C4 > $O/r02b_c4.json 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:sinkhorn_kernel -s 3 -c 1 -o $O/r02b_c4 -f $C4 > $O/r02b_ncu_c4.log 2>&1
tail -3 $O/r02b_tests.log; tail -2 $O/r02b_bench.err; ls $O
