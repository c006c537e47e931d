#!/bin/bash
# round 2, final session: final state of the round (after the FFMA feature-map rework) — full GPU suite, smoke(),
# the default bench line, the reference arm, and the launch list of the bench command
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > $O/r02z_pytest_gpu.log 2>&1
echo "tests rc=$?" >> $O/r02z_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r02z_smoke.log 2>&1
echo "smoke rc=$?" >> $O/r02z_smoke.log
timeout 1200 python bench.py > $O/r02z_bench.json 2> $O/r02z_bench.err
echo "bench rc=$?" >> $O/r02z_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02z_bench_reference.json 2> $O/r02z_bench_reference.err
echo "ref rc=$?" >> $O/r02z_bench_reference.err
B="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $B > $O/r02z_b.json 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02z_launches_config2.csv $B > $O/r02z_ncu.log 2>&1
tail -3 $O/r02z_pytest_gpu.log; tail -2 $O/r02z_smoke.log; tail -2 $O/r02z_bench.err; tail -2 $O/r02z_bench_reference.err; cat $O/r02z_bench.json | cut -c1-600
