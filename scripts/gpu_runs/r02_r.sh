#!/bin/bash
# round 2, call r: the whole GPU suite, the default bench line, config 1's line, the launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > $O/r02r_gpu.log 2>&1
echo "suite rc=$?" >> $O/r02r_gpu.log
tail -3 $O/r02r_gpu.log
timeout 900 python bench.py > $O/r02r_bench.json 2> $O/r02r_bench.err
echo "bench rc=$?" >> $O/r02r_bench.err
timeout 300 python bench.py --config 1 --no-extra > $O/r02r_bench_config1.json 2>> $O/r02r_bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $CMD > $O/r02r_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/r02r_launches.csv $CMD > $O/r02r_ncu_launches.log 2>&1
echo "ncu rc=$?"
tail -3 $O/r02r_bench.err
