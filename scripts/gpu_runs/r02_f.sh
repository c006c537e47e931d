#!/bin/bash
# round 2, call f: the whole GPU suite, the default bench line, the launch list of the bench
# command and one full capture of the dominant (hybrid) kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > $O/r02f_gpu.log 2>&1
echo "suite rc=$?" >> $O/r02f_gpu.log
tail -4 $O/r02f_gpu.log
timeout 900 python bench.py > $O/r02f_bench.json 2> $O/r02f_bench.err
echo "bench rc=$?" >> $O/r02f_bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $CMD > $O/r02f_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/r02f_launches.csv $CMD > $O/r02f_ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid -s 3 -c 1 -o $O/r02f_hybrid -f $CMD > $O/r02f_ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/r02f_ncu_full.log
tail -2 $O/r02f_bench.err; tail -2 $O/r02f_ncu_full.log
