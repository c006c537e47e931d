#!/bin/bash
# round 2, call m: the whole GPU suite, the default bench line, the launch list of the bench
# command, one full capture of the dominant (implicit) kernel and of the K3 feature map
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > $O/r02m_gpu.log 2>&1
echo "suite rc=$?" >> $O/r02m_gpu.log
tail -4 $O/r02m_gpu.log
timeout 900 python bench.py > $O/r02m_bench.json 2> $O/r02m_bench.err
echo "bench rc=$?" >> $O/r02m_bench.err
timeout 300 python scripts/time_features.py > $O/r02m_features.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $CMD > $O/r02m_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/r02m_launches.csv $CMD > $O/r02m_ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 3 -c 1 -o $O/r02m_implicit -f $CMD > $O/r02m_ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/r02m_ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:feature_map_kernel -s 2 -c 1 -o $O/r02m_ftc -f python scripts/time_features.py > $O/r02m_ncu_ftc.log 2>&1
echo "ncu ftc rc=$?" >> $O/r02m_ncu_ftc.log
tail -2 $O/r02m_bench.err; tail -1 $O/r02m_ncu_full.log; tail -1 $O/r02m_ncu_ftc.log; cat $O/r02m_features.log
