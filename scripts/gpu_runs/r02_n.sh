#!/bin/bash
# round 2, call n: the default bench line, the launch list of the bench command, full captures
# of the implicit kernel and of the K3 feature map — summarised on the box (the raw reports
# exceed the 64 MiB return limit)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python bench.py > $O/r02n_bench.json 2> $O/r02n_bench.err
echo "bench rc=$?" >> $O/r02n_bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $CMD > $O/r02n_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/r02n_launches.csv $CMD > $O/r02n_ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 3 -c 1 -o /tmp/r02n_implicit -f $CMD > $O/r02n_ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/r02n_ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:feature_map_kernel -s 2 -c 1 -o /tmp/r02n_ftc -f python scripts/time_features.py > $O/r02n_ncu_ftc.log 2>&1
echo "ncu ftc rc=$?" >> $O/r02n_ncu_ftc.log
for k in implicit ftc; do
  python scripts/ncu_summary.py /tmp/r02n_$k.ncu-rep 30 > $O/r02n_${k}_summary.txt 2>&1
  ncu -i /tmp/r02n_$k.ncu-rep --page source --csv --print-source sass > $O/r02n_${k}_sass.csv 2>/dev/null
  ncu -i /tmp/r02n_$k.ncu-rep --page raw --csv > $O/r02n_${k}_raw.csv 2>/dev/null
  python scripts/sass_stalls.py $O/r02n_${k}_sass.csv >> $O/r02n_${k}_summary.txt 2>&1
done
du -sh $O
tail -2 $O/r02n_bench.err; tail -1 $O/r02n_ncu_full.log; tail -1 $O/r02n_ncu_ftc.log
