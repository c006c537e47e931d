#!/bin/bash
# round 2 (session 3): ncu captures — resident kernel (config 1), implicit grid kernel (config 2
# bench command, boundary overlap on), launch list of the bench command
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python scripts/prof_one.py --config 1 --variant implicit --T 200 > $O/s9_prof1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:resident_kernel -s 1 -c 1 -o $O/s9_resident_c1 -f python scripts/prof_one.py --config 1 --variant implicit --T 200 > $O/s9_ncu_res.log 2>&1
echo "ncu res rc=$?" >> $O/s9_ncu_res.log
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $CMD > $O/s9_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/s9_launches.csv $CMD > $O/s9_ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 3 -c 1 -o $O/s9_implicit -f $CMD > $O/s9_ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/s9_ncu_full.log
tail -n 2 $O/s9_ncu_res.log $O/s9_ncu_full.log
# summaries on the box (the reports exceed the copy-back limit)
python scripts/ncu_summary.py $O/s9_resident_c1.ncu-rep 30 > $O/s9_resident_c1_summary.txt 2>&1
python scripts/ncu_summary.py $O/s9_implicit.ncu-rep 30 > $O/s9_implicit_c2_summary.txt 2>&1
ncu -i $O/s9_resident_c1.ncu-rep --page source --csv --print-source sass > $O/s9_resident_sass.csv 2>/dev/null
python scripts/sass_stalls.py $O/s9_resident_sass.csv > $O/s9_resident_sass_stalls.txt 2>&1
ls -la $O; rm -f $O/*.ncu-rep $O/s9_resident_sass.csv
