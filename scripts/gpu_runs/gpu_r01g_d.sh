ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01g_launches_config2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alt > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 1 -c 1 -o /tmp/ic2 -f python scripts/prof_one.py --config 2 --variant implicit --T 20 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/ic2.ncu-rep 30 > gpurun_out/r01g_implicit_c2_full.txt 2>&1
ncu -i /tmp/ic2.ncu-rep --page source --csv --print-source sass > /tmp/ic2_sass.csv 2>/dev/null
python scripts/sass_stalls.py /tmp/ic2_sass.csv > gpurun_out/r01g_implicit_c2_sass.txt 2>&1
python scripts/launch_table.py gpurun_out/r01g_launches_config2.csv | head -2
