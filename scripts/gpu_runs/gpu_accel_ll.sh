python scripts/sweep.py --config 2 --variant accel --T 5 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/accel_ll.csv python scripts/sweep.py --config 2 --variant accel --T 5 --reps 1 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/accel_ll.csv
