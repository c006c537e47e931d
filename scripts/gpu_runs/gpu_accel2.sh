timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "accel" 2>&1 | tail -2
for rep in 1 2; do for L in "" scripts/variants/liblsk_prev.so; do echo -n "accel c2 [$L] "; LSK_LIB_PATH=$L timeout 300 python scripts/sweep.py --config 2 --variant accel --T 100 --reps 3 | tail -1; done; done
python scripts/prof_one.py --config 2 --variant stream --T 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:pass_kernel -c 6 python scripts/sweep.py --config 2 --variant accel --T 2 --reps 1 2>/dev/null | grep -v "^==" | tail -20
