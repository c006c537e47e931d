S="python scripts/sweep.py --reps 1"
LSK_TRACE=gpurun_out/tr_impl.bin $S --variant implicit --T 30 > /dev/null
LSK_TRACE=gpurun_out/tr_impl1.bin $S --variant implicit --T 30 --cps 1 > /dev/null
python scripts/prof_one.py --variant implicit --T 20 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:implicit -s 1 -c 1 -o gpurun_out/prof_impl4 python scripts/prof_one.py --variant implicit --T 20 > gpurun_out/ncu6.log 2>&1
