LSK_TRACE=gpurun_out/tr_impl5.bin python scripts/sweep.py --variant implicit --T 30 --reps 1 > /dev/null; python scripts/trace_analyze.py gpurun_out/tr_impl5.bin
LSK_TRACE=gpurun_out/tr_impl6.bin python scripts/sweep.py --config 5 --variant implicit --n 500000 --T 4 --reps 1 > /dev/null; python scripts/trace_analyze.py gpurun_out/tr_impl6.bin
