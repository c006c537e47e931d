S="python scripts/sweep.py --reps 1"
LSK_TRACE=gpurun_out/tr_stream.bin $S --variant stream --T 30 > /dev/null
LSK_TRACE=gpurun_out/tr_stream_dbg.bin LSK_DEBUG=1 $S --variant stream --T 30 > /dev/null
