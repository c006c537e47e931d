S="python scripts/sweep.py --reps 1"
LSK_TRACE=/tmp/tr_stream.bin $S --variant stream --T 20 > /dev/null && python scripts/trace_analyze.py /tmp/tr_stream.bin
LSK_TRACE=/tmp/tr_small.bin $S --variant stream --T 50 --n 4736 > /dev/null && python scripts/trace_analyze.py /tmp/tr_small.bin
