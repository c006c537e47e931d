S="python scripts/sweep.py"
echo "== t1 (128,1,2,16)"; LSK_LIB_PATH=scripts/variants/liblsk_t1.so LSK_ICFG=128,1,2,16,0 LSK_TRACE=/tmp/tr.bin timeout 120 $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin 2>/dev/null | head -4
echo "== hybrid 0.001"; LSK_HYB=0.001 LSK_TRACE=/tmp/tr.bin timeout 120 $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin 2>/dev/null | head -4
