S="python scripts/sweep.py"
for H in 0.001 0.3; do echo "== nostr HYB=$H"; LSK_LIB_PATH=scripts/variants/liblsk_nostr.so LSK_HYB=$H LSK_TRACE=/tmp/tr.bin timeout 120 $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin 2>/dev/null | head -4; done
