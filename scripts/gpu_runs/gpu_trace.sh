S="python scripts/sweep.py"
for V in stream implicit; do
  LSK_TRACE=/tmp/tr_$V.bin $S --config 2 --variant $V --T 50 --reps 1 > /dev/null
  echo "== $V"; python scripts/trace_analyze.py /tmp/tr_$V.bin
done
LSK_ICFG=128,2,2,8,1 LSK_TRACE=/tmp/tr_p.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null
echo "== implicit pipe 128,2,2,8"; python scripts/trace_analyze.py /tmp/tr_p.bin
