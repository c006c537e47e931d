timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
S="python scripts/sweep.py"
for V in implicit stream; do echo "c2 $V"; timeout 120 $S --config 2 --variant $V --T 100; done
echo c3; $S --config 3 --variant stream --n 200000 --T 20
LSK_TRACE=/tmp/tr.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin
