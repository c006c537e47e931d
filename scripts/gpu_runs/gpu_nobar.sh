timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
S="python scripts/sweep.py"
for V in implicit stream; do echo "c2 $V"; timeout 120 $S --config 2 --variant $V --T 100; done
echo c1; $S --config 1 --variant implicit --T 200
echo c3; $S --config 3 --variant stream --n 200000 --T 20
echo c4; $S --config 4 --T 50
echo c5; $S --config 5 --variant implicit --n 1048576 --T 2
LSK_TRACE=/tmp/tr.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin
