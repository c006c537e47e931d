timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
S="python scripts/sweep.py"
for V in stream implicit; do echo "c2 $V"; timeout 120 $S --config 2 --variant $V --T 100; done
echo c1; timeout 60 $S --config 1 --variant implicit --T 200
echo c3; timeout 120 $S --config 3 --variant stream --n 200000 --T 20
echo c4; timeout 120 $S --config 4 --T 50
echo c5; timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2
for V in stream implicit; do LSK_TRACE=/tmp/tr_$V.bin $S --config 2 --variant $V --T 50 --reps 1 > /dev/null; echo "== trace $V"; python scripts/trace_analyze.py /tmp/tr_$V.bin; done
