S="python scripts/sweep.py --T 200"
for f in 0 0.15 0.25 0.3 0.35 0.4 0.5; do LSK_L2RES=$f $S --variant stream; done
