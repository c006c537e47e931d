S="python scripts/sweep.py"
for H in 0 0.001 0.2 0.3 0.35 0.4 0.5; do echo -n "HYB=$H "; LSK_HYB=$H timeout 120 $S --config 2 --variant implicit --T 200 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"])'; done
