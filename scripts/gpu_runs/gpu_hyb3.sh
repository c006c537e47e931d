S="python scripts/sweep.py"
for H in 0 0.001 0.1 0.3; do echo -n "HYB=$H "; LSK_HYB=$H timeout 120 $S --config 2 --variant implicit --T 200 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"])'; done
for H in 0.001 0.3; do echo -n "HYB=$H DBG=2 "; LSK_DEBUG=2 LSK_HYB=$H timeout 120 $S --config 2 --variant implicit --T 200 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"])'; done
