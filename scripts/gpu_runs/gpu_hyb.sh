LSK_HYB=0.3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit or config" 2>&1 | tail -3
for H in 0 0.2 0.3 0.4 0.5; do echo -n "c2 HYB=$H "; LSK_HYB=$H timeout 60 python scripts/sweep.py --config 2 --variant implicit --T 200 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'; done
for H in 0 0.3; do echo -n "c1 HYB=$H "; LSK_HYB=$H timeout 60 python scripts/sweep.py --config 1 --variant implicit --T 200 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'; done
