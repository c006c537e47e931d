timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for G in 1 2 4 8; do echo -n "c4 BGPP=$G "; LSK_BGPP=$G timeout 300 python scripts/sweep.py --config 4 --T 30 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in d if k in ("ms","GBs","it_s","us_per_pass")})'; done
for V in implicit stream; do echo -n "c2 $V "; timeout 120 python scripts/sweep.py --config 2 --variant $V --T 200 --reps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"], d["GBs"])'; done
