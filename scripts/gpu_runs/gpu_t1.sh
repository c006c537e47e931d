L=scripts/variants/liblsk_t1.so
for C in "" "128,1,2,16,0" "128,1,2,8,0"; do echo -n "c2 [$C] "; LSK_LIB_PATH=$L LSK_ICFG=$C timeout 60 python scripts/sweep.py --config 2 --variant implicit --T 100 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'; done
