# A/B of tuning builds (LSK_LIB_PATH); args: variant names ("main" = in-tree library)
S="python scripts/sweep.py"
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then L=""; else L=scripts/variants/liblsk_$v.so; fi
  for c in 2; do echo -n "$v c$c "; LSK_LIB_PATH=$L timeout 120 $S --config $c --variant implicit --T 200 --reps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'; done
  if [ -n "$AB_C5" ]; then echo -n "$v c5 "; LSK_LIB_PATH=$L timeout 120 $S --config 5 --variant implicit --n 1048576 --T 4 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'; fi
  if [ -n "$AB_C1" ]; then echo -n "$v c1 "; LSK_LIB_PATH=$L timeout 120 $S --config 1 --variant implicit --T 200 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'; fi
done
done
