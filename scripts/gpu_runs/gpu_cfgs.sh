S="python scripts/sweep.py"
L=scripts/variants/liblsk_cfgs.so
for rep in 1 2; do
for C in "" "256,2,1,16,0" "256,2,1,8,0" "128,4,2,8,0" "128,3,2,8,0"; do
  echo -n "cfg [$C] c2 "; LSK_LIB_PATH=$L LSK_ICFG=$C timeout 120 $S --config 2 --variant implicit --T 200 --reps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'
done; done
