S="python scripts/sweep.py"
for v in main sr1 nostr; do if [ $v = main ]; then L=""; else L=scripts/variants/liblsk_$v.so; fi
 for H in 0.001 0.3; do echo -n "$v HYB=$H "; LSK_LIB_PATH=$L LSK_HYB=$H timeout 120 $S --config 2 --variant implicit --T 200 --reps 3 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"])'; done; done
