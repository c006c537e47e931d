S="python scripts/sweep.py"
for H in 0 0.3; do for D in 0 2; do echo "== HYB=$H DBG=$D"; LSK_DEBUG=$D LSK_HYB=$H LSK_TRACE=/tmp/tr.bin timeout 120 $S --config 2 --variant implicit --T 50 --reps 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"])'; python scripts/trace_analyze.py /tmp/tr.bin | head -4; done; done
echo "== 1-team only rows 70% equivalent: HYB=0.3 with no stream rows?"; 
