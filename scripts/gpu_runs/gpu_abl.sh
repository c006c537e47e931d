# ablations of the implicit tile loop (timing only; results are wrong by construction)
S="python scripts/sweep.py"
for v in base noex2 noxch nobar noxb; do
  L=scripts/variants/liblsk_$v.so
  echo "== $v"; LSK_LIB_PATH=$L timeout 120 $S --config 2 --variant implicit --T 200 --reps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"])'
  LSK_LIB_PATH=$L LSK_TRACE=/tmp/tr.bin timeout 120 $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin | head -2
done
