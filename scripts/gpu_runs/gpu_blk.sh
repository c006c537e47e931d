timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
AB_C5=1 AB_C1=1 bash scripts/gpu_runs/gpu_ab.sh main base
for V in implicit stream; do LSK_TRACE=/tmp/tr.bin timeout 120 python scripts/sweep.py --config 2 --variant $V --T 50 --reps 1 > /dev/null; echo "== $V"; python scripts/trace_analyze.py /tmp/tr.bin; done
for L in "" scripts/variants/liblsk_base.so; do echo -n "stream c2 [$L] "; LSK_LIB_PATH=$L timeout 120 python scripts/sweep.py --config 2 --variant stream --T 200 --reps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_pass"], d["it_s"], d["GBs"])'; done
