timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
for v in stream implicit; do for c in 1 2; do
python bench.py --variant $v --ctas-per-sm $c --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); print('$v cps=$c', round(d['value']), 'it/s', d['roofline']['frac'], d['kernel_ms'])"
done; done
