timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
python bench.py --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads([l for l in sys.stdin if l.startswith("{")][-1]); print(d["value"], d["roofline"]["frac"], d["alt_variant"]["value"], d["alt_variant"]["roofline"]["frac"], d["clocks"])'
