timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "accelerated" 2>&1 | tail -3
S="python scripts/sweep.py"
$S --config 2 --variant accel --T 100
$S --config 3 --variant accel --n 200000 --T 20
$S --config 1 --variant accel --T 100
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/accel_launches.csv python scripts/sweep.py --config 2 --variant accel --T 10 --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open('/tmp/accel_launches.csv')) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try: agg[r[ki][:60]][0] += 1; agg[r[ki][:60]][1] += float(r[vi].replace(',', ''))
    except: pass
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]): print("%-60s %5d %10.1f us %6.1f us/launch %5.1f%%" % (k, v[0], v[1] / 1e3, v[1] / 1e3 / v[0], 100 * v[1] / tot))
PY
