"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    a = agg[r[ki][:70]]
    if r[mi] == "gpu__time_duration.sum":
        a[0] += 1; a[1] += v
    elif r[mi].startswith("dram__bytes"):
        a[2] += v
tot = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    n = max(v[0], 1)
    print("%-70s %4d %10.1f us %8.2f us/launch %5.1f%% %10.3g B/launch" % (k, v[0], v[1] / 1e3, v[1] / 1e3 / n, 100 * v[1] / tot, v[2] / n))
