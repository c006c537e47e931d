import sys, numpy as np
d = open(sys.argv[1], 'rb').read()
P, G = np.frombuffer(d[:8], dtype=np.int32)
t = np.frombuffer(d[8:], dtype=np.uint64).reshape(P, G, 4).astype(np.float64)
rows = []
for p in range(2, P - 2):
    a = t[p]
    if a[:, 0].min() == 0: continue
    arr0, arr1 = a[:, 0].min(), a[:, 0].max()          # tiles done: first / last CTA
    b1 = a[:, 1]; r2 = a[:, 2]; b2 = a[:, 3]
    prev_b2 = t[p - 1][:, 3]
    rows.append([
        (arr0 - prev_b2.max()) / 1e3,                      # fastest CTA pass compute (after prev boundary)
        (arr1 - prev_b2.max()) / 1e3,                      # slowest CTA pass compute
        (b1.min() - arr1) / 1e3,                           # barrier-1 latency after last arrival
        (r2.max() - b1.min()) / 1e3,                       # R2 (incl. spread)
        (b2.min() - r2.max()) / 1e3,                       # barrier-2 latency after last R2
        (b2.max() - b2.min()) / 1e3,                       # release spread
    ])
rows = np.array(rows)
names = ["compute_fastest", "compute_slowest", "bar1_latency", "R2_span", "bar2_latency", "release_spread"]
for n, c in zip(names, rows.T):
    print("%-16s median %.2f us  p90 %.2f us" % (n, np.median(c), np.percentile(c, 90)))
