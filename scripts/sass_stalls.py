"""Summarise an `ncu --page source --print-source sass --csv` export: stall samples per SASS
address range (regions split at barriers / labelled by the caller), and the top instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    addr = int(r[0], 16)
    ins.append((addr, r[1].strip(), int(r[idx["Warp Stall Sampling (All Samples)"]] or 0),
                int(r[idx["Instructions Executed"]] or 0),
                {h[6:]: int(r[i] or 0) for h, i in idx.items() if h.startswith("stall_") and "Not Issued" not in h}))
base = ins[0][0]
tot = sum(x[2] for x in ins)
print("total samples", tot, "instructions executed", sum(x[3] for x in ins))
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else None
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
sel = [x for x in ins if lo is None or (lo <= x[0] - base < hi)]
s = sum(x[2] for x in sel)
st = collections.Counter()
for x in sel:
    st.update(x[4])
print("range samples %d (%.1f%%), executed %d" % (s, 100.0 * s / tot, sum(x[3] for x in sel)))
print("stalls:", ", ".join("%s %.1f%%" % (k, 100.0 * v / max(s, 1)) for k, v in st.most_common(10)))
print("top instructions:")
for x in sorted(sel, key=lambda x: -x[2])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    top = sorted(x[4].items(), key=lambda kv: -kv[1])[:3]
    print("  %05x %5.2f%% %-60s %s" % (x[0] - base, 100.0 * x[2] / tot, x[1][:60], top))
