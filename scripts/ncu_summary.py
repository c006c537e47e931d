"""Summarise an ncu report: headline metrics + hottest source lines with stall reasons."""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
for h, u, v in zip(rows[0], rows[1], vals):
    if h in want:
        print("%-60s %s %s" % (h, v[:90], u))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; res = []; H = None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": H = r; continue
    if H and len(r) > 5 and r[0].isdigit() and r[2] == "-":
        try: res.append((float(r[4]), cur, int(r[0]), r[1], r))
        except ValueError: pass
tot = sum(x[0] for x in res) or 1
sc = [i for i, h in enumerate(H or []) if h.startswith("stall_") and "Not Issued" not in h]
for s, f, l, code, r in sorted(res, key=lambda x: -x[0])[:top]:
    t = sorted([(float(r[i] or 0), H[i][6:]) for i in sc], reverse=True)[:2]
    print("%5.1f%% %-16s %4d %-62s %s" % (100 * s / tot, f[:16], l, code.strip()[:62], [(a, int(b)) for b, a in t]))
