import csv, subprocess, sys, io
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur=None; H=None; res=[]
for r in csv.reader(io.StringIO(src)):
    if r and r[0]=="File Path": cur=r[1].split('/')[-1]; continue
    if r and r[0]=="Line No": H=r; continue
    if H and len(r)>8 and r[0].isdigit() and r[2]=="-":
        try: res.append((int(r[7]), int(r[4]), cur, int(r[0]), r[1].strip()[:70]))
        except ValueError: pass
tot=sum(x[0] for x in res); tots=sum(x[1] for x in res)
print("total warp insts", tot)
for ie, s, f, l, c in sorted(res, reverse=True)[:int(sys.argv[2]) if len(sys.argv)>2 else 30]:
    print("%5.1f%% inst %5.1f%% samp %-16s %4d %s" % (100*ie/tot, 100*s/tots, f[:16], l, c))
