ncu --set full --clock-control none --import-source on -k regex:feature_map_tc -s 2 -c 1 -o /tmp/tc -f python /tmp/fm_once.py > /dev/null 2>&1
ncu -i /tmp/tc.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/tc_sass.csv
python3 - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/tc_sass.csv')))
for i,r in enumerate(rows):
    if r and r[0]=='Address': H=r; start=i+1; break
idx={h:i for i,h in enumerate(H)}
data=[r for r in rows[start:] if len(r)>=len(H)]
tot=sum(int(r[idx['Warp Stall Sampling (All Samples)']]) for r in data)
top=sorted(range(len(data)), key=lambda i:-int(data[i][idx['Warp Stall Sampling (All Samples)']]))[:12]
for i in sorted(top):
    r=data[i]
    print("%5.1f%% exec=%9s %s" % (100*int(r[idx['Warp Stall Sampling (All Samples)']])/tot, r[idx['Instructions Executed']], r[1][:90]))
    for j in range(max(0,i-3), i):
        print("          prev: %s" % data[j][1][:90])
PY
