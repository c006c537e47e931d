cat > /tmp/fm_once.py <<'PY'
import sys, os; sys.path.insert(0, os.getcwd())
import torch, paper_2006_07057_b200 as L, synth
c = synth.get_config(4); n = 1 << 20
X = torch.randn((n, c.d), device="cuda") * (1.0 / c.d) ** 0.5
p = L.lsk_feature_params_init(c.eps, c.d, c.r, 0.0, c.anchor_seed, X, X)
U = torch.empty((c.r, c.d), device="cuda"); L.lsk_draw_anchors(p, U)
Xi = torch.empty((n, c.r), device="cuda")
for _ in range(3): L.lsk_feature_map(p, U, X, Xi)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); L.lsk_feature_map(p, U, X, Xi); e1.record(); e1.synchronize(); print("fm ms", e0.elapsed_time(e1))
PY
python /tmp/fm_once.py
ncu --set full --clock-control none -k regex:feature_map_tc -s 2 -c 1 -o /tmp/tc -f python /tmp/fm_once.py > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/tc.ncu-rep 5
ncu -i /tmp/tc.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h,u,v=rows[0],rows[1],rows[2]
want=['sm__pipe_tensor_op_utcmma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active','sm__throughput.avg.pct_of_peak_sustained_elapsed','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','sm__ctas_launched.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed']
for a,b,c in zip(h,u,v):
    if a in want or 'tensor' in a and 'pct' in a: print(a,c,b)
out=sorted(((float(v[i]),k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')) for i,k in enumerate(h) if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')),reverse=True)[:8]
print(out)"
