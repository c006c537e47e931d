import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2006_07057_b200 as L, synth
cfg = synth.get_config(2); prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
n, m, r, d = cfg.n, cfg.m, cfg.r, cfg.d
p = L.lsk_feature_params_init(cfg.eps, d, r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((r, d), device="cuda"); L.lsk_draw_anchors(p, U)
Xi = torch.empty((n, r), device="cuda"); Ze = torch.empty((m, r), device="cuda")
L.lsk_feature_map(p, U, X, Xi); L.lsk_feature_map(p, U, Y, Ze)
u = torch.ones(n, device="cuda"); v = torch.ones(m, device="cuda")
for _ in range(3): L.lsk_rot_gradient(p, U, X, Y, Xi, Ze, u, v)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); L.lsk_rot_gradient(p, U, X, Y, Xi, Ze, u, v); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print("f2 gradients, config 2: median %.4f ms (min %.4f); two reads of each factor = %.0f GB/s"
      % (ts[len(ts) // 2], ts[0], 2 * (n + m) * r * 4 / ts[len(ts) // 2] / 1e6))
