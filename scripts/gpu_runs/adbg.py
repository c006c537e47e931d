import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch, oracle as O, synth
import paper_2006_07057_b200 as L
from test_gpu_parity import _accel_pair
try:
    gpu, ref, _ = _accel_pair(L, 1, 500, 500, 60)
except Exception as e:
    print("ERR", e)
cfg = synth.get_config(1); prob = synth.make_problem(cfg)
R = O.max_norm(prob["X"], prob["Y"]); p = O.gaussian_params(cfg.eps, cfg.d, cfg.r, R)
Uo = O.draw_anchors(cfg.r, cfg.d, p["sigma"], cfg.anchor_seed)
xi = O.feature_matrix(prob["X"], Uo, cfg.eps, p["q"]); zeta = O.feature_matrix(prob["Y"], Uo, cfg.eps, p["q"])
a = prob["a"].astype(np.float64); a/=a.sum(); b = prob["b"].astype(np.float64); b/=b.sum()
Kv = xi.T @ (zeta @ np.ones(500)); print("oracle S1", Kv.sum(), "n1", ((Kv/Kv.sum()-a)**2).sum())
