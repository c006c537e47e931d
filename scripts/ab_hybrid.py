"""A/B of the implicit solver's pure-recompute vs hybrid split on config 2 with bench.py's
protocol (L2 flush before every timed solve, CUDA events around the solve), interleaved."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 2
phis = [float(x) for x in sys.argv[2:]] or [-1.0, 0.25, 0.2]
cfg = synth.get_config(key)
prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
L.lsk_draw_anchors(p, U)
u = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
v = torch.empty(cfg.m, dtype=torch.float32, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
res = {phi: [] for phi in phis}
for rnd in range(5):
    for phi in phis:
        opts = L.make_opts(cfg.T, stream_fraction=phi)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=False)
        e1.record()
        e1.synchronize()
        if rnd > 0:
            res[phi].append(e0.elapsed_time(e1))
L.lsk_stream_status()
for phi in phis:
    ms = np.array(res[phi])
    print("config %d phi %5.2f  median %.3f ms  min %.3f  max %.3f  -> %.0f it/s"
          % (key, phi, np.median(ms), ms.min(), ms.max(), cfg.T / (np.median(ms) / 1e3)), flush=True)
