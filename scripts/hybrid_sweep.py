"""Sweep the stream fraction phi of the warp-specialised hybrid (lsk_hybrid.cu) on a config:
per phi, the persistent solve's CUDA-event time (mean of K after W warm-ups), us per pass,
and the ROT against the pure-recompute solve (phi < 0).
usage: python scripts/hybrid_sweep.py [config] [phi ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 2
phis = [float(x) for x in sys.argv[2:]] or [-1.0, 0.2, 0.3, 0.35, 0.4, 0.45, 0.5]
cfg = synth.get_config(key)
prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
L.lsk_draw_anchors(p, U)
u = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
v = torch.empty(cfg.m, dtype=torch.float32, device="cuda")
base = None
for phi in phis:
    opts = L.make_opts(cfg.T, stream_fraction=phi)
    rep = L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v)
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=False)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    L.lsk_stream_status()
    ms = float(np.mean(ts[1:]))
    if base is None:
        base = rep.rot
    print("config %d phi %5.2f  %8.3f ms  %6.2f us/pass  %8.0f it/s  rot %.12f  rel %.2e"
          % (key, phi, ms, 1e3 * ms / (2 * cfg.T + 1), cfg.T / (ms / 1e3), rep.rot,
             abs(rep.rot - base) / abs(base)), flush=True)
