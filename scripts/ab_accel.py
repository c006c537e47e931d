"""Interleaved A/B of the accelerated solve (Alg. 2, NEXT f4): the graph-driven line search
(one CUDA graph per solve, decisions on the device) against the host-driven loop (one
synchronisation per trial).  Tuning build only (LSK_ACCEL_HOST=1 selects the host loop):
LSK_LIB_PATH=scripts/variants/liblsk_tuning.so python scripts/ab_accel.py [config] [iters]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = synth.get_config(key)
prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
L.lsk_draw_anchors(p, U)
Xi = torch.empty((X.shape[0], cfg.r), device="cuda")
Ze = torch.empty((Y.shape[0], cfg.r), device="cuda")
L.lsk_feature_map(p, U, X, Xi)
L.lsk_feature_map(p, U, Y, Ze)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
arms = {"host": "1", "graph": "0"}
res = {k: [] for k in arms}
out = {}
for rnd in range(5):
    for name, val in arms.items():
        os.environ["LSK_ACCEL_HOST"] = val
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = L.lsk_accelerated_sinkhorn(Xi, Ze, a, b, cfg.eps, T, traces=True)
        e1.record()
        e1.synchronize()
        if rnd > 0:
            res[name].append(e0.elapsed_time(e1))
        out[name] = r
for name in arms:
    ms = np.array(res[name])
    r = out[name]
    print("config %d accel %-6s median %.3f ms for %d iterations (%d trials): %.1f us/trial, "
          "%.0f it/s  F %.12f L %.4g plan_err %.3e"
          % (key, name, np.median(ms), r["iters"], r["trials"], 1e3 * np.median(ms) / r["trials"],
             r["iters"] / (np.median(ms) / 1e3), r["F"], r["L"], r["plan_err"]), flush=True)
h, g = out["host"], out["graph"]
print("graph vs host: F rel %.2e, same iters %s, same trials %s, eta1 max abs %.2e, L traces equal %s"
      % (abs(g["F"] - h["F"]) / abs(h["F"]), g["iters"] == h["iters"], g["trials"] == h["trials"],
         float((g["eta1"] - h["eta1"]).abs().max()),
         bool(np.array_equal(g["L_trace"], h["L_trace"]))))
