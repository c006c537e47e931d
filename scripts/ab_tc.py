"""A/B of the implicit solver's tensor-core exponent kernel (lsk_implicit_tc.cu, tuning builds
only: LSK_LIB_PATH=scripts/variants/liblsk_tuning.so from `build.py --tuning`) against the
FFMA-exponent recompute kernel and the hybrid, with bench.py's protocol (L2 flush before every
timed solve, CUDA events around the solve), interleaved; plus the ROT of each."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = synth.get_config(key)
if T:
    cfg = synth.get_config(key, T=T)
prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
L.lsk_draw_anchors(p, U)
u = torch.empty(cfg.n, dtype=torch.float32, device="cuda")
v = torch.empty(cfg.m, dtype=torch.float32, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
arms = {"tc": dict(stream_fraction=-1.0), "ffma": dict(stream_fraction=-1.0),
        "hybrid": dict(stream_fraction=0.25)}
res = {k: [] for k in arms}
out = {}
for rnd in range(6):
    for name, kw in arms.items():
        os.environ["LSK_ITC"] = "1" if name == "tc" else "0"   # read per call (tuning builds)
        opts = L.make_opts(cfg.T, **kw)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=False)
        e1.record()
        e1.synchronize()
        if rnd > 0:
            res[name].append(e0.elapsed_time(e1))
        if rnd == 0:
            rep = L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v)
            out[name] = (rep["rot"] if isinstance(rep, dict) else rep.rot, u.clone(), v.clone())
L.lsk_stream_status()
passes = 2 * cfg.T + 1
for name in arms:
    ms = np.array(res[name])
    print("config %d %-7s median %.3f ms (%.2f us/pass) min %.3f max %.3f -> %.0f it/s  rot %.12f"
          % (key, name, np.median(ms), 1e3 * np.median(ms) / passes, ms.min(), ms.max(),
             cfg.T / (np.median(ms) / 1e3), out[name][0]), flush=True)
r0, u0, v0 = out["ffma"]
for name in ("tc", "hybrid"):
    r1, u1, v1 = out[name]
    print("%s vs ffma: rot rel %.2e, u max rel %.2e, v max rel %.2e" % (
        name, abs(r1 - r0) / abs(r0), float(((u1 - u0).abs() / u0).max()),
        float(((v1 - v0).abs() / v0).max())))
