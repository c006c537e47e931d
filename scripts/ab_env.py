"""Interleaved A/B of tuning-build environment knobs on the implicit solver, with bench.py's
protocol (L2 flush before every timed solve, CUDA events around the solve).  Needs a tuning
build (LSK_LIB_PATH=scripts/variants/liblsk_tuning.so from `build.py --tuning`): the product
library reads no environment.

usage: python scripts/ab_env.py <config> <T or 0> NAME=VAR:VAL[+VAR:VAL] [NAME=...] ...
e.g.   python scripts/ab_env.py 2 0 off=LSK_STAGGER:0 on=LSK_STAGGER:1
Prints median ms, us/pass and it/s per arm, and each arm's ROT / scalings against the first."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

key = int(sys.argv[1])
T = int(sys.argv[2])
arms = {}
for spec in sys.argv[3:]:
    name, kv = spec.split("=", 1)
    arms[name] = dict(x.split(":", 1) for x in kv.split("+") if x)
cfg = synth.get_config(key, T=T) if T else synth.get_config(key)
n = int(os.environ.get("AB_N", "0")) or None
prob = synth.make_problem(cfg, n=n, m=n)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
L.lsk_draw_anchors(p, U)
u = torch.empty(X.shape[0], dtype=torch.float32, device="cuda")
v = torch.empty(Y.shape[0], dtype=torch.float32, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
opts = L.make_opts(cfg.T)
res = {k: [] for k in arms}
out = {}
rounds = int(os.environ.get("AB_ROUNDS", "7"))
for rnd in range(rounds):
    for name, env in arms.items():
        for k, val in env.items():
            os.environ[k] = val
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=False)
        e1.record()
        e1.synchronize()
        if rnd > 0:
            res[name].append(e0.elapsed_time(e1))
        else:
            rep = L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v)
            out[name] = (rep["rot"] if isinstance(rep, dict) else rep.rot, u.clone(), v.clone())
        for k in env:
            del os.environ[k]
L.lsk_stream_status()
passes = 2 * cfg.T + 1
for name in arms:
    ms = np.array(res[name])
    print("config %d %-10s median %.3f ms (%.2f us/pass) min %.3f max %.3f -> %.0f it/s  rot %.12f"
          % (key, name, np.median(ms), 1e3 * np.median(ms) / passes, ms.min(), ms.max(),
             cfg.T / (np.median(ms) / 1e3), out[name][0]), flush=True)
names = list(arms)
r0, u0, v0 = out[names[0]]
for name in names[1:]:
    r1, u1, v1 = out[name]
    print("%s vs %s: rot rel %.2e, u max rel %.2e, v max rel %.2e, bit-identical %s" % (
        name, names[0], abs(r1 - r0) / abs(r0), float(((u1 - u0).abs() / u0).max()),
        float(((v1 - v0).abs() / v0).max()), bool(torch.equal(u0, u1) and torch.equal(v0, v1))))
