"""Debug helper (GPU): one emulated-rank or cluster-mode case, printing as it goes."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def emul(variant, N, n, T, key=2):
    cfg = synth.get_config(key)
    prob = synth.make_problem(cfg, n=n, m=n)
    X, Y, a, b = (dev(prob[k]) for k in ("X", "Y", "a", "b"))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    v = torch.empty(n, dtype=torch.float32, device="cuda")
    t0 = time.time()
    if variant == "stream":
        Xi = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
        Ze = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
        reps = L.lsk_factored_sinkhorn_emulated(N, Xi, Ze, a, b, cfg.eps, L.make_opts(T), u, v)
    else:
        reps = L.lsk_factored_sinkhorn_implicit_emulated(N, p, U, X, Y, a, b, L.make_opts(T), u, v)
    single = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant=variant)
    print("emul", variant, N, n, T, "%.2fs" % (time.time() - t0), [rp.rot for rp in reps],
          single["rot"], flush=True)


def cluster(variant, n, T):
    cfg = synth.get_config(1)
    print("plan", L.lsk_solve_plan(n, n, cfg.r, cfg.d, 1, variant, cluster=True), flush=True)
    prob = synth.make_problem(cfg, n=n, m=n)
    X, Y, a, b = (dev(prob[k]) for k in ("X", "Y", "a", "b"))
    t0 = time.time()
    res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant=variant)
    print("cluster", variant, n, T, "%.3fs" % (time.time() - t0), res["rot"], flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "emul":
        emul(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
    else:
        cluster(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
