"""One small solve per variant for compute-sanitizer (racecheck / synccheck / memcheck), one
tool per gpurun call (B200_PROFILING.md).  Cases exercise every synchronisation pattern of the
persistent kernels: mbarrier rings (stream producer/consumers, implicit loaders), named team
barriers, the cross-CTA group barrier with sentinel polling (gpp > 1), the batched problem loop
(groups of gpp CTAs over several problems) and the emulated cross-rank exchange.
usage: python scripts/sanitize_case.py [case ...]   (default: all)"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def single(variant, key, n, T):
    cfg = synth.get_config(key)
    prob = synth.make_problem(cfg, n=n, m=n - 3)
    X, Y, a, b = (dev(prob[k]) for k in ("X", "Y", "a", "b"))
    res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant=variant)
    print(variant, key, n, "rot", res["rot"], flush=True)


def tol_mode(variant):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    X, Y, a, b = (dev(prob[k]) for k in ("X", "Y", "a", "b"))
    res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, max_iters=100, tol=1e-6, variant=variant)
    print("tol", variant, res["report"]["iters"], flush=True)


def batched_loop():
    cfg = synth.get_config(4)
    B, n = 12, 1024
    bp = synth.make_batched(cfg, batch=B, n=n, m=n)
    X, Y, a, b = (dev(bp[k]) for k in ("X", "Y", "a", "b"))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, 1, X.reshape(-1, cfg.d), Y.reshape(-1, cfg.d))
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((B, n, cfg.r), dtype=torch.float32, device="cuda")
    Ze = torch.empty((B, n, cfg.r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map_batched(p, U, X, Xi)
    L.lsk_feature_map_batched(p, U, Y, Ze)
    u = torch.empty((B, n), dtype=torch.float32, device="cuda")
    v = torch.empty((B, n), dtype=torch.float32, device="cuda")
    reps = L.lsk_factored_sinkhorn_batched(Xi, Ze, a, b, cfg.eps, L.make_opts(5), u, v)
    print("batched", L.lsk_solve_plan(n, n, cfg.r, 1, B, "stream"), reps[0].rot, flush=True)


def emulated(variant):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    X, Y, a, b = (dev(prob[k]) for k in ("X", "Y", "a", "b"))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(500, dtype=torch.float32, device="cuda")
    v = torch.empty(500, dtype=torch.float32, device="cuda")
    if variant == "stream":
        Xi = torch.empty((500, cfg.r), dtype=torch.float32, device="cuda")
        Ze = torch.empty((500, cfg.r), dtype=torch.float32, device="cuda")
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
        reps = L.lsk_factored_sinkhorn_emulated(2, Xi, Ze, a, b, cfg.eps, L.make_opts(5), u, v)
    else:
        reps = L.lsk_factored_sinkhorn_implicit_emulated(2, p, U, X, Y, a, b, L.make_opts(5), u, v)
    print("emulated", variant, reps[0].rot, flush=True)


CASES = {
    "c1_stream": lambda: single("stream", 1, 500, 6),
    "c1_implicit": lambda: single("implicit", 1, 500, 6),
    "c2_stream": lambda: single("stream", 2, 3001, 3),
    "c2_implicit": lambda: single("implicit", 2, 3001, 3),
    "c5_implicit": lambda: single("implicit", 5, 2049, 2),
    "tol_stream": lambda: tol_mode("stream"),
    "tol_implicit": lambda: tol_mode("implicit"),
    "batched": batched_loop,
    "emul_stream": lambda: emulated("stream"),
    "emul_implicit": lambda: emulated("implicit"),
}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
    torch.cuda.synchronize()
    L.lsk_stream_status()
    print("sanitize_case done", flush=True)
