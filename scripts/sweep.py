"""Kernel-time sweep for tuning: times lsk_factored_sinkhorn(_implicit) only (CUDA events)."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_07057_b200 as L
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--variant", default="stream")
ap.add_argument("--T", type=int, default=100)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--cps", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
ap2 = None
cfg = synth.get_config(a.config)
if a.config == 4:
    B = int(os.environ.get("SWEEP_BATCH", "256"))
    n = a.n or cfg.n
    bp = synth.make_batched(cfg, batch=B, n=n, m=n)
    X, Y, A_, B_ = (torch.from_numpy(bp[k]).cuda() for k in ("X", "Y", "a", "b"))
    r, d = cfg.r, cfg.d
    p = L.lsk_feature_params_init(cfg.eps, d, r, 0.0, cfg.anchor_seed, X.reshape(-1, d), Y.reshape(-1, d))
    U = torch.empty((r, d), device="cuda"); L.lsk_draw_anchors(p, U)
    Xi = torch.empty((B, n, r), device="cuda"); Ze = torch.empty((B, n, r), device="cuda")
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True); f1 = torch.cuda.Event(enable_timing=True)
    f0.record(); L.lsk_feature_map_batched(p, U, X, Xi); L.lsk_feature_map_batched(p, U, Y, Ze); f1.record()
    torch.cuda.synchronize()
    u = torch.empty((B, n), device="cuda"); v = torch.empty((B, n), device="cuda")
    opts = L.make_opts(a.T, 0.0, False, a.cps)
    run = lambda: L.lsk_factored_sinkhorn_batched(Xi, Ze, A_, B_, cfg.eps, opts, u, v, report=False)
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    bytes_ = 4.0 * r * B * (n + a.T * 2 * n)
    print(json.dumps(dict(variant="batched", B=B, n=n, r=r, T=a.T, feature_map_ms=round(f0.elapsed_time(f1), 3),
                          ms=round(ms, 3), GBs=round(bytes_ / ms / 1e6), it_s=round(a.T / ms * 1e3))))
    sys.exit(0)
prob = synth.make_problem(cfg, n=a.n, m=a.n)
X, Y, A_, B_ = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
n, m, r, d = X.shape[0], Y.shape[0], cfg.r, cfg.d
p = L.lsk_feature_params_init(cfg.eps, d, r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((r, d), device="cuda"); L.lsk_draw_anchors(p, U)
u = torch.empty(n, device="cuda"); v = torch.empty(m, device="cuda")
opts = L.make_opts(a.T, 0.0, False, a.cps)
if a.variant == "accel":   # Alg. 2: three factor passes per line-search trial
    Xi = torch.empty((n, r), device="cuda"); Ze = torch.empty((m, r), device="cuda")
    L.lsk_feature_map(p, U, X, Xi); L.lsk_feature_map(p, U, Y, Ze)
    reps = []
    def run():
        reps.append(L.lsk_accelerated_sinkhorn(Xi, Ze, A_, B_, cfg.eps, a.T))
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = min(ts); tr = reps[-1]["trials"]
    pass_bytes = 4.0 * r * (2 * m + n) * tr      # bytes the three passes of every trial read
    print(json.dumps(dict(variant="accel", n=n, r=r, T=a.T, trials=tr, ms=round(ms, 3),
                          us_per_iter=round(1e3 * ms / a.T, 2), us_per_trial=round(1e3 * ms / tr, 2),
                          pass_GBs=round(pass_bytes / ms / 1e6), F=reps[-1]["F"])))
    sys.exit(0)
if a.variant == "stream":
    Xi = torch.empty((n, r), device="cuda"); Ze = torch.empty((m, r), device="cuda")
    L.lsk_feature_map(p, U, X, Xi); L.lsk_feature_map(p, U, Y, Ze)
    run = lambda: L.lsk_factored_sinkhorn(Xi, Ze, A_, B_, cfg.eps, opts, u, v, report=False)
else:
    run = lambda: L.lsk_factored_sinkhorn_implicit(p, U, X, Y, A_, B_, opts, u, v, report=False)
run(); torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
ms = min(ts)
passes = 2 * a.T + 1
bytes_ = 4.0 * r * (n + a.T * (n + m))
print(json.dumps(dict(variant=a.variant, n=n, r=r, T=a.T, env={k: os.environ.get(k) for k in ("LSK_GPP", "LSK_NSTAGE")},
                      cps=a.cps, ms=round(ms, 3), us_per_pass=round(1e3 * ms / passes, 2),
                      GBs=round(bytes_ / ms / 1e6), it_s=round(a.T / ms * 1e3))))
