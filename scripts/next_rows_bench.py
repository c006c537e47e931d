"""Timing of the NEXT rows (f1-f4) on their workloads, kernel-level (CUDA events, min of 3
after a warm-up), with each one's algorithmic bytes or flops for a roofline fraction.
  f1 divergence  : config 2 (3 solves, T = 500), both variants
  f2 gradients   : config 2 at its scalings (one pass over Xi and Zeta + r x d outputs)
  f3 arc-cosine  : config 4 clouds (d = 128, tcgen05) and config 2 (d = 2, FFMA), s = 1
  f4 Alg. 2      : config 2, 100 iterations; f4 stabilised map: config 2, eps = 0.01
Prints one JSON line per measurement."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_07057_b200 as L
import synth

PEAK_HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6454.6) if os.path.exists("MEASURED_PEAKS.json") else 6454.6


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def emit(**kw):
    print(json.dumps(kw), flush=True)


cfg = synth.get_config(2)
prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
n, m, r, d = cfg.n, cfg.m, cfg.r, cfg.d

# f1: divergence, 3 solves of T = 500
for var in ("stream", "implicit"):
    ms = timed(lambda: L.sinkhorn_divergence(X, Y, a, b, cfg.eps, r, cfg.anchor_seed, iters=cfg.T, variant=var), reps=2)
    emit(row="f1", what="sinkhorn divergence (3 solves, T=500)", workload="config2", variant=var, ms=round(ms, 3),
         solves_per_s=round(3e3 / ms, 1), iter_per_s=round(3 * cfg.T * 1e3 / ms))

# f2: gradients at the config-2 scalings
p = L.lsk_feature_params_init(cfg.eps, d, r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((r, d), device="cuda"); L.lsk_draw_anchors(p, U)
Xi = torch.empty((n, r), device="cuda"); Ze = torch.empty((m, r), device="cuda")
L.lsk_feature_map(p, U, X, Xi); L.lsk_feature_map(p, U, Y, Ze)
u = torch.empty(n, device="cuda"); v = torch.empty(m, device="cuda")
L.lsk_factored_sinkhorn(Xi, Ze, a, b, cfg.eps, L.make_opts(cfg.T, 0.0, False, 0), u, v)
ms = timed(lambda: L.lsk_rot_gradient(p, U, X, Y, Xi, Ze, u, v))
gbytes = 4.0 * r * (n + m) * 2     # each factor read for s (xi^T u / zeta^T v) and for the row sums
emit(row="f2", what="envelope gradients dW/dX, dW/dY, dW/dU", workload="config2", ms=round(ms, 4),
     GBs=round(gbytes / ms / 1e6), hbm_frac=round(gbytes / ms / 1e6 / PEAK_HBM, 3),
     note="algorithmic bytes = two reads of each factor (4 r (n+m) x 2)")

# f3: arc-cosine features
for key in (4, 2):
    c = synth.get_config(key)
    nn = 1 << 20 if key == 4 else c.n
    Xa = torch.randn((nn, c.d), device="cuda") * (1.0 / c.d) ** 0.5
    pa = L.arccos_params(c.d, c.r, 1.5, c.anchor_seed, c.eps)
    Ua = torch.empty((c.r, c.d), device="cuda"); L.lsk_draw_anchors(pa, Ua)
    Xia = torch.empty((nn, c.r + 4), device="cuda")
    ms = timed(lambda: L.lsk_feature_map_arccos(pa, 1, 0.1, Ua, Xa, Xia))
    flops = 2.0 * nn * c.r * c.d
    wbytes = 4.0 * nn * (c.r + 4)
    emit(row="f3", what="arc-cosine feature map (s=1)", workload="config%d d=%d n=%d r=%d" % (key, c.d, nn, c.r), ms=round(ms, 4),
         TFLOPs_useful=round(flops / ms / 1e9, 1), write_GBs=round(wbytes / ms / 1e6),
         write_hbm_frac=round(wbytes / ms / 1e6 / PEAK_HBM, 3))

# f4: accelerated Sinkhorn and the stabilised feature map
res = {}
def acc():
    res["r"] = L.lsk_accelerated_sinkhorn(Xi, Ze, a, b, cfg.eps, 100)
ms = timed(acc, reps=2)
tr = res["r"]["trials"]
emit(row="f4", what="accelerated Sinkhorn (Alg. 2), 100 iterations", workload="config2", ms=round(ms, 3),
     trials=tr, us_per_trial=round(1e3 * ms / tr, 1), pass_GBs=round(4.0 * r * (n + 2 * m) * tr / ms / 1e6),
     pass_hbm_frac_of_trial=round(4.0 * r * (n + 2 * m) * tr / ms / 1e6 / PEAK_HBM, 3))
ps = L.lsk_feature_params_init(0.01, d, r, 0.0, cfg.anchor_seed, X, Y)
Us = torch.empty((r, d), device="cuda"); L.lsk_draw_anchors(ps, Us)
A = torch.empty(n, dtype=torch.float64, device="cuda")
ms_s = timed(lambda: L.lsk_feature_map_stabilized(ps, Us, X, Xi, A))
ms_p = timed(lambda: L.lsk_feature_map(ps, Us, X, Xi))
emit(row="f4", what="stabilised vs plain feature map (eps=0.01)", workload="config2 X", ms_stabilized=round(ms_s, 4),
     ms_plain=round(ms_p, 4), write_GBs_stabilized=round(4.0 * n * r / ms_s / 1e6),
     write_hbm_frac_stabilized=round(4.0 * n * r / ms_s / 1e6 / PEAK_HBM, 3))
