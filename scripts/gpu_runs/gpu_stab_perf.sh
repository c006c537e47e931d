python scripts/eps_probe2.py
python - <<'PY'
import sys, os, json; sys.path.insert(0, '.')
import torch, paper_2006_07057_b200 as L, synth
cfg = synth.get_config(2); prob = synth.make_problem(cfg)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
p = L.lsk_feature_params_init(cfg.eps, 2, cfg.r, 0.0, cfg.anchor_seed, X, Y)
U = torch.empty((cfg.r, 2), device="cuda"); L.lsk_draw_anchors(p, U)
u = torch.empty(cfg.n, device="cuda"); v = torch.empty(cfg.m, device="cuda")
for stab in (False, True):
    o = L.make_opts(cfg.T, 0.0, False, 0, stabilize=stab)
    f = lambda: L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, o, u, v, report=False)
    f(); torch.cuda.synchronize(); best = 1e9
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(json.dumps(dict(stabilize=stab, ms=round(best, 3), it_s=round(cfg.T * 1e3 / best))))
PY
