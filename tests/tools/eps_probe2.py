"""Probe: the stabilised stream path (row log-offsets, reading C30) at small eps vs the fp64
oracle (config-2 generator, n = m = 4000, r = 1000, T = 300)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O, synth
import paper_2006_07057_b200 as L
cfg = synth.get_config(2)
prob = synth.make_problem(cfg, n=4000, m=4000)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
for eps in (0.1, 0.05, 0.02, 0.015, 0.01, 0.007, 0.005):
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], eps, cfg.r, cfg.anchor_seed, T=300)
    line = "eps %.3f oracle rot %.8f" % (eps, ref["rot"])
    for var in ("stream", "implicit"):
        try:
            res = L.rot(X, Y, a, b, eps, cfg.r, cfg.anchor_seed, iters=300, stabilize=True, variant=var)
            line += " | %s-stab %.8f rel %.1e" % (var, res["rot"], abs(res["rot"] - ref["rot"]) / abs(ref["rot"]))
        except Exception as e:
            line += " | %s-stab FAIL %s" % (var, str(e)[:40])
    print(line, flush=True)
