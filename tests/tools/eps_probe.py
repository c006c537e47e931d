"""Probe: smallest eps the fp32 GPU path handles on the config-2 generator (n = m = 4000,
r = 1000) vs the fp64 oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O, synth
import paper_2006_07057_b200 as L
cfg = synth.get_config(2)
prob = synth.make_problem(cfg, n=4000, m=4000)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
for eps in (0.1, 0.05, 0.03, 0.02, 0.01):
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], eps, cfg.r, cfg.anchor_seed, T=300)
    line = "eps %.3f oracle rot %.6f" % (eps, ref["rot"])
    for var in ("stream", "implicit"):
        try:
            res = L.rot(X, Y, a, b, eps, cfg.r, cfg.anchor_seed, iters=300, variant=var)
            line += " | %s %.6f rel %.1e" % (var, res["rot"], abs(res["rot"] - ref["rot"]) / abs(ref["rot"]))
        except Exception as e:
            line += " | %s FAIL %s" % (var, str(e)[:60])
    print(line, flush=True)
