"""Run the hot path once (after one warm-up) for ncu captures: python scripts/prof_one.py
--config 2 --variant stream --T 50.  Prints the report; no timing claims."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--variant", default="stream")
ap.add_argument("--T", type=int, default=50)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--ctas-per-sm", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = synth.get_config(args.config)
prob = synth.make_problem(cfg, n=args.n, m=args.n)
X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
for _ in range(args.reps):
    res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=args.T, variant=args.variant,
                ctas_per_sm=args.ctas_per_sm)
torch.cuda.synchronize()
print(res["report"])
