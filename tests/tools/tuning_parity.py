"""Parity of the TUNING build's alternatives (scripts/variants/liblsk_tuning.so, built with
`python paper_2006_07057_b200/build.py --tuning`) against the fp64 oracle: the implicit
kernel's expanded exponent forced (LSK_FACT=0) and every instantiated alternative
configuration (pipelined teams, warp-private kernel, the round-1 hybrid with stream warps).
The product liblsk.so contains none of these.  usage (GPU): python tests/tools/tuning_parity.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LSK_LIB_PATH"] = os.path.join(ROOT, "scripts", "variants", "liblsk_tuning.so")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

CASES = [
    (2, 4099, 3907, 200, {"LSK_ICFG": "128,4,2,4,0"}),
    (2, 4099, 3907, 200, {"LSK_ICFG": "128,3,2,8,0"}),
    (2, 4099, 3907, 200, {"LSK_IWARP": "1"}),
    (2, 4099, 3907, 200, {"LSK_IWARP": "1", "LSK_IWCFG": "8,8,2"}),
    (2, 4099, 3907, 200, {"LSK_ICFG": "128,2,2,8,1"}),
    (5, 6151, 6143, 40, {"LSK_ICFG": "512,1,2,4,0"}),
    (5, 6151, 6143, 40, {"LSK_ICFG": "256,1,4,2,1"}),
    (1, 500, 500, 200, {"LSK_IWARP": "1"}),
    (1, 500, 500, 200, {"LSK_IWARP": "1", "LSK_IWCFG": "8,4,4"}),
]
bad = 0
for fact in ("0", "1"):
    for key, n, m, T, env in CASES:
        for k in ("LSK_ICFG", "LSK_IWARP", "LSK_IWCFG"):
            os.environ.pop(k, None)
        os.environ.update(env)
        os.environ["LSK_FACT"] = fact
        cfg = synth.get_config(key)
        prob = synth.make_problem(cfg, n=n, m=m)
        ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
        X, Y, a, b = (torch.from_numpy(prob[k]).cuda() for k in ("X", "Y", "a", "b"))
        res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant="implicit",
                    stream_fraction=-1.0)
        re = abs(res["rot"] - ref["rot"]) / abs(ref["rot"])
        ue = float(np.max(np.abs(res["u"].cpu().double().numpy() - ref["u"]) / ref["u"]))
        ve = float(np.max(np.abs(res["v"].cpu().double().numpy() - ref["v"]) / ref["v"]))
        ok = re <= 1e-5 and ue <= 1e-4 and ve <= 1e-4
        bad += not ok
        print("%s FACT=%s config %d %s: rot %.1e u %.1e v %.1e" % ("ok " if ok else "BAD", fact, key,
                                                                   env, re, ue, ve), flush=True)
sys.exit(1 if bad else 0)
