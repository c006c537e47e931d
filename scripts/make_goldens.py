"""Write the full-size parity goldens of configs 3, 4 and 5 (tests/golden/full_config*.npz).

Calls ONLY ``oracle/`` (the fp64 CPU oracle) and ``synth/`` (the seeded inputs): no value here
comes from the CUDA path.  Each golden is the oracle's Alg. 1 run for the
config's full T from u^0 = 1 on the config's full-size inputs, followed by the dual estimate
(PAPER.md:261).  Stored: the ROT value, the iteration count, the final marginal error, and u, v
at a fixed sample of row indices (spread over the whole range, plus the first and last 64 rows:
the ragged tails of the GPU's CTA partition) — the GPU parity tests compare element by element
at those indices (tests/test_gpu_full.py).

  config 3 (n=m=200000, d=16, r=2048, T=1000): numpy oracle on materialised fp64 factors.
  config 4 (256 pairs, n=m=4096, d=128, r=512, T=300): numpy oracle per pair; one anchor draw
           with R = max norm over all 256 pairs (reading C3).
  config 5 (n=m=2^23, d=3, r=4096, T=200): the matrix-free plain-C oracle (oracle/lsk_oracle_mf.c,
           OpenMP; fp64 factors would take 550 GB), anchors from the numpy oracle.

Usage: python scripts/make_goldens.py 3 4 5      (config 5 takes about an hour on 8 cores)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def sample_rows(total: int, k: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = np.concatenate([np.arange(min(64, total)), np.arange(max(0, total - 64), total),
                          rng.choice(total, size=min(k, total), replace=False)])
    return np.unique(idx).astype(np.int64)


def golden_config3():
    cfg = synth.get_config(3)
    prob = synth.make_problem(cfg)
    t0 = time.time()
    res = oracle.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r,
                     cfg.anchor_seed, T=cfg.T)
    err = oracle.marginal_error(res["u"], res["v"],
                                res["zeta"].T @ (res["xi"] @ res["u"]), prob["b"])
    iu = sample_rows(cfg.n, 4096, 31)
    iv = sample_rows(cfg.m, 4096, 32)
    out = dict(rot=res["rot"], T=cfg.T, iters=res["iters"], marginal_err=err,
               R=res["params"]["R"], iu=iu, u=res["u"][iu], iv=iv, v=res["v"][iv],
               seconds=time.time() - t0)
    np.savez_compressed(os.path.join(GOLD, "full_config3.npz"), **out)
    print("config 3: rot=%.15g err=%.3g %.0fs" % (out["rot"], err, out["seconds"]), flush=True)


def golden_config4():
    cfg = synth.get_config(4)
    B = cfg.batch
    t0 = time.time()
    R = 0.0
    for p in range(B):   # reading C3: one R over all pairs (shared anchor draw)
        pr = synth.make_problem(cfg, pair=p)
        R = max(R, oracle.max_norm(pr["X"], pr["Y"]))
    idx = sample_rows(cfg.n, 192, 41)
    rots, us, vs, errs = [], [], [], []
    for p in range(B):
        pr = synth.make_problem(cfg, pair=p)
        res = oracle.rot(pr["X"], pr["Y"], pr["a"], pr["b"], cfg.eps, cfg.r, cfg.anchor_seed,
                         T=cfg.T, R=R)
        rots.append(res["rot"])
        us.append(res["u"][idx])
        vs.append(res["v"][idx])
        errs.append(oracle.marginal_error(res["u"], res["v"],
                                          res["zeta"].T @ (res["xi"] @ res["u"]), pr["b"]))
        if p % 32 == 0:
            print("config 4 pair %d rot=%.12g %.0fs" % (p, res["rot"], time.time() - t0), flush=True)
    out = dict(rot=np.array(rots), T=cfg.T, R=R, idx=idx, u=np.array(us), v=np.array(vs),
               marginal_err=np.array(errs), seconds=time.time() - t0)
    np.savez_compressed(os.path.join(GOLD, "full_config4.npz"), **out)
    print("config 4: %d pairs %.0fs" % (B, out["seconds"]), flush=True)


def golden_config5():
    from oracle import matrix_free as mf
    cfg = synth.get_config(5)
    prob = synth.make_problem(cfg)
    t0 = time.time()
    R = oracle.max_norm(prob["X"], prob["Y"])
    prm = oracle.gaussian_params(cfg.eps, cfg.d, cfg.r, R)
    U = oracle.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
    sol = mf.sinkhorn_matrix_free(prob["X"], prob["Y"], U, prob["a"], prob["b"], cfg.eps,
                                  prm["q"], T=cfg.T, record_last_err=True, verbose=True)
    iu = sample_rows(cfg.n, 4096, 51)
    iv = sample_rows(cfg.m, 4096, 52)
    rot = oracle.dual_estimate(sol["u"], sol["v"], prob["a"], prob["b"], cfg.eps)
    out = dict(rot=rot, T=cfg.T, iters=sol["iters"], marginal_err=sol["last_err"], R=R,
               iu=iu, u=sol["u"][iu], iv=iv, v=sol["v"][iv], seconds=time.time() - t0)
    np.savez_compressed(os.path.join(GOLD, "full_config5.npz"), **out)
    print("config 5: rot=%.15g err=%.3g %.0fs" % (rot, out["marginal_err"], out["seconds"]),
          flush=True)


if __name__ == "__main__":
    todo = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
    for k in todo:
        {3: golden_config3, 4: golden_config4, 5: golden_config5}[k]()
