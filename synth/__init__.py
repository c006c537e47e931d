"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module holds *only* input generation (points, weights, sizes, seeds).  It contains
none of the method's arithmetic: no feature map, no Lambert W, no Sinkhorn, no read-out.
Both sides (oracle/ and the CUDA path) receive the same fp32 arrays from here.

The five workloads are BASELINE.json ``configs`` (see DESIGN.md §"Input recipe"):

1. tiny        n=m=500,   d=2,   eps=0.5,  r=100,  T=200   (PAPER.md:58 distribution)
2. illus       n=m=40000, d=2,   eps=0.1,  r=1000, T=500   (Fig. 1 shape)
3. moddim      n=m=200000,d=16,  eps=0.2,  r=2048, T=1000  (Dirichlet(1) weights)
4. batched     256 pairs, n=m=4096, d=128, eps=1.0, r=512, T=300 (shared anchors)
5. large       n=m=2^23,  d=3,   eps=0.05, r=4096, T=200   (8-component mixture)

Reading C15: "N(0, 0.1 I)" is variance 0.1; "N(1, I)" has mean (1,..,1);
"rescaled by max norm" divides a cloud by its own max norm; "clipped to unit ball" is the
radial projection p <- p / max(1, |p|).  Uniform weights are fp32(1/n); Dirichlet weights
are drawn in fp64 and cast to fp32 without renormalisation (C10).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    key: int
    name: str
    n: int
    m: int
    d: int
    eps: float
    r: int
    T: int
    batch: int = 1
    data_seed: int = 0
    anchor_seed: int = 0
    description: str = ""


CONFIGS = {
    1: Config(1, "tiny", 500, 500, 2, 0.5, 100, 200, 1, 20061, 7058,
              "x~N(0,0.1I), y~N(1,I)/max|y|, uniform weights"),
    2: Config(2, "illus", 40000, 40000, 2, 0.1, 1000, 500, 1, 20062, 7059,
              "Fig.1 shape: x~N(0,0.1I), y~N(1,I)/max|y|, uniform weights"),
    3: Config(3, "moddim", 200000, 200000, 16, 0.2, 2048, 1000, 1, 20063, 7060,
              "x~N(0,I)/max, y~N(0.5*1,2I)/max, Dirichlet(1) weights"),
    4: Config(4, "batched", 4096, 4096, 128, 1.0, 512, 300, 256, 20064, 7061,
              "256 pairs x,y~N(0,I/d) seeded 40000+p, uniform, shared anchors"),
    5: Config(5, "large", 1 << 23, 1 << 23, 3, 0.05, 4096, 200, 1, 20065, 7062,
              "x~8-Gaussian mixture (var .05, means U[-1,1]^3), y~N(0,.5I), clipped"),
}


def get_config(key: int, **overrides) -> Config:
    return dataclasses.replace(CONFIGS[key], **overrides)


def _uniform_weights(n: int) -> np.ndarray:
    return np.full(n, 1.0 / n, dtype=np.float64).astype(np.float32)


def _gauss_pair_illus(rng: np.random.Generator, n: int, m: int, d: int):
    # PAPER.md:58 / 432: mu = N(0, 0.1 I_d), nu = N(1, I_d) scaled by its max norm.
    x = rng.normal(0.0, np.sqrt(0.1), size=(n, d))
    y = rng.normal(1.0, 1.0, size=(m, d))
    y = y / np.max(np.linalg.norm(y, axis=1))
    return x, y


def _moddim(rng: np.random.Generator, n: int, m: int, d: int):
    x = rng.normal(0.0, 1.0, size=(n, d))
    y = rng.normal(0.5, np.sqrt(2.0), size=(m, d))
    x = x / np.max(np.linalg.norm(x, axis=1))
    y = y / np.max(np.linalg.norm(y, axis=1))
    a = rng.dirichlet(np.ones(n))
    b = rng.dirichlet(np.ones(m))
    return x, y, a, b


def _clip_unit(p: np.ndarray) -> np.ndarray:
    nrm = np.linalg.norm(p, axis=1, keepdims=True)
    return p / np.maximum(1.0, nrm)


def _large(rng: np.random.Generator, n: int, m: int, d: int):
    means = rng.uniform(-1.0, 1.0, size=(8, d))
    comp = rng.integers(0, 8, size=n)
    x = means[comp] + rng.normal(0.0, np.sqrt(0.05), size=(n, d))
    y = rng.normal(0.0, np.sqrt(0.5), size=(m, d))
    return _clip_unit(x), _clip_unit(y)


def make_problem(cfg: Config, n: Optional[int] = None, m: Optional[int] = None,
                 pair: int = 0, identical_points: bool = False) -> dict:
    """Return fp32 arrays X (n,d), Y (m,d), a (n,), b (m,) for one problem of ``cfg``.

    ``n``/``m`` override the sizes (reduced or ragged test sizes); the distribution is
    unchanged.  ``pair`` selects the per-pair seed of config 4.  ``identical_points``
    replaces every x_i by x_0 and every y_j by y_0 (rank-one kernel, pin P11).
    """
    n = cfg.n if n is None else n
    m = cfg.m if m is None else m
    d = cfg.d
    if cfg.key == 4:
        rng = np.random.default_rng(40000 + pair)
        x = rng.normal(0.0, np.sqrt(1.0 / d), size=(n, d))
        y = rng.normal(0.0, np.sqrt(1.0 / d), size=(m, d))
        a, b = None, None
    else:
        rng = np.random.default_rng(cfg.data_seed)
        if cfg.key in (1, 2):
            x, y = _gauss_pair_illus(rng, n, m, d)
            a, b = None, None
        elif cfg.key == 3:
            x, y, a, b = _moddim(rng, n, m, d)
        elif cfg.key == 5:
            x, y = _large(rng, n, m, d)
            a, b = None, None
        else:
            raise ValueError(cfg.key)
    if identical_points:
        x = np.repeat(x[:1], n, axis=0)
        y = np.repeat(y[:1], m, axis=0)
    a = _uniform_weights(n) if a is None else a.astype(np.float32)
    b = _uniform_weights(m) if b is None else b.astype(np.float32)
    return dict(X=np.ascontiguousarray(x, dtype=np.float32),
                Y=np.ascontiguousarray(y, dtype=np.float32),
                a=a, b=b, eps=cfg.eps, r=cfg.r, T=cfg.T, seed=cfg.anchor_seed, d=d)


def make_batched(cfg: Config, batch: Optional[int] = None, n: Optional[int] = None,
                 m: Optional[int] = None) -> dict:
    """Config 4: ``batch`` independent pairs stacked as X (B,n,d), Y (B,m,d), a (B,n), b (B,m)."""
    batch = cfg.batch if batch is None else batch
    probs = [make_problem(cfg, n=n, m=m, pair=p) for p in range(batch)]
    return dict(X=np.stack([p["X"] for p in probs]), Y=np.stack([p["Y"] for p in probs]),
                a=np.stack([p["a"] for p in probs]), b=np.stack([p["b"] for p in probs]),
                eps=cfg.eps, r=cfg.r, T=cfg.T, seed=cfg.anchor_seed, d=cfg.d)


def random_small(seed: int, n: int, m: int, d: int, spread: float = 0.5) -> dict:
    """Small generic problem with non-uniform positive weights (for pins / edge cases)."""
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, spread, size=(n, d))
    y = rng.normal(0.3, spread, size=(m, d))
    a = rng.uniform(0.5, 1.5, size=n)
    b = rng.uniform(0.5, 1.5, size=m)
    return dict(X=x.astype(np.float32), Y=y.astype(np.float32),
                a=(a / a.sum()).astype(np.float32), b=(b / b.sum()).astype(np.float32))
