"""ORACLE — matrix-free Alg. 1 for inputs whose fp64 factors do not fit in host memory.

TEST INFRASTRUCTURE ONLY (see oracle/lsk_oracle.py).  The two factor products run in plain C
(oracle/lsk_oracle_mf.c, OpenMP, fp64, every entry regenerated in the direct difference form of
PAPER.md:934 with the 1/sqrt(r) of PAPER.md:297); this module is Alg. 1
written out over them, exactly as ``lsk_oracle.sinkhorn``:
    u^0 = 1;  repeat T times:  v <- b / K^T u ;  u <- a / K v,
with K^T u = zeta^T (xi u) and K v = xi^T (zeta v) (K_theta = xi^T zeta).
Pinned in tests/test_oracle_matrix_free.py against the numpy oracle (materialised factors) and
the rank-one closed form (P11).

The shared library is built by ``build_lib()`` (called by __graft_entry__.build()) or on first
use; LSK_ORACLE_MARCH overrides the -march (default x86-64-v3: AVX2 + FMA).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lsk_oracle_mf.c")
_LIB = os.path.join(_HERE, "liblsk_oracle_mf.so")
_lib = None


def build_lib(force: bool = False) -> str:
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    march = os.environ.get("LSK_ORACLE_MARCH", "x86-64-v3")
    tmp = "%s.%d.tmp" % (_LIB, os.getpid())   # renamed into place: a loaded copy stays valid
    cmd = ["gcc", "-O3", "-march=" + march, "-fno-math-errno", "-fopenmp", "-fPIC", "-shared",
           _SRC, "-o", tmp, "-lm", "-lmvec"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("oracle C build failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        dp = ctypes.POINTER(ctypes.c_double)
        for name in ("lsk_mf_apply", "lsk_mf_apply_t"):
            fn = getattr(_lib, name)
            fn.restype = None
            fn.argtypes = [dp, ctypes.c_int64, dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                           ctypes.c_double, dp, dp]
        _lib.lsk_mf_half.restype = None
        _lib.lsk_mf_half.argtypes = [dp, ctypes.c_int64, dp, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, dp, dp, dp, dp, dp]
        _lib.lsk_mf_threads.restype = ctypes.c_int
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def threads() -> int:
    return int(_load().lsk_mf_threads())


def apply(P, U, eps: float, q: float, w) -> np.ndarray:
    """xi w = (sum_i xi[k][i] w_i)_k for the features xi of the points P (np x d) under the
    anchors U (r x d); r outputs."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    s = np.empty(U.shape[0])
    _load().lsk_mf_apply(_p(P), P.shape[0], _p(U), U.shape[0], U.shape[1], eps, q, _p(w), _p(s))
    return s


def apply_t(P, U, eps: float, q: float, s) -> np.ndarray:
    """xi^T s = (sum_k xi[k][i] s_k)_i; np outputs."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.empty(P.shape[0])
    _load().lsk_mf_apply_t(_p(P), P.shape[0], _p(U), U.shape[0], U.shape[1], eps, q, _p(s),
                           _p(out))
    return out


def half_iteration(P, U, eps: float, q: float, s, c):
    """One half-iteration of Alg. 1 over one side's points P: t = xi^T s (the
    kernel product K^T u or K v, as s = xi u or zeta v), out = c / t, and the product the next
    half-iteration needs, s_next = xi out.  Returns (out, t, s_next)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    out = np.empty(P.shape[0])
    t = np.empty(P.shape[0])
    s_next = np.empty(U.shape[0])
    _load().lsk_mf_half(_p(P), P.shape[0], _p(U), U.shape[0], U.shape[1], eps, q, _p(s), _p(c),
                        _p(out), _p(t), _p(s_next))
    return out, t, s_next


def sinkhorn_matrix_free(X, Y, U, a, b, eps: float, q: float, T: int,
                         record_last_err: bool = False, verbose: bool = False) -> dict:
    """Alg. 1 for exactly T iterations from u^0 = 1 (reading C6) on
    K_theta = xi^T zeta, xi = phi_theta(X), zeta = phi_theta(Y).  With record_last_err the
    stopping quantity |v o K^T u - b|_1 of the final (u, v) is evaluated."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    u = np.ones(X.shape[0])
    v = np.ones(Y.shape[0])
    t0 = time.time()
    s_v = apply(X, U, eps, q, u)                                   # xi u^0
    for t in range(T):
        v, _, s_u = half_iteration(Y, U, eps, q, s_v, b)           # v <- b / K^T u ; zeta v
        u, _, s_v = half_iteration(X, U, eps, q, s_u, a)           # u <- a / K v   ; xi u
        if verbose and (t % 10 == 0 or t == T - 1):
            print("  matrix-free iteration %d/%d  %.0fs" % (t + 1, T, time.time() - t0), flush=True)
    out = dict(u=u, v=v, iters=T)
    if record_last_err:                                            # |v o K^T u - b|_1
        out["last_err"] = float(np.abs(v * apply_t(Y, U, eps, q, s_v) - b).sum())
    return out

    # (each half-iteration regenerates every entry of its side once and uses it in both sums
    #  that contain it: the same sums as apply_t(P, .., apply(..)) — pinned in
    #  tests/test_oracle_matrix_free.py)
