"""lsk — B200 (sm_100a) linear-time Sinkhorn with positive features (arXiv 2006.07057).

Thin ctypes binding over ``liblsk.so`` (C ABI: include/lsk.h).  Every function here only
marshals arguments (torch CUDA tensors -> device pointers, the current CUDA stream ->
cudaStream_t); every step of the method runs in the library's CUDA kernels.  There is no
CPU fallback: importing this package without the built library raises ImportError, and the
calls raise LskError on any library error.

Function names mirror the C ABI: lsk_feature_params_init, lsk_draw_anchors,
lsk_feature_map(_batched), lsk_factored_sinkhorn(_implicit|_batched),
lsk_rot_value(_batched), lsk_rot_host, lsk_comm_*, lsk_shard_range.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSK_LIB_PATH") or os.path.join(_HERE, "liblsk.so")   # override: tuning builds

if not os.path.exists(LIB_PATH):
    raise ImportError("liblsk.so not built: run `python -m paper_2006_07057_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

c_f32p = ctypes.c_void_p
c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32


class lsk_feature_params(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("R", ctypes.c_double), ("q", ctypes.c_double),
                ("sigma", ctypes.c_double), ("log_scale", ctypes.c_double),
                ("d", c_i32), ("r", c_i32), ("seed", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class lsk_solve_opts(ctypes.Structure):
    _fields_ = [("max_iters", c_i32), ("want_marginal_err", c_i32), ("tol", ctypes.c_double),
                ("ctas_per_sm", c_i32), ("flags", c_i32), ("stream_fraction", ctypes.c_double)]


class lsk_report(ctypes.Structure):
    _fields_ = [("iters", c_i32), ("converged", c_i32), ("marginal_err", ctypes.c_double),
                ("rot", ctypes.c_double), ("sum_a_log_u", ctypes.c_double),
                ("sum_b_log_v", ctypes.c_double), ("breakdown", c_i32), ("reserved", c_i32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class lsk_accel_opts(ctypes.Structure):
    _fields_ = [("max_iters", c_i32), ("reserved", c_i32), ("tol", ctypes.c_double),
                ("L0", ctypes.c_double)]


class lsk_accel_report(ctypes.Structure):
    _fields_ = [("iters", c_i32), ("trials", c_i32), ("converged", c_i32), ("reserved", c_i32),
                ("F", ctypes.c_double), ("L", ctypes.c_double), ("plan_err", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


P = ctypes.POINTER
_SIGS = {
    "lsk_version": (ctypes.c_char_p, []),
    "lsk_last_error": (ctypes.c_char_p, []),
    "lsk_launch_count": (c_i64, [c_i32]),
    "lsk_stream_status": (c_i32, [ctypes.c_void_p]),
    "lsk_stream_rows": (c_i32, [c_i64, c_i64, c_i32, c_i32, P(lsk_solve_opts), P(c_i64), P(c_i64)]),
    "lsk_factored_sinkhorn_emulated": (c_i32, [c_i32, c_f32p, c_i64, c_f32p, c_i64, c_i32, c_f32p,
                                               c_f32p, ctypes.c_double, P(lsk_solve_opts), c_f32p,
                                               c_f32p, ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_factored_sinkhorn_implicit_emulated": (c_i32, [c_i32, P(lsk_feature_params), c_f32p,
                                                        c_f32p, c_i64, c_f32p, c_i64, c_f32p,
                                                        c_f32p, P(lsk_solve_opts), c_f32p,
                                                        c_f32p, ctypes.c_void_p,
                                                        ctypes.c_void_p]),
    "lsk_solve_plan": (c_i32, [c_i64, c_i64, c_i32, c_i32, c_i32, c_i32, P(c_i32), P(c_i32),
                               P(c_i32)]),
    "lsk_resident_plan": (c_i32, [c_i64, c_i64, c_i32, P(c_i32)]),
    "lsk_lambert_w0": (c_i32, [ctypes.c_double, P(ctypes.c_double)]),
    "lsk_feature_params_init": (c_i32, [ctypes.c_double, c_i32, c_i32, ctypes.c_double,
                                        ctypes.c_uint64, c_f32p, c_i64, c_f32p, c_i64,
                                        P(lsk_feature_params), ctypes.c_void_p,
                                        ctypes.c_void_p]),
    "lsk_draw_anchors": (c_i32, [P(lsk_feature_params), c_f32p, ctypes.c_void_p]),
    "lsk_philox_words": (c_i32, [ctypes.c_uint64, c_i32, c_i32, ctypes.c_void_p,
                                 ctypes.c_void_p]),
    "lsk_feature_map": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64, c_f32p,
                                ctypes.c_void_p]),
    "lsk_feature_map_batched": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64, c_i32,
                                        c_f32p, ctypes.c_void_p]),
    "lsk_feature_map_arccos": (c_i32, [P(lsk_feature_params), c_i32, ctypes.c_double, c_f32p,
                                       c_f32p, c_i64, c_f32p, ctypes.c_void_p]),
    "lsk_factored_sinkhorn": (c_i32, [c_f32p, c_i64, c_f32p, c_i64, c_i32, c_f32p, c_f32p,
                                      ctypes.c_double, P(lsk_solve_opts), c_f32p, c_f32p,
                                      P(lsk_report), ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_factored_sinkhorn_implicit": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64,
                                               c_f32p, c_i64, c_f32p, c_f32p,
                                               P(lsk_solve_opts), c_f32p, c_f32p,
                                               P(lsk_report), ctypes.c_void_p,
                                               ctypes.c_void_p]),
    "lsk_factored_sinkhorn_batched": (c_i32, [c_f32p, c_i64, c_f32p, c_i64, c_i32, c_i32,
                                              c_f32p, c_f32p, ctypes.c_double,
                                              P(lsk_solve_opts), c_f32p, c_f32p,
                                              ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_factored_sinkhorn_implicit_batched": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p,
                                                       c_i64, c_f32p, c_i64, c_i32, c_f32p,
                                                       c_f32p, P(lsk_solve_opts), c_f32p,
                                                       c_f32p, ctypes.c_void_p,
                                                       ctypes.c_void_p]),
    "lsk_rot_value": (c_i32, [c_f32p, c_f32p, c_f32p, c_f32p, c_i64, c_i64, ctypes.c_double,
                              P(ctypes.c_double), ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_rot_value_batched": (c_i32, [c_f32p, c_f32p, c_f32p, c_f32p, c_i64, c_i64, c_i32,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_sinkhorn_divergence": (c_i32, [c_f32p, c_i64, c_f32p, c_i64, c_i32, c_f32p, c_f32p,
                                        ctypes.c_double, P(lsk_solve_opts), ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_sinkhorn_divergence_implicit": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64,
                                                 c_f32p, c_i64, c_f32p, c_f32p,
                                                 P(lsk_solve_opts), ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_rot_gradient": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64, c_f32p, c_i64,
                                 c_f32p, c_f32p, c_f32p, c_f32p, c_f32p, c_f32p, c_f32p,
                                 ctypes.c_void_p]),
    "lsk_implicit_row_offsets": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64,
                                         ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_feature_map_stabilized": (c_i32, [P(lsk_feature_params), c_f32p, c_f32p, c_i64, c_f32p,
                                           ctypes.c_void_p, ctypes.c_void_p]),
    "lsk_rot_value_offset": (c_i32, [c_f32p, c_f32p, c_f32p, c_f32p, ctypes.c_void_p,
                                     ctypes.c_void_p, c_i64, c_i64, ctypes.c_double,
                                     P(ctypes.c_double), ctypes.c_void_p]),
    "lsk_accelerated_sinkhorn": (c_i32, [c_f32p, c_i64, c_f32p, c_i64, c_i32, c_f32p, c_f32p,
                                         ctypes.c_double, P(lsk_accel_opts), ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, P(lsk_accel_report),
                                         ctypes.c_void_p]),
    "lsk_rot_host": (c_i32, [c_f32p, c_i64, c_f32p, c_i64, c_i32, c_f32p, c_f32p,
                             ctypes.c_double, c_i32, ctypes.c_uint64, ctypes.c_double,
                             P(lsk_solve_opts), c_i32, c_f32p, c_f32p, P(lsk_report)]),
    "lsk_shard_range": (c_i32, [c_i64, c_i32, c_i32, P(c_i64), P(c_i64)]),
    "lsk_comm_get_unique_id": (c_i32, [ctypes.c_void_p]),
    "lsk_comm_init": (c_i32, [P(ctypes.c_void_p), c_i32, c_i32, ctypes.c_void_p, c_i32]),
    "lsk_comm_destroy": (c_i32, [ctypes.c_void_p]),
    "lsk_comm_enable_p2p": (c_i32, [ctypes.c_void_p, c_i32, ctypes.c_void_p]),
}
EXPORTED = sorted(_SIGS)
for _name, (_res, _args) in _SIGS.items():
    if not hasattr(_lib, _name):
        raise ImportError("liblsk.so is stale (missing %s): rebuild with "
                          "`python paper_2006_07057_b200/build.py`" % _name)
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

LSK_OK, LSK_NOT_CONVERGED = 0, 1
STATUS_NAMES = {0: "LSK_OK", 1: "LSK_NOT_CONVERGED", -1: "LSK_EINVAL", -2: "LSK_EDIM",
                -3: "LSK_EDOMAIN", -4: "LSK_EWEIGHTS", -5: "LSK_EBREAKDOWN", -6: "LSK_ECUDA",
                -7: "LSK_ENCCL", -8: "LSK_ENOMEM", -9: "LSK_EUNSUPPORTED"}


class LskError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.lsk_last_error().decode(errors="replace")
        super().__init__("%s: %s (%s)" % (where, STATUS_NAMES.get(status, status), msg))


def _check(status: int, where: str) -> int:
    if status < 0:
        raise LskError(status, where)
    return status


def version() -> str:
    return _lib.lsk_version().decode()


def lsk_stream_status(stream=None) -> int:
    """Synchronise the stream and raise the sticky error (LSK_EBREAKDOWN / LSK_EWEIGHTS /
    LSK_ENCCL) of a report-less solve enqueued on it; clears it (include/lsk.h Conventions)."""
    return _check(_lib.lsk_stream_status(_stream(stream)), "lsk_stream_status")


def lsk_resident_plan(n: int, m: int, r: int) -> int:
    """Cluster CTAs of the resident small-problem kernel for this shape, 0 = grid kernels
    (diagnostic; include/lsk.h)."""
    g = c_i32()
    _check(_lib.lsk_resident_plan(int(n), int(m), int(r), ctypes.byref(g)), "lsk_resident_plan")
    return g.value


def lsk_solve_plan(n: int, m: int, r: int, d: int, batch: int = 1, variant: str = "stream",
                   cluster: bool = False):
    """(gpp, grid) — and with cluster=True (gpp, grid, cluster) — of the launch a solve of this
    shape uses (diagnostic; include/lsk.h)."""
    g, gr, cx = c_i32(), c_i32(), c_i32()
    _check(_lib.lsk_solve_plan(int(n), int(m), int(r), int(d), int(batch),
                               1 if variant == "stream" else 2, ctypes.byref(g), ctypes.byref(gr),
                               ctypes.byref(cx)), "lsk_solve_plan")
    return (g.value, gr.value, cx.value) if cluster else (g.value, gr.value)


def lsk_stream_rows(n: int, m: int, r: int, d: int, opts: lsk_solve_opts = None):
    """(ns0, ns1): rows of X and Y the implicit solver streams from HBM (hybrid kernel)."""
    a, b = c_i64(), c_i64()
    _check(_lib.lsk_stream_rows(int(n), int(m), int(r), int(d),
                                ctypes.byref(opts) if opts is not None else None,
                                ctypes.byref(a), ctypes.byref(b)), "lsk_stream_rows")
    return a.value, b.value


def launch_count(reset: bool = False) -> int:
    return int(_lib.lsk_launch_count(1 if reset else 0))


# ---------------------------------------------------------------- marshalling helpers ----
def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _f32(t):
    import torch
    if t.dtype != torch.float32:
        raise ValueError("expected float32, got %s" % t.dtype)
    return _ptr(t)


def _stream(stream=None) -> int:
    import torch
    if stream is None:
        if not torch.cuda.is_available():
            return None          # host-only entry points (validation, a1 with R given)
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


LSK_SOLVE_STABILIZE = 1
LSK_SOLVE_NO_RESIDENT = 2


def make_opts(iters: int, tol: float = 0.0, want_err: bool = False,
              ctas_per_sm: int = 0, stabilize: bool = False,
              stream_fraction: float = 0.0, resident: bool = True) -> lsk_solve_opts:
    """stream_fraction (implicit solver): 0 = library default, < 0 = pure recompute,
    (0, 0.9] = that fraction of rows streamed from HBM (include/lsk.h).  resident=False:
    never the resident small-problem kernel (LSK_SOLVE_NO_RESIDENT)."""
    flags = (LSK_SOLVE_STABILIZE if stabilize else 0) | (0 if resident else LSK_SOLVE_NO_RESIDENT)
    return lsk_solve_opts(int(iters), 1 if want_err else 0, float(tol), int(ctas_per_sm),
                          flags, float(stream_fraction))


# ---------------------------------------------------------------- C-ABI mirrors ----------
def lsk_lambert_w0(z: float) -> float:
    w = ctypes.c_double()
    _check(_lib.lsk_lambert_w0(float(z), ctypes.byref(w)), "lsk_lambert_w0")
    return w.value


def lsk_shard_range(total: int, nranks: int, rank: int):
    b, e = c_i64(), c_i64()
    _check(_lib.lsk_shard_range(total, nranks, rank, ctypes.byref(b), ctypes.byref(e)),
           "lsk_shard_range")
    return b.value, e.value


def lsk_feature_params_init(eps, d, r, R=0.0, seed=0, X=None, Y=None, comm=None,
                            stream=None) -> lsk_feature_params:
    p = lsk_feature_params()
    n = 0 if X is None else X.shape[0]
    m = 0 if Y is None else Y.shape[0]
    _check(_lib.lsk_feature_params_init(float(eps), int(d), int(r), float(R), int(seed),
                                        _f32(X) if X is not None else None, n,
                                        _f32(Y) if Y is not None else None, m,
                                        ctypes.byref(p), comm, _stream(stream)),
           "lsk_feature_params_init")
    return p


def lsk_draw_anchors(p: lsk_feature_params, U, stream=None):
    _check(_lib.lsk_draw_anchors(ctypes.byref(p), _f32(U), _stream(stream)), "lsk_draw_anchors")
    return U


def lsk_philox_words(seed: int, r: int, d: int, out, stream=None):
    _check(_lib.lsk_philox_words(int(seed), int(r), int(d), _ptr(out), _stream(stream)),
           "lsk_philox_words")
    return out


def lsk_feature_map(p: lsk_feature_params, U, X, Xi, stream=None):
    _check(_lib.lsk_feature_map(ctypes.byref(p), _f32(U), _f32(X), X.shape[0], _f32(Xi),
                                _stream(stream)), "lsk_feature_map")
    return Xi


def lsk_feature_map_arccos(p, s_degree, kappa, U, X, Xi, stream=None):
    """Arc-cosine features into Xi (n x (r+4)); see include/lsk.h."""
    _check(_lib.lsk_feature_map_arccos(ctypes.byref(p), int(s_degree), float(kappa), _f32(U),
                                       _f32(X), X.shape[0], _f32(Xi), _stream(stream)),
           "lsk_feature_map_arccos")
    return Xi


def arccos_params(d, r, sigma, seed, eps):
    """lsk_feature_params for the arc-cosine map: only d, r, sigma, seed (anchors) and eps
    (the Sinkhorn temperature) are used."""
    return lsk_feature_params(float(eps), 0.0, 0.0, float(sigma), 0.0, int(d), int(r), int(seed))


def lsk_feature_map_batched(p: lsk_feature_params, U, X, Xi, stream=None):
    B, n = X.shape[0], X.shape[1]
    _check(_lib.lsk_feature_map_batched(ctypes.byref(p), _f32(U), _f32(X), n, B, _f32(Xi),
                                        _stream(stream)), "lsk_feature_map_batched")
    return Xi


def lsk_factored_sinkhorn(Xi, Zeta, a, b, eps, opts: lsk_solve_opts, u, v, report=True,
                          comm=None, stream=None):
    rep = lsk_report() if report else None
    st = _lib.lsk_factored_sinkhorn(_f32(Xi), Xi.shape[0], _f32(Zeta), Zeta.shape[0],
                                    Xi.shape[1], _f32(a), _f32(b), float(eps),
                                    ctypes.byref(opts), _f32(u), _f32(v),
                                    ctypes.byref(rep) if rep is not None else None, comm,
                                    _stream(stream))
    _check(st, "lsk_factored_sinkhorn")
    return rep


def lsk_factored_sinkhorn_implicit(p: lsk_feature_params, U, X, Y, a, b, opts, u, v,
                                   report=True, comm=None, stream=None):
    rep = lsk_report() if report else None
    st = _lib.lsk_factored_sinkhorn_implicit(ctypes.byref(p), _f32(U), _f32(X), X.shape[0],
                                             _f32(Y), Y.shape[0], _f32(a), _f32(b),
                                             ctypes.byref(opts), _f32(u), _f32(v),
                                             ctypes.byref(rep) if rep is not None else None,
                                             comm, _stream(stream))
    _check(st, "lsk_factored_sinkhorn_implicit")
    return rep


def lsk_factored_sinkhorn_batched(Xi, Zeta, a, b, eps, opts, u, v, report=True, stream=None):
    B, n, r = Xi.shape
    m = Zeta.shape[1]
    reps = (lsk_report * B)() if report else None
    st = _lib.lsk_factored_sinkhorn_batched(_f32(Xi), n, _f32(Zeta), m, r, B, _f32(a),
                                            _f32(b), float(eps), ctypes.byref(opts), _f32(u),
                                            _f32(v), reps, _stream(stream))
    _check(st, "lsk_factored_sinkhorn_batched")
    return list(reps) if reps is not None else None


def lsk_factored_sinkhorn_implicit_batched(p, U, X, Y, a, b, opts, u, v, report=True,
                                           stream=None):
    """X (B, n, d), Y (B, m, d), a/u (B, n), b/v (B, m): B independent recompute solves."""
    B = X.shape[0]
    reps = (lsk_report * B)() if report else None
    _check(_lib.lsk_factored_sinkhorn_implicit_batched(
        ctypes.byref(p), _f32(U), _f32(X), X.shape[1], _f32(Y), Y.shape[1], B, _f32(a), _f32(b),
        ctypes.byref(opts), _f32(u), _f32(v), reps, _stream(stream)),
        "lsk_factored_sinkhorn_implicit_batched")
    return list(reps) if report else None


def lsk_factored_sinkhorn_emulated(nranks, Xi, Zeta, a, b, eps, opts, u, v, report=True,
                                   stream=None):
    """N emulated ranks of one row-sharded streaming solve in one cooperative launch (the
    in-kernel cross-GPU exchange on one GPU; include/lsk.h).  Returns the N reports."""
    reps = (lsk_report * nranks)() if report else None
    _check(_lib.lsk_factored_sinkhorn_emulated(int(nranks), _f32(Xi), Xi.shape[0], _f32(Zeta),
                                               Zeta.shape[0], Xi.shape[1], _f32(a), _f32(b),
                                               float(eps), ctypes.byref(opts), _f32(u), _f32(v),
                                               reps, _stream(stream)),
           "lsk_factored_sinkhorn_emulated")
    return list(reps) if report else None


def lsk_factored_sinkhorn_implicit_emulated(nranks, p, U, X, Y, a, b, opts, u, v, report=True,
                                            stream=None):
    reps = (lsk_report * nranks)() if report else None
    _check(_lib.lsk_factored_sinkhorn_implicit_emulated(
        int(nranks), ctypes.byref(p), _f32(U), _f32(X), X.shape[0], _f32(Y), Y.shape[0], _f32(a),
        _f32(b), ctypes.byref(opts), _f32(u), _f32(v), reps, _stream(stream)),
        "lsk_factored_sinkhorn_implicit_emulated")
    return list(reps) if report else None


def lsk_rot_value(u, v, a, b, eps, comm=None, stream=None) -> float:
    out = ctypes.c_double()
    _check(_lib.lsk_rot_value(_f32(u), _f32(v), _f32(a), _f32(b), u.shape[0], v.shape[0],
                              float(eps), ctypes.byref(out), comm, _stream(stream)),
           "lsk_rot_value")
    return out.value


def lsk_rot_value_batched(u, v, a, b, eps, stream=None):
    B, n = u.shape
    m = v.shape[1]
    out = (ctypes.c_double * B)()
    _check(_lib.lsk_rot_value_batched(_f32(u), _f32(v), _f32(a), _f32(b), n, m, B, float(eps),
                                      out, _stream(stream)), "lsk_rot_value_batched")
    return list(out)


def _div_result(out, reps):
    return dict(div=out[0], xy=out[1], xx=out[2], yy=out[3],
                reports=[rp.as_dict() for rp in reps])


def lsk_sinkhorn_divergence(Xi, Zeta, a, b, eps, opts, stream=None):
    """W_bar(mu,nu) = W(mu,nu) - (W(mu,mu) + W(nu,nu))/2 on device factors."""
    out = (ctypes.c_double * 4)()
    reps = (lsk_report * 3)()
    _check(_lib.lsk_sinkhorn_divergence(_f32(Xi), Xi.shape[0], _f32(Zeta), Zeta.shape[0],
                                        Xi.shape[1], _f32(a), _f32(b), float(eps),
                                        ctypes.byref(opts), out, reps, _stream(stream)),
           "lsk_sinkhorn_divergence")
    return _div_result(out, reps)


def lsk_sinkhorn_divergence_implicit(p, U, X, Y, a, b, opts, stream=None):
    out = (ctypes.c_double * 4)()
    reps = (lsk_report * 3)()
    _check(_lib.lsk_sinkhorn_divergence_implicit(ctypes.byref(p), _f32(U), _f32(X), X.shape[0],
                                                 _f32(Y), Y.shape[0], _f32(a), _f32(b),
                                                 ctypes.byref(opts), out, reps,
                                                 _stream(stream)),
           "lsk_sinkhorn_divergence_implicit")
    return _div_result(out, reps)


def lsk_feature_map_stabilized(p, U, X, Xi, logoff, stream=None):
    """Row-normalised features Xi (n, r) and fp64 row log-offsets logoff (n) (reading C30)."""
    _check(_lib.lsk_feature_map_stabilized(ctypes.byref(p), _f32(U), _f32(X), X.shape[0],
                                           _f32(Xi), _ptr(logoff), _stream(stream)),
           "lsk_feature_map_stabilized")


def lsk_implicit_row_offsets(p, U, X, logoff, stream=None):
    """fp64 row offsets A (n) of the stabilised implicit solver: u = u~ e^{-A}."""
    _check(_lib.lsk_implicit_row_offsets(ctypes.byref(p), _f32(U), _f32(X), X.shape[0],
                                         _ptr(logoff), _stream(stream)), "lsk_implicit_row_offsets")


def lsk_rot_value_offset(u, v, a, b, A, B, eps, stream=None) -> float:
    out = ctypes.c_double()
    _check(_lib.lsk_rot_value_offset(_f32(u), _f32(v), _f32(a), _f32(b), _ptr(A), _ptr(B),
                                     u.shape[0], v.shape[0], float(eps), ctypes.byref(out),
                                     _stream(stream)), "lsk_rot_value_offset")
    return out.value


def lsk_accelerated_sinkhorn(Xi, Zeta, a, b, eps, max_iters, tol=0.0, L0=1.0, eta1=None,
                             eta2=None, traces=False, stream=None):
    """Alg. 2 on device factors Xi (n, r), Zeta (m, r).  Returns a dict with
    the report fields, the fp64 dual point eta1 (n), eta2 (m) and, with traces=True, the
    per-iteration F, accepted L and block."""
    import torch
    import numpy as np
    n, m = Xi.shape[0], Zeta.shape[0]
    if eta1 is None:
        eta1 = torch.empty(n, dtype=torch.float64, device=Xi.device)
    if eta2 is None:
        eta2 = torch.empty(m, dtype=torch.float64, device=Xi.device)
    o = lsk_accel_opts(int(max_iters), 0, float(tol), float(L0))
    rep = lsk_accel_report()
    tr = None
    if traces:
        tr = (np.zeros(max_iters), np.zeros(max_iters), np.zeros(max_iters, np.int32))
    ptr = (lambda x: x.ctypes.data) if traces else (lambda x: None)
    st = _lib.lsk_accelerated_sinkhorn(_f32(Xi), n, _f32(Zeta), m, Xi.shape[1], _f32(a),
                                       _f32(b), float(eps), ctypes.byref(o), _ptr(eta1),
                                       _ptr(eta2), ptr(tr[0]) if tr else None,
                                       ptr(tr[1]) if tr else None, ptr(tr[2]) if tr else None,
                                       ctypes.byref(rep), _stream(stream))
    _check(st, "lsk_accelerated_sinkhorn")
    out = rep.as_dict()
    out.update(eta1=eta1, eta2=eta2, status=st)
    if traces:
        k = rep.iters
        out.update(F_trace=tr[0][:k], L_trace=tr[1][:k], blocks=tr[2][:k])
    return out


def sinkhorn_divergence(X, Y, a, b, eps, r, seed, iters=None, tol=0.0, R=0.0,
                        variant="stream", max_iters=None, stream=None):
    """Whole divergence path on device tensors: shared params/anchors, features, 3 solves."""
    import torch
    d = X.shape[1]
    p = lsk_feature_params_init(eps, d, r, R, seed, X, Y, stream=stream)
    U = torch.empty((r, d), dtype=torch.float32, device=X.device)
    lsk_draw_anchors(p, U, stream)
    opts = make_opts(iters if iters is not None else (max_iters or 1000), tol)
    if variant == "implicit":
        return lsk_sinkhorn_divergence_implicit(p, U, X, Y, a, b, opts, stream)
    Xi = torch.empty((X.shape[0], r), dtype=torch.float32, device=X.device)
    Ze = torch.empty((Y.shape[0], r), dtype=torch.float32, device=X.device)
    lsk_feature_map(p, U, X, Xi, stream)
    lsk_feature_map(p, U, Y, Ze, stream)
    return lsk_sinkhorn_divergence(Xi, Ze, a, b, eps, opts, stream)


def lsk_rot_gradient(p, U, X, Y, Xi, Zeta, u, v, want=("X", "Y", "U"), stream=None):
    """Envelope gradients dW/dX, dW/dY, dW/dU at the scalings (u, v)."""
    import torch
    d, r = X.shape[1], U.shape[0]
    out = {k: torch.empty(shp, dtype=torch.float32, device=X.device)
           for k, shp in (("X", (X.shape[0], d)), ("Y", (Y.shape[0], d)), ("U", (r, d)))
           if k in want}
    _check(_lib.lsk_rot_gradient(ctypes.byref(p), _f32(U), _f32(X), X.shape[0], _f32(Y),
                                 Y.shape[0], _f32(Xi), _f32(Zeta), _f32(u), _f32(v),
                                 _f32(out["X"]) if "X" in out else None,
                                 _f32(out["Y"]) if "Y" in out else None,
                                 _f32(out["U"]) if "U" in out else None, _stream(stream)),
           "lsk_rot_gradient")
    return out


def lsk_rot_host(X, Y, a, b, eps, r, seed, opts, R=0.0, variant=0, u_out=None, v_out=None):
    """Host-buffer end-to-end call.  X, Y, a, b, u_out, v_out: CPU float32 tensors (pinned
    for async copies) or numpy float32 arrays."""
    def hp(t):
        if t is None:
            return None
        if hasattr(t, "data_ptr"):
            if t.is_cuda:
                raise ValueError("lsk_rot_host expects host tensors")
            return t.data_ptr()
        return t.ctypes.data
    rep = lsk_report()
    st = _lib.lsk_rot_host(hp(X), X.shape[0], hp(Y), Y.shape[0], X.shape[1], hp(a), hp(b),
                           float(eps), int(r), int(seed), float(R), ctypes.byref(opts),
                           int(variant), hp(u_out), hp(v_out), ctypes.byref(rep))
    _check(st, "lsk_rot_host")
    return rep


def lsk_comm_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.lsk_comm_get_unique_id(buf), "lsk_comm_get_unique_id")
    return buf.raw


def lsk_comm_init(nranks: int, rank: int, unique_id: bytes, device: int):
    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(_lib.lsk_comm_init(ctypes.byref(h), nranks, rank, buf, device), "lsk_comm_init")
    return h


def lsk_comm_destroy(comm):
    _check(_lib.lsk_comm_destroy(comm), "lsk_comm_destroy")


def lsk_comm_enable_p2p(comm, r_max: int, stream=None):
    """Collective: map every rank's inbox over NVLink so that solves on `comm` run as one
    persistent launch per GPU with the cross-GPU r-vector sum inside the kernel."""
    _check(_lib.lsk_comm_enable_p2p(comm, int(r_max), _stream(stream)), "lsk_comm_enable_p2p")


# ---------------------------------------------------------------- convenience -----------
def rot(X, Y, a, b, eps, r, seed, iters=None, tol=0.0, R=0.0, variant="stream",
        want_err=False, max_iters=None, ctas_per_sm=0, comm=None, stream=None, stabilize=False,
        stream_fraction=0.0, resident=True):
    """Whole hot path on device tensors: a1 params -> a2 anchors -> a3 features -> Alg. 1 ->
    a9 read-out.  variant: "stream" (materialise xi, zeta) or "implicit" (recompute).
    stabilize=True: row-normalised features with log offsets (reading C30; stream: d <= 16,
    implicit: d <= 8); u, v are then the scalings of the normalised problem and A, B the
    offsets."""
    import torch
    dev = X.device
    d = X.shape[1]
    n, m = X.shape[0], Y.shape[0]
    p = lsk_feature_params_init(eps, d, r, R, seed, X, Y, comm=comm, stream=stream)
    U = torch.empty((r, d), dtype=torch.float32, device=dev)
    lsk_draw_anchors(p, U, stream)
    u = torch.empty(n, dtype=torch.float32, device=dev)
    v = torch.empty(m, dtype=torch.float32, device=dev)
    T = iters if iters is not None else (max_iters or 1000)
    opts = make_opts(T, tol, want_err, ctas_per_sm, stabilize=stabilize and variant == "implicit",
                     stream_fraction=stream_fraction, resident=resident)
    out = dict(params=p.as_dict(), U=U, u=u, v=v)
    if variant == "implicit":
        rep = lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, comm=comm,
                                             stream=stream)
        if stabilize:
            A = torch.empty(n, dtype=torch.float64, device=dev)
            B = torch.empty(m, dtype=torch.float64, device=dev)
            lsk_implicit_row_offsets(p, U, X, A, stream)
            lsk_implicit_row_offsets(p, U, Y, B, stream)
            out.update(A=A, B=B)
    else:
        Xi = torch.empty((n, r), dtype=torch.float32, device=dev)
        Zeta = torch.empty((m, r), dtype=torch.float32, device=dev)
        if stabilize:
            A = torch.empty(n, dtype=torch.float64, device=dev)
            B = torch.empty(m, dtype=torch.float64, device=dev)
            lsk_feature_map_stabilized(p, U, X, Xi, A, stream)
            lsk_feature_map_stabilized(p, U, Y, Zeta, B, stream)
            out.update(A=A, B=B)
        else:
            lsk_feature_map(p, U, X, Xi, stream)
            lsk_feature_map(p, U, Y, Zeta, stream)
        rep = lsk_factored_sinkhorn(Xi, Zeta, a, b, eps, opts, u, v, comm=comm, stream=stream)
        out.update(Xi=Xi, Zeta=Zeta)
    out.update(report=rep.as_dict(), rot=rep.rot)
    if variant != "implicit" and stabilize:
        out["rot"] = lsk_rot_value_offset(u, v, a, b, out["A"], out["B"], eps, stream)
    return out
