"""ORACLE — plain, slow, fp64 CPU reference of the factored-Sinkhorn hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` leg may import this module.  The product package
(``paper_2006_07057_b200``) never imports it and shares no code, header, table or constant
generator with it; the only shared module is ``synth`` (seeded inputs, no method arithmetic).

Every function follows the paper's order and notation (PAPER.md = arXiv 2006.07057 LaTeX in
/root/reference; line numbers cite the full-paper fragment).  Layout
follows the paper: feature matrices are r x n, xi = [phi_theta(x_1), ..., phi_theta(x_n)]
(PAPER.md:278), so K_theta = xi^T zeta.  Arithmetic is fp64 throughout; fp32
inputs are promoted.  Library primitives used as single steps: numpy matmul / exp / log,
numpy's Philox-free integer ops.  No blocking, fusion or reordering.

Readings of silent/garbled passages are the C-numbered items of DESIGN.md §Readings.

Pins (tests/test_oracle_*.py) — every function below is pinned to something outside itself:
  lambert_w0            scipy.special.lambertw, W(1)=Omega constant, residual  (P1)
  gaussian_params       q = e^{W0(z)}/2 identity, q W0 2 eps d = R^2            (P2)
  gaussian_phi          phi(0,0)=(2q)^{d/4}; Gauss-Hermite kernel identity;     (P3,P4,P6)
                        ratio bound 2(2q)^{d/2}
  philox4x32_10         Random123 known-answer vectors (tests/golden/philox_kat.txt)
  standard_normals      moment test + Box-Muller closed form on known words
  feature_matrix        == gaussian_phi per entry; Monte-Carlo rate slope -1/2   (P5,P7)
  sinkhorn_*            dense == factored (P8), n=m=1 (P9), 2x2 closed form (P10),
                        rank-1 closed form (P11), marginals (P12), convergence (P13),
                        primal == dual (P14), gauge invariance (P15), dual range (P17)
  dual_estimate         P9/P10/P11/P14
  accelerated_sinkhorn  (NEXT f4, Alg. 2) == Alg. 1's converged W_hat on random factored
                        instances (independent algorithm, unique dual optimum); 2x2 and
                        rank-one closed forms; weak duality at every iterate; accepted
                        L <= 4 (phi is 2-smooth); plan marginals -> (a, b), unit mass
                        (tests/test_oracle_accel.py)
  max_norm              hand-computed norms of Pythagorean triples, max in X or in Y
  marginal_error        a 2x2 case worked by hand (tests/test_oracle_sinkhorn.py)
  C29 allowance         without it the accepted L leaves the smoothness bound 4 in the
                        rounding regime; with it L <= 4 (tests/test_oracle_accel.py)
  matrix_free.py + lsk_oracle_mf.c (config 5's full-size oracle) == the materialised numpy
                        oracle; rank-one closed form at n = 2e5; P9 (test_oracle_matrix_free.py)
  exact gaussian ROT    paper RE behaviour on the Fig. 1 setup (P16, qualitative: the
                        paper prints no numbers — "parity unpinned" for the RE values
                        themselves; only the sign/monotonic trends are asserted)
"""
from __future__ import annotations

import math
from typing import Callable, Optional

import numpy as np

LOG2E = 1.0 / math.log(2.0)


# ---------------------------------------------------------------------------------------
# a1. Feature parameters: Lambert W_0, q, sigma (Lemma decomp-RBF)
# ---------------------------------------------------------------------------------------
def lambert_w0(z: float, tol: float = 1e-15, max_iter: int = 100) -> float:
    """Principal branch W_0(z): the w >= -1 with w e^w = z ("W_0 is the Lambert
    function"; positive real branch).  Halley iteration from log(1+z) for
    z >= 0 (the only domain the feature map uses; z = R^2/(eps d) > 0)."""
    if z < -1.0 / math.e:
        raise ValueError("lambert_w0: z < -1/e")
    if z == 0.0:
        return 0.0
    w = math.log1p(z) if z > 0 else -0.5
    for _ in range(max_iter):
        ew = math.exp(w)
        f = w * ew - z
        wp1 = w + 1.0
        denom = ew * wp1 - (w + 2.0) * f / (2.0 * wp1)
        step = f / denom
        w -= step
        if abs(step) <= tol * (1.0 + abs(w)):
            break
    return w


def max_norm(X: np.ndarray, Y: np.ndarray) -> float:
    """R = max over both clouds of the Euclidean norm (reading C3), fp64 from fp32 inputs."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    return float(max(np.sqrt((X * X).sum(axis=1)).max(), np.sqrt((Y * Y).sum(axis=1)).max()))


def gaussian_params(eps: float, d: int, r: int, R: float) -> dict:
    """q = R^2 / (2 eps d W_0(R^2/(eps d)));  sigma^2 = q eps / 4
    (rho_q = N(0, q/(4 eps^-1) Id));
    log_scale = (d/4) ln(2q) - (1/2) ln r  collects the (2q)^{d/4} factor of phi
     and the 1/sqrt(r) of phi_theta."""
    z = R * R / (eps * d)
    W = lambert_w0(z)
    q = z / (2.0 * W)
    sigma = math.sqrt(q * eps / 4.0)
    log_scale = 0.25 * d * math.log(2.0 * q) - 0.5 * math.log(r)
    return dict(z=z, W=W, q=q, sigma=sigma, log_scale=log_scale, R=R, eps=eps, d=d, r=r)


# ---------------------------------------------------------------------------------------
# a2. Anchors u_1..u_r ~ rho = N(0, sigma^2 Id), i.i.d.
#     Reading C5: counter-based Philox4x32-10 + fp64 Box-Muller, rounded to fp32.
# ---------------------------------------------------------------------------------------
_PHILOX_M0 = np.uint64(0xD2511F53)
_PHILOX_M1 = np.uint64(0xCD9E8D57)
_PHILOX_W0 = 0x9E3779B9
_PHILOX_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key) -> np.ndarray:
    """Philox4x32 with 10 rounds (Salmon, Moraes, Dror, Shaw, SC'11).  ``ctr`` is (N,4)
    uint32, ``key`` is (k0,k1).  One round: (hi0,lo0)=M0*c0, (hi1,lo1)=M1*c2,
    c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0); between rounds k <- k + (W0,W1) mod 2^32."""
    c = np.asarray(ctr, dtype=np.uint64).reshape(-1, 4).copy()
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + _PHILOX_W0) & 0xFFFFFFFF
            k1 = (k1 + _PHILOX_W1) & 0xFFFFFFFF
        p0 = _PHILOX_M0 * c[:, 0]
        p1 = _PHILOX_M1 * c[:, 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        n0 = hi1 ^ c[:, 1] ^ np.uint64(k0)
        n2 = hi0 ^ c[:, 3] ^ np.uint64(k1)
        c = np.stack([n0, lo1, n2, lo0], axis=1)
    return c.astype(np.uint32)


def philox_words(r: int, d: int, seed: int) -> np.ndarray:
    """Raw words for anchors: counter (k, p, 0, 0) for anchor k and coordinate block
    p = 0..ceil(d/4)-1, key = (seed mod 2^32, seed >> 32).  Returns (r, P, 4) uint32."""
    P = (d + 3) // 4
    kk, pp = np.meshgrid(np.arange(r, dtype=np.uint64), np.arange(P, dtype=np.uint64),
                         indexing="ij")
    ctr = np.stack([kk.ravel(), pp.ravel(), np.zeros(r * P, np.uint64),
                    np.zeros(r * P, np.uint64)], axis=1)
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return philox4x32_10(ctr, key).reshape(r, P, 4)


def standard_normals(r: int, d: int, seed: int) -> np.ndarray:
    """Box-Muller in fp64 on each word pair: u1 = (w0+1) 2^-32 in (0,1], u2 = w1 2^-32,
    z = sqrt(-2 ln u1) (cos 2 pi u2, sin 2 pi u2); the same for (w2, w3).  Coordinates
    4p..4p+3 of anchor k come from block p.  Returns (r, d) fp64."""
    w = philox_words(r, d, seed).astype(np.float64)
    u1a = (w[..., 0] + 1.0) * 2.0 ** -32
    u2a = w[..., 1] * 2.0 ** -32
    u1b = (w[..., 2] + 1.0) * 2.0 ** -32
    u2b = w[..., 3] * 2.0 ** -32
    ra = np.sqrt(-2.0 * np.log(u1a))
    rb = np.sqrt(-2.0 * np.log(u1b))
    z = np.stack([ra * np.cos(2.0 * np.pi * u2a), ra * np.sin(2.0 * np.pi * u2a),
                  rb * np.cos(2.0 * np.pi * u2b), rb * np.sin(2.0 * np.pi * u2b)], axis=-1)
    return z.reshape(r, -1)[:, :d]


def draw_anchors(r: int, d: int, sigma: float, seed: int) -> np.ndarray:
    """theta = (u_1..u_r), u_k ~ N(0, sigma^2 Id) i.i.d.; values are
    rounded to fp32 (the stored precision) and returned promoted to fp64, shape (r, d)."""
    return (sigma * standard_normals(r, d, seed)).astype(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------------------
# a3. Gaussian positive feature map (Lemma decomp-RBF, appendix form PAPER.md:915, 934;
#     reading C1: the main-text exponent at PAPER.md:389 is garbled)
# ---------------------------------------------------------------------------------------
def gaussian_phi(x: np.ndarray, u: np.ndarray, eps: float, q: float) -> np.ndarray:
    """phi(x,u) = (2q)^{d/4} exp(-2 eps^-1 |x-u|^2) exp(eps^-1 |u|^2 / q).
    Broadcasts over leading axes of x and u (last axis = coordinates)."""
    x = np.asarray(x, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    d = x.shape[-1]
    sq = ((x - u) ** 2).sum(axis=-1)
    uu = (u * u).sum(axis=-1)
    return (2.0 * q) ** (d / 4.0) * np.exp(-2.0 / eps * sq) * np.exp(uu / (eps * q))


def feature_matrix(X: np.ndarray, U: np.ndarray, eps: float, q: float) -> np.ndarray:
    """xi = [phi_theta(x_1), ..., phi_theta(x_n)] in R_+^{r x n} with
    phi_theta(x) = r^{-1/2} (phi(x,u_1), ..., phi(x,u_r)).  Direct
    difference form, fp64: xi[k,i] = exp(-(2/eps) sum_c (x_ic-u_kc)^2 + |u_k|^2/(eps q)
    + (d/4) ln 2q - (1/2) ln r)."""
    X = np.asarray(X, dtype=np.float64)
    U = np.asarray(U, dtype=np.float64)
    r, d = U.shape
    sq = np.zeros((r, X.shape[0]))
    for c in range(d):
        sq += (U[:, c][:, None] - X[:, c][None, :]) ** 2
    uu = (U * U).sum(axis=1)
    log_scale = 0.25 * d * math.log(2.0 * q) - 0.5 * math.log(r)
    return np.exp(-2.0 / eps * sq + (uu / (eps * q))[:, None] + log_scale)


def feature_entries_scaled(X: np.ndarray, U: np.ndarray, eps: float, q: float, r: int,
                           rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """phi(x_i, u_k)/sqrt(r) for each sampled pair (rows[j], cols[j])."""
    x = np.asarray(X, dtype=np.float64)[rows]
    u = np.asarray(U, dtype=np.float64)[cols]
    return gaussian_phi(x, u, eps, q) / math.sqrt(r)


# ---------------------------------------------------------------------------------------
# Alg. 1 Sinkhorn on a generic positive operator K
# ---------------------------------------------------------------------------------------
def sinkhorn(K_mv: Callable[[np.ndarray], np.ndarray],
             Kt_mv: Callable[[np.ndarray], np.ndarray],
             a: np.ndarray, b: np.ndarray, T: Optional[int] = None,
             tol: Optional[float] = None, max_iter: int = 100000,
             record_err: bool = False, u0: Optional[np.ndarray] = None) -> dict:
    """Alg. 1: inputs K, a, b, delta, u.  u^0 = 1_n (reading C6).  Repeat
    v <- b / K^T u ; u <- a / K v  until |v o K^T u - b|_1 < delta.

    Fixed-T mode (tol None): exactly T iterations.  Tolerance mode: stop after the first
    iteration t whose err_t = |v^t o K^T u^t - b|_1 < tol (checked every iteration).
    Returns u, v, iters, errs (err_t per iteration when recorded), converged."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    u = np.ones(a.shape[0]) if u0 is None else np.asarray(u0, dtype=np.float64)
    v = np.ones(b.shape[0])
    errs = []
    iters = 0
    converged = False
    n_iter = T if tol is None else max_iter
    for _ in range(n_iter):
        v = b / Kt_mv(u)
        u = a / K_mv(v)
        iters += 1
        if tol is not None or record_err:
            err = float(np.abs(v * Kt_mv(u) - b).sum())
            errs.append(err)
            if tol is not None and err < tol:
                converged = True
                break
    return dict(u=u, v=v, iters=iters, errs=np.array(errs), converged=converged)


def sinkhorn_factored(xi: np.ndarray, zeta: np.ndarray, a, b, T=None, tol=None,
                      record_err=False, max_iter=100000, u0=None) -> dict:
    """Alg. 1 with K_theta = xi^T zeta: K v = xi^T (zeta v),
    K^T u = zeta^T (xi u) — r(n+m) operations per application.
    xi is r x n, zeta is r x m (paper layout)."""
    xi = np.asarray(xi, dtype=np.float64)
    zeta = np.asarray(zeta, dtype=np.float64)
    return sinkhorn(lambda v: xi.T @ (zeta @ v), lambda u: zeta.T @ (xi @ u), a, b, T, tol,
                    max_iter, record_err, u0)


def sinkhorn_dense(K: np.ndarray, a, b, T=None, tol=None, record_err=False,
                   max_iter=100000) -> dict:
    """Alg. 1 on an explicitly stored n x m kernel (2nm operations)."""
    K = np.asarray(K, dtype=np.float64)
    return sinkhorn(lambda v: K @ v, lambda u: K.T @ u, a, b, T, tol, max_iter, record_err)


# ---------------------------------------------------------------------------------------
# a9. Dual estimate and primal objective
# ---------------------------------------------------------------------------------------
def dual_estimate(u, v, a, b, eps: float) -> float:
    """W_hat = eps (a^T log u + b^T log v)  (eq. dual-estimate).  No separate
    +eps: the -eps u^T K v + eps pair cancels because u^T K v = 1 after one loop
    (reading C7)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(eps * (a @ np.log(u) + b @ np.log(v)))


def primal_objective(P: np.ndarray, C: np.ndarray, eps: float) -> float:
    """<P, C> - eps H(P) + eps with H(P) = -sum P (log P - 1)."""
    H = -float((P * (np.log(P) - 1.0)).sum())
    return float((P * C).sum()) - eps * H + eps


def gaussian_kernel_dense(X, Y, eps: float) -> np.ndarray:
    """k(x,y) = exp(-|x-y|^2 / eps)  (Lemma decomp-RBF statement)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    sq = (X * X).sum(1)[:, None] + (Y * Y).sum(1)[None, :] - 2.0 * X @ Y.T
    sq = np.maximum(sq, 0.0)
    return np.exp(-sq / eps)


def marginal_error(u, v, Kt_u, b) -> float:
    """|v o K^T u - b|_1 (stopping criterion of Alg. 1)."""
    return float(np.abs(v * Kt_u - np.asarray(b, dtype=np.float64)).sum())


# ---------------------------------------------------------------------------------------
# The whole hot path, in paper order: a1 -> a2 -> a3 -> Alg. 1 -> a9
# ---------------------------------------------------------------------------------------
def rot(X, Y, a, b, eps: float, r: int, seed: int, T: Optional[int] = None,
        tol: Optional[float] = None, R: Optional[float] = None, record_err=False,
        U: Optional[np.ndarray] = None) -> dict:
    """W_hat_{eps,c_theta}(mu, nu) for mu = sum a_i delta_{x_i}, nu = sum b_j delta_{y_j}
    (problem statement PAPER.md:220-222), computed by Alg. 1 on K_theta = xi^T zeta."""
    d = np.asarray(X).shape[1]
    if R is None:
        R = max_norm(X, Y)
    prm = gaussian_params(eps, d, r, R)
    if U is None:
        U = draw_anchors(r, d, prm["sigma"], seed)
    xi = feature_matrix(X, U, eps, prm["q"])
    zeta = feature_matrix(Y, U, eps, prm["q"])
    sol = sinkhorn_factored(xi, zeta, a, b, T=T, tol=tol, record_err=record_err)
    sol.update(rot=dual_estimate(sol["u"], sol["v"], a, b, eps), U=U, xi=xi, zeta=zeta,
               params=prm)
    return sol


# ---------------------------------------------------------------------------------------
# NEXT row f1: Sinkhorn divergence (eq. reg-sdiv)
# ---------------------------------------------------------------------------------------
def sinkhorn_divergence(X, Y, a, b, eps: float, r: int, seed: int, T: Optional[int] = None,
                        tol: Optional[float] = None, R: Optional[float] = None) -> dict:
    """W_bar(mu,nu) = W(mu,nu) - (W(mu,mu) + W(nu,nu)) / 2, each W the dual
    estimate of Alg. 1 on K_theta with ONE anchor draw theta shared by the three problems
    (c_theta is a single cost, eq. cost).  R defaults to the max norm over both
    clouds, so the three solves use the same (q, sigma, theta)."""
    if R is None:
        R = max_norm(X, Y)
    d = np.asarray(X).shape[1]
    prm = gaussian_params(eps, d, r, R)
    U = draw_anchors(r, d, prm["sigma"], seed)
    xi = feature_matrix(X, U, eps, prm["q"])
    zeta = feature_matrix(Y, U, eps, prm["q"])
    out = {}
    for name, (F, G, wa, wb) in {"xy": (xi, zeta, a, b), "xx": (xi, xi, a, a),
                                  "yy": (zeta, zeta, b, b)}.items():
        s = sinkhorn_factored(F, G, wa, wb, T=T, tol=tol)
        out[name] = dual_estimate(s["u"], s["v"], wa, wb, eps)
    out["div"] = out["xy"] - 0.5 * (out["xx"] + out["yy"])
    out.update(R=R, U=U)
    return out


# ---------------------------------------------------------------------------------------
# NEXT row f2: envelope gradients (Prop. diff-gene, chain rule PAPER.md:414-420)
# ---------------------------------------------------------------------------------------
def envelope_gradients(X, Y, U, xi, zeta, u, v, eps: float, q: float) -> dict:
    """Gradients of W_{eps,c_theta} at the optimal scalings (u, v), with the anchors theta = U
    and q held fixed.  Prop. diff-gene: dW/dK = -eps u v^T; with K = xi^T zeta (paper layout,
    xi r x n) this gives dW/dxi = -eps (zeta v) u^T and dW/dzeta = -eps (xi u) v^T
    (PAPER.md:414-420).  For the Gaussian map,
      d xi_ki / d x_i = -(4/eps) (x_i - u_k) xi_ki,
      d xi_ki / d u_k = xi_ki ( (4/eps)(x_i - u_k) + 2 u_k / (eps q) ),
    and the same for zeta with y_j.  Returns gX (n,d), gY (m,d), gU (r,d)."""
    X = np.asarray(X, np.float64)
    Y = np.asarray(Y, np.float64)
    U = np.asarray(U, np.float64)
    dW_dxi = -eps * np.outer(zeta @ v, u)           # r x n
    dW_dzeta = -eps * np.outer(xi @ u, v)           # r x m
    diffx = X[None, :, :] - U[:, None, :]           # r x n x d  (x_i - u_k)
    diffy = Y[None, :, :] - U[:, None, :]
    gX = np.einsum("ki,kid->id", dW_dxi * xi, -(4.0 / eps) * diffx)
    gY = np.einsum("kj,kjd->jd", dW_dzeta * zeta, -(4.0 / eps) * diffy)
    gU = (np.einsum("ki,kid->kd", dW_dxi * xi, (4.0 / eps) * diffx)
          + np.einsum("kj,kjd->kd", dW_dzeta * zeta, (4.0 / eps) * diffy)
          + ((dW_dxi * xi).sum(1) + (dW_dzeta * zeta).sum(1))[:, None] * 2.0 * U / (eps * q))
    return dict(gX=gX, gY=gY, gU=gU)


# ---------------------------------------------------------------------------------------
# NEXT row f3: perturbed arc-cosine positive features (Lemma decomp-arccos, PAPER.md:947-989;
# main text PAPER.md:377-382).  Reading C21: k_s uses the main-text Theta_s = sqrt(2) max(0,.)^s
# (PAPER.md:379), i.e. Cho & Saul's k_s = (1/pi)|x|^s|y|^s J_s(angle); the appendix proof drops
# the factor 2 of sqrt(2)^2 — the map as stated is unbiased for k_s + kappa with this k_s.
# ---------------------------------------------------------------------------------------
def arccos_phi(x, u, sigma: float, s: int, kappa: float) -> np.ndarray:
    """phi(x,u) = (sigma^{d/2} sqrt(2) max(0,u^T x)^s exp(-|u|^2/4 (1 - 1/sigma^2)), sqrt(kappa))
    (PAPER.md:951-953).  Returns (..., 2)."""
    x = np.asarray(x, np.float64)
    u = np.asarray(u, np.float64)
    d = x.shape[-1]
    ux = (x * u).sum(-1)
    relu = np.maximum(0.0, ux)
    pw = np.where(ux > 0, 1.0, 0.0) if s == 0 else relu ** s
    first = sigma ** (d / 2.0) * math.sqrt(2.0) * pw * np.exp(-(u * u).sum(-1) / 4.0 * (1.0 - 1.0 / sigma ** 2))
    return np.stack([first, np.full_like(first, math.sqrt(kappa))], axis=-1)


def arccos_kernel(x, y, s: int) -> float:
    """k_s(x,y) = (1/pi)|x|^s|y|^s J_s(theta) (Cho & Saul 2009, the kernel of PAPER.md:379):
    J_0 = pi - theta, J_1 = sin + (pi - theta) cos, J_2 = 3 sin cos + (pi - theta)(1 + 2 cos^2)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    nx, ny = np.linalg.norm(x), np.linalg.norm(y)
    c = float(np.clip(x @ y / (nx * ny), -1.0, 1.0))
    th = math.acos(c)
    sn = math.sin(th)
    J = {0: math.pi - th, 1: sn + (math.pi - th) * c,
         2: 3.0 * sn * c + (math.pi - th) * (1.0 + 2.0 * c * c)}[s]
    return (nx ** s) * (ny ** s) * J / math.pi


def feature_matrix_arccos(X, U, sigma: float, s: int, kappa: float) -> np.ndarray:
    """xi for the arc-cosine map in the paper layout with the kappa slot collapsed: rows
    0..r-1 = phi_1(x_i, u_k)/sqrt(r), row r = sqrt(kappa) (the r identical kappa slots of
    phi_theta(x) = r^{-1/2}(phi(x,u_1),...,phi(x,u_r)) contribute exactly kappa to every
    k_theta(x,y), as one column sqrt(kappa) does).  Shape (r+1, n)."""
    X = np.asarray(X, np.float64)
    U = np.asarray(U, np.float64)
    r = U.shape[0]
    ph = arccos_phi(X[None, :, :], U[:, None, :], sigma, s, kappa)[..., 0] / math.sqrt(r)
    return np.vstack([ph, np.full((1, X.shape[0]), math.sqrt(kappa))])


# ---------------------------------------------------------------------------------------
# NEXT f4. Accelerated Sinkhorn (Alg. 2; Eq. dual-smooth)
# ---------------------------------------------------------------------------------------
def accelerated_sinkhorn(K_mv: Callable[[np.ndarray], np.ndarray],
                         Kt_mv: Callable[[np.ndarray], np.ndarray],
                         a, b, eps: float, L0: float = 1.0, T: Optional[int] = None,
                         tol: Optional[float] = None, max_iter: int = 100000,
                         allowance: float = 1e-13, max_trials: int = 2000) -> dict:
    """Alg. 2 step by step, with the readings of DESIGN.md C22-C27:
      C22  phi(eta) := -F_theta(eta)/eps = log<e^{eta1}, K e^{eta2}> - <eta1,a> - <eta2,b>
           is the objective minimised; Eq. (dual-smooth)'s "<K e^{eta2}>" is <e^{eta1}, K e^{eta2}>.
      C23  "lambda^k = tau_k zeta^k + (1-tau_k) zeta^k" reads lambda^k = tau_k zeta^k + (1-tau_k) eta^k.
      C24  the duplicated "L_{k+1} = L_k/2" is one halving before the line search; each
           rejected trial doubles L_{k+1} ("Set L_{k+1} = 2 L_{k+1}").
      C25  the unchanged block: "eta_2^{k+1} = lambda_2^{k+1}" reads eta_2^{k+1} = lambda_2^k
           (and symmetrically eta_1^{k+1} = lambda_1^k).
      C26  "zeta^{k+1} = zeta^k - a_{k+1} grad F_theta(lambda^k)" and the acceptance test use
           grad phi (the gradient of the minimised objective, C22).
      C27  x_hat is kept through its marginals x_hat 1 and x_hat^T 1 (z is n x m); argmax ties
           pick block 1.  Stopping (tolerance mode): |x_hat 1 - a|_1 + |x_hat^T 1 - b|_1 < tol.
      C29  the acceptance test carries an fp64 rounding allowance of 1e-13 max(1, |phi(lambda)|):
           near the optimum the required decrease |grad|^2/(2L) falls below the rounding of
           phi itself, and a strict test would double L without bound.
      C28  a, b in the simplex (the theorem's "a, b in Delta_n"): the weights are
           divided by their fp64 sums first — with sum a != sum b, F_theta grows without bound
           along the gauge direction (eta1 + t, eta2 - t) and Alg. 2 drifts.
    Returns eta1, eta2, F = F_theta(eta) (= -eps phi(eta)), the primal marginals p1, p2,
    per-iteration traces (F, accepted L, block, trials) and the iteration count."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    a = a / a.sum()                                                     # C28
    b = b / b.sum()
    n, m = a.shape[0], b.shape[0]

    def phi(e1, e2):
        return math.log(np.exp(e1) @ K_mv(np.exp(e2))) - e1 @ a - e2 @ b

    # Init: A_0 = alpha_0 = 0, eta^0 = zeta^0 = lambda^0 = 0
    ak, Lk = 0.0, float(L0)
    eta1, eta2 = np.zeros(n), np.zeros(m)
    zet1, zet2 = np.zeros(n), np.zeros(m)
    p1, p2 = np.zeros(n), np.zeros(m)
    F_tr, L_tr, blk_tr, trials_tr, g_tr = [], [], [], [], []
    converged = False
    n_iter = T if tol is None else max_iter
    it = 0
    for _ in range(n_iter):
        L1 = Lk / 2.0                                                   # C24
        trials = 0
        while True:
            trials += 1
            a1 = 1.0 / (2.0 * L1) + math.sqrt(1.0 / (4.0 * L1 * L1) + ak * ak * Lk / L1)
            tau = 1.0 / (a1 * L1)
            lam1 = tau * zet1 + (1.0 - tau) * eta1                      # C23
            lam2 = tau * zet2 + (1.0 - tau) * eta2
            Kv = K_mv(np.exp(lam2))                                     # K e^{lambda2}
            Ktu = Kt_mv(np.exp(lam1))                                   # K^T e^{lambda1}
            c = float(np.exp(lam1) @ Kv)                                # <e^{l1}, K e^{l2}>
            g1 = np.exp(lam1) * Kv / c - a                              # grad_1 phi(lambda)
            g2 = np.exp(lam2) * Ktu / c - b                             # grad_2 phi(lambda)
            n1, n2 = float(g1 @ g1), float(g2 @ g2)
            blk = 1 if n1 >= n2 else 2                                  # argmax block (C27)
            if blk == 1:
                new1 = lam1 + np.log(a) - np.log(np.exp(lam1) * Kv)
                new2 = lam2                                             # C25
            else:
                new1 = lam1
                new2 = lam2 + np.log(b) - np.log(np.exp(lam2) * Ktu)
            ph_lam = phi(lam1, lam2)
            if phi(new1, new2) <= ph_lam - (n1 + n2) / (2.0 * L1) + allowance * max(1.0, abs(ph_lam)):
                zet1 = zet1 - a1 * g1                                   # C26
                zet2 = zet2 - a1 * g2
                # x_hat^{k+1} = (a_{k+1} c^{-1} z + L_k a_k^2 x_hat^k) / (L_{k+1} a_{k+1}^2)
                p1 = (a1 * (np.exp(lam1) * Kv) / c + Lk * ak * ak * p1) / (L1 * a1 * a1)
                p2 = (a1 * (np.exp(lam2) * Ktu) / c + Lk * ak * ak * p2) / (L1 * a1 * a1)
                eta1, eta2 = new1, new2
                ak, Lk = a1, L1
                break
            L1 = 2.0 * L1
            if trials >= max_trials:
                raise RuntimeError("Alg. 2 line search: %d rejected trials (L = %g)" % (trials, L1))
        it += 1
        F_tr.append(-eps * phi(eta1, eta2))
        L_tr.append(Lk)
        blk_tr.append(blk)
        trials_tr.append(trials)
        g_tr.append((n1, n2))
        if tol is not None and float(np.abs(p1 - a).sum() + np.abs(p2 - b).sum()) < tol:
            converged = True
            break
    return dict(eta1=eta1, eta2=eta2, F=-eps * phi(eta1, eta2), p1=p1, p2=p2, iters=it,
                F_trace=np.array(F_tr), L_trace=np.array(L_tr), blocks=np.array(blk_tr),
                trials=np.array(trials_tr), grad_norms=np.array(g_tr).reshape(-1, 2),
                converged=converged)


def accelerated_sinkhorn_factored(xi: np.ndarray, zeta: np.ndarray, a, b, eps: float,
                                  L0: float = 1.0, T=None, tol=None, max_iter=100000,
                                  **kw) -> dict:
    """Alg. 2 on K_theta = xi^T zeta: every K application costs r(n+m)."""
    xi = np.asarray(xi, dtype=np.float64)
    zeta = np.asarray(zeta, dtype=np.float64)
    return accelerated_sinkhorn(lambda v: xi.T @ (zeta @ v), lambda u: zeta.T @ (xi @ u), a, b,
                                eps, L0, T, tol, max_iter, **kw)


# ---------------------------------------------------------------------------------------
# NEXT f4 (second half). Small-eps stabilisation by row log-offsets (reading C30)
# ---------------------------------------------------------------------------------------
def feature_matrix_stabilized(X: np.ndarray, U: np.ndarray, eps: float, q: float):
    """Row-normalised features: xi_tilde[:, i] = xi[:, i] / max_k xi[k, i] and the natural-log
    offsets A_i = max_k log xi[k, i], so xi = xi_tilde e^{A} exactly (reading C30: Alg. 1 on
    K_tilde = diag(e^-A) K diag(e^-B) from u_tilde^0 = 1 is Alg. 1 on K from u^0 = e^{-A},
    "any arbitrary positive vector", PAPER.md:232 — same limit, and the same iterates as
    from u^0 = 1 when started at u_tilde^0 = e^{A}).  Computed
    from log phi (PAPER.md:934 written as an exponent), so nothing underflows before the
    shift.  Returns (xi_tilde r x n, A n)."""
    X = np.asarray(X, dtype=np.float64)
    U = np.asarray(U, dtype=np.float64)
    r, d = U.shape
    logphi = ((d / 4.0) * math.log(2.0 * q)
              - (2.0 / eps) * ((X[None, :, :] - U[:, None, :]) ** 2).sum(-1)
              + (U ** 2).sum(-1)[:, None] / (eps * q)
              - 0.5 * math.log(r))                                   # log(phi / sqrt(r)), r x n
    A = logphi.max(axis=0)
    return np.exp(logphi - A[None, :]), A


def dual_estimate_offset(u_t, v_t, a, b, A, B, eps: float) -> float:
    """W_hat from the scalings of the row-normalised problem: K = diag(e^A)
    K_tilde diag(e^B) gives u = u_tilde e^{-A}, v = v_tilde e^{-B}, so
    W_hat = eps (a^T (log u_tilde - A) + b^T (log v_tilde - B))."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return eps * (a @ (np.log(u_t) - A) + b @ (np.log(v_t) - B))
