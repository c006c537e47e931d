"""Oracle pins for the small-eps stabilisation (NEXT f4, reading C30): row log-offsets keep the
factorisation and the value of Alg. 1."""
import math

import numpy as np

import oracle as O
import synth


def _setup(eps, n=300, m=280, r=64, seed=7):
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=n, m=m)
    R = O.max_norm(prob["X"], prob["Y"])
    p = O.gaussian_params(eps, 2, r, R)
    U = O.draw_anchors(r, 2, p["sigma"], seed)
    return prob, U, p


def test_stabilized_features_reconstruct_exactly():
    prob, U, p = _setup(0.1)
    xi = O.feature_matrix(prob["X"], U, 0.1, p["q"])
    xt, A = O.feature_matrix_stabilized(prob["X"], U, 0.1, p["q"])
    assert np.allclose(xt * np.exp(A)[None, :], xi, rtol=1e-12, atol=0)
    assert np.all(xt.max(axis=0) == 1.0) and np.all(xt <= 1.0) and np.all(xt > 0.0)


def test_stabilized_sinkhorn_same_value():
    """Sinkhorn on the row-normalised factors with offsets = Sinkhorn on the plain factors
    (a gauge transformation of the scalings): started at u_tilde^0 = e^{A} the iterates map
    exactly (same W_hat to 1e-12 at every T); from u_tilde^0 = 1 the limit is the same."""
    eps = 0.1
    prob, U, p = _setup(eps)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    xi = O.feature_matrix(prob["X"], U, eps, p["q"])
    zeta = O.feature_matrix(prob["Y"], U, eps, p["q"])
    xt, A = O.feature_matrix_stabilized(prob["X"], U, eps, p["q"])
    zt, B = O.feature_matrix_stabilized(prob["Y"], U, eps, p["q"])
    for T in (1, 5, 50):
        s0 = O.sinkhorn_factored(xi, zeta, a, b, T=T)
        s1 = O.sinkhorn_factored(xt, zt, a, b, T=T, u0=np.exp(A))
        w0 = O.dual_estimate(s0["u"], s0["v"], a, b, eps)
        w1 = O.dual_estimate_offset(s1["u"], s1["v"], a, b, A, B, eps)
        assert abs(w0 - w1) <= 1e-12 * abs(w0)
        assert np.allclose(s1["u"] * np.exp(-A), s0["u"], rtol=1e-10)
    a, b = a / a.sum(), b / b.sum()   # the limit's gauge is free only when sum a = sum b
    c0 = O.sinkhorn_factored(xi, zeta, a, b, tol=1e-13, max_iter=100000)
    c1 = O.sinkhorn_factored(xt, zt, a, b, tol=1e-13, max_iter=100000)
    w0 = O.dual_estimate(c0["u"], c0["v"], a, b, eps)
    w1 = O.dual_estimate_offset(c1["u"], c1["v"], a, b, A, B, eps)
    assert abs(w0 - w1) <= 1e-10 * abs(w0)


def test_stabilized_reaches_small_eps_in_fp32_range():
    """eps = 0.01 (the paper's failure regime): the plain features of some rows
    fall below the fp32 normal range (1.2e-38), the row-normalised ones keep every row's
    largest entry at 1 (what the fp32 GPU path needs)."""
    eps = 0.01
    prob, U, p = _setup(eps)
    xi = O.feature_matrix(prob["X"], U, eps, p["q"])
    xt, A = O.feature_matrix_stabilized(prob["X"], U, eps, p["q"])
    assert (xi.max(axis=0) < 1.2e-38).any() or (xi < 1.2e-38).mean() > 0.5
    assert np.all(xt.max(axis=0) == 1.0)
