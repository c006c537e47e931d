"""Pins for the matrix-free oracle (oracle/matrix_free.py + oracle/lsk_oracle_mf.c), the oracle
of config 5's full-size golden (fp64 factors of 2^23 x 4096 would take 550 GB).

It is pinned to the materialised-factor numpy oracle (itself pinned by quadrature, closed forms
and brute force: tests/test_oracle_*.py) and directly to closed forms of Alg. 1 (P9, P11)."""
import math

import numpy as np
import pytest

import oracle as O
import synth
from oracle import matrix_free as MF


def _prob(n, m, r, key=5, seed=3):
    cfg = synth.get_config(key)
    pr = synth.make_problem(cfg, n=n, m=m)
    R = O.max_norm(pr["X"], pr["Y"])
    prm = O.gaussian_params(cfg.eps, cfg.d, r, R)
    U = O.draw_anchors(r, cfg.d, prm["sigma"], seed)
    return cfg, pr, prm, U


def test_products_match_materialised_factors():
    cfg, pr, prm, U = _prob(1501, 1203, 96)
    xi = O.feature_matrix(pr["X"], U, cfg.eps, prm["q"])           # r x n
    w = np.random.default_rng(0).uniform(0.1, 1.0, 1501)
    s = MF.apply(pr["X"], U, cfg.eps, prm["q"], w)
    assert np.allclose(s, xi @ w, rtol=1e-13, atol=0)
    t = MF.apply_t(pr["X"], U, cfg.eps, prm["q"], s)
    assert np.allclose(t, xi.T @ s, rtol=1e-13, atol=0)


def test_half_iteration_is_the_two_products():
    """The fused half-iteration computes the same sums as apply_t then apply (same blocks,
    same order): bit-identical."""
    cfg, pr, prm, U = _prob(2001, 999, 64)
    s = MF.apply(pr["X"], U, cfg.eps, prm["q"], np.ones(2001))
    out, t, s_next = MF.half_iteration(pr["Y"], U, cfg.eps, prm["q"], s, pr["b"])
    t_ref = MF.apply_t(pr["Y"], U, cfg.eps, prm["q"], s)
    assert np.array_equal(t, t_ref)
    assert np.array_equal(out, pr["b"].astype(np.float64) / t_ref)
    assert np.array_equal(s_next, MF.apply(pr["Y"], U, cfg.eps, prm["q"], out))


@pytest.mark.parametrize("key,n,m,r,T", [(5, 3001, 2999, 128, 15), (2, 777, 1234, 100, 30),
                                         (1, 500, 500, 100, 200)])
def test_sinkhorn_matches_numpy_oracle(key, n, m, r, T):
    cfg, pr, prm, U = _prob(n, m, r, key=key)
    ref = O.rot(pr["X"], pr["Y"], pr["a"], pr["b"], cfg.eps, r, 3, T=T, U=U, record_err=True)
    sol = MF.sinkhorn_matrix_free(pr["X"], pr["Y"], U, pr["a"], pr["b"], cfg.eps, prm["q"], T=T,
                                  record_last_err=True)
    assert np.max(np.abs(sol["u"] / ref["u"] - 1.0)) < 1e-11
    assert np.max(np.abs(sol["v"] / ref["v"] - 1.0)) < 1e-11
    rot = O.dual_estimate(sol["u"], sol["v"], pr["a"], pr["b"], cfg.eps)
    assert abs(rot - ref["rot"]) <= 1e-11 * abs(ref["rot"])
    # |v o K^T u - b|_1 near convergence cancels: compare to the rounding of its terms
    assert abs(sol["last_err"] - ref["errs"][-1]) <= 1e-9 * ref["errs"][-1] + 1e-13 * pr["b"].sum()


def test_rank_one_closed_form_large():
    """P11 at a size where the numpy oracle would not be used: all x_i = x_0 and all y_j = y_0
    make K = k 1 1^T with k = k_theta(x0, y0) = (1/r) sum_k phi(x0,u_k) phi(y0,u_k) (PAPER.md:297,
    934; phi pinned by quadrature).  From u^0 = 1, Alg. 1 gives u = alpha a, v = beta b with
      T = 1: alpha = n / Sb,          beta = 1 / (k n),
      T = 2: alpha = n Sa / Sb^2,     beta = Sb / (k n Sa)       (Sa = sum a, Sb = sum b),
    so W_hat / eps = sum a ln a + sum b ln b + Sa ln alpha + Sb ln beta — with Sa = Sb = 1 the
    textbook sum a ln a + sum b ln b - ln k.  (The fp32 uniform weights' sums are 1 +- 1e-7.)"""
    cfg = synth.get_config(5)
    n, m, r = 200003, 150001, 256
    pr = synth.make_problem(cfg, n=n, m=m, identical_points=True)
    R = O.max_norm(pr["X"], pr["Y"])
    prm = O.gaussian_params(cfg.eps, cfg.d, r, R)
    U = O.draw_anchors(r, cfg.d, prm["sigma"], 9)
    k = float(np.mean(O.gaussian_phi(pr["X"][:1].astype(np.float64), U, cfg.eps, prm["q"])
                      * O.gaussian_phi(pr["Y"][:1].astype(np.float64), U, cfg.eps, prm["q"])))
    a = pr["a"].astype(np.float64)
    b = pr["b"].astype(np.float64)
    Sa, Sb = a.sum(), b.sum()
    base = a @ np.log(a) + b @ np.log(b)
    for T, alpha, beta in ((1, n / Sb, 1.0 / (k * n)), (2, n * Sa / Sb ** 2, Sb / (k * n * Sa))):
        sol = MF.sinkhorn_matrix_free(pr["X"], pr["Y"], U, pr["a"], pr["b"], cfg.eps, prm["q"], T=T)
        got = O.dual_estimate(sol["u"], sol["v"], pr["a"], pr["b"], cfg.eps)
        exact = cfg.eps * (base + Sa * math.log(alpha) + Sb * math.log(beta))
        assert abs(got - exact) <= 1e-12 * abs(exact)
        assert abs(got - cfg.eps * (base - math.log(k))) <= 1e-5 * abs(exact)
        assert np.allclose(sol["u"], alpha * a, rtol=1e-12) and np.allclose(sol["v"], beta * b, rtol=1e-12)


def test_single_point():
    """P9: n = m = 1 gives W_hat = -eps ln k_theta(x, y) = c_theta(x, y) (eq. cost)."""
    eps, d, r = 0.05, 3, 64
    x = np.array([[0.2, -0.1, 0.3]])
    y = np.array([[-0.4, 0.1, 0.0]])
    prm = O.gaussian_params(eps, d, r, O.max_norm(x, y))
    U = O.draw_anchors(r, d, prm["sigma"], 4)
    k = float(np.mean(O.gaussian_phi(x, U, eps, prm["q"]) * O.gaussian_phi(y, U, eps, prm["q"])))
    sol = MF.sinkhorn_matrix_free(x, y, U, [1.0], [1.0], eps, prm["q"], T=3)
    assert abs(O.dual_estimate(sol["u"], sol["v"], [1.0], [1.0], eps) + eps * math.log(k)) < 1e-14
