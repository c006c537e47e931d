"""Oracle pins for NEXT f4: the accelerated Sinkhorn algorithm (Alg. 2).

Alg. 2 maximises the smooth dual F_theta (Eq. dual-smooth) by a different
route than Alg. 1, so its limit is pinned to Alg. 1's converged value (the dual optimum is
unique), to closed forms, to weak duality at every iterate and to the smoothness bound
L <= 2 of phi = -F/eps (Var of a sum over the two blocks; "L <= 2 eps^-1" in the
paper's scaling), which bounds every accepted L of the doubling line search by 4.
"""
import math

import numpy as np
import pytest

import oracle as O
import synth


def _small_factored(seed=0, n=23, m=31, r=7, eps=0.5, d=2):
    prob = synth.random_small(seed, n, m, d)
    R = O.max_norm(prob["X"], prob["Y"])
    p = O.gaussian_params(eps, d, r, R)
    U = O.draw_anchors(r, d, p["sigma"], 100 + seed)
    xi = O.feature_matrix(prob["X"], U, eps, p["q"])
    zeta = O.feature_matrix(prob["Y"], U, eps, p["q"])
    return prob, xi, zeta, eps


def test_accel_two_by_two_closed_form():
    """The P10 instance: F -> -ln 2 - ln(1 + e^-1) (eps = 1)."""
    K = np.exp(-np.array([[0.0, 1.0], [1.0, 0.0]]))
    a = b = np.array([0.5, 0.5])
    res = O.accelerated_sinkhorn_factored(K.T.copy(), np.eye(2), a, b, 1.0, T=80)
    assert abs(res["F"] - (-math.log(2.0) - math.log(1.0 + math.exp(-1.0)))) < 1e-12


def test_accel_rank_one_closed_form():
    """K = alpha beta^T: F -> eps(sum a ln a + sum b ln b - sum a ln alpha - sum b ln beta)."""
    rng = np.random.default_rng(3)
    n, m, eps = 17, 12, 0.7
    alpha, beta = rng.uniform(0.1, 2, n), rng.uniform(0.1, 2, m)
    a = rng.uniform(0.5, 1.5, n); a /= a.sum()
    b = rng.uniform(0.5, 1.5, m); b /= b.sum()
    expect = eps * (a @ np.log(a) + b @ np.log(b) - a @ np.log(alpha) - b @ np.log(beta))
    res = O.accelerated_sinkhorn_factored(alpha[None, :], beta[None, :], a, b, eps, T=200)
    assert abs(res["F"] - expect) < 1e-10


@pytest.mark.parametrize("seed,n,m,r", [(0, 8, 8, 5), (1, 8, 8, 8), (2, 23, 31, 7)])
def test_accel_matches_alg1_weak_duality_and_L_bound(seed, n, m, r):
    """Independent algorithms, one optimum: Alg. 2's F equals Alg. 1's converged W_hat;
    every iterate's F is below it (weak duality); every accepted L <= 4; the averaged plan's
    marginals converge to (a, b) and keep unit mass."""
    prob, xi, zeta, eps = _small_factored(seed, n, m, r)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    a, b = a / a.sum(), b / b.sum()          # reading C28: Alg. 2 works on the simplex
    s1 = O.sinkhorn_factored(xi, zeta, a, b, tol=1e-14, max_iter=200000)
    W = O.dual_estimate(s1["u"], s1["v"], a, b, eps)
    res = O.accelerated_sinkhorn_factored(xi, zeta, a, b, eps, L0=1.0, T=3000)
    assert abs(res["F"] - W) <= 1e-8 * abs(W), (res["F"], W)
    assert np.all(res["F_trace"] <= W + 1e-12 * abs(W))
    assert res["L_trace"].max() <= 4.0
    assert abs(res["p1"].sum() - 1.0) < 1e-12 and abs(res["p2"].sum() - 1.0) < 1e-12
    assert np.abs(res["p1"] - a).sum() + np.abs(res["p2"] - b).sum() < 1e-3


def test_accel_normalises_unbalanced_weights():
    """Reading C28: weights whose sums differ (fp32 rounding) are put on the simplex, so the
    result equals the run on explicitly normalised weights and stays bounded."""
    prob, xi, zeta, eps = _small_factored(0, 8, 8, 5)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    assert a.sum() != b.sum()
    r1 = O.accelerated_sinkhorn_factored(xi, zeta, a, b, eps, T=500)
    r2 = O.accelerated_sinkhorn_factored(xi, zeta, a / a.sum(), b / b.sum(), eps, T=500)
    assert abs(r1["F"] - r2["F"]) < 1e-14 and r1["L_trace"].max() <= 4.0


def test_accel_tolerance_mode_stops_on_plan_marginals():
    prob, xi, zeta, eps = _small_factored(5, 30, 20, 6)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    a, b = a / a.sum(), b / b.sum()
    res = O.accelerated_sinkhorn_factored(xi, zeta, a, b, eps, tol=1e-3, max_iter=100000)
    assert res["converged"]
    assert np.abs(res["p1"] - a).sum() + np.abs(res["p2"] - b).sum() < 1e-3
    again = O.accelerated_sinkhorn_factored(xi, zeta, a, b, eps, T=res["iters"] - 1)
    assert np.abs(again["p1"] - a).sum() + np.abs(again["p2"] - b).sum() >= 1e-3


@pytest.mark.parametrize("seed,n,m,r,eps", [(13, 8, 8, 5, 0.5), (17, 8, 8, 5, 0.5),
                                            (18, 23, 31, 7, 0.1)])
def test_accel_rounding_allowance_keeps_L_within_smoothness_bound(seed, n, m, r, eps):
    """Reading C29.  phi is 2-smooth, so in exact arithmetic every L >= 2 passes the acceptance
    test of the exact block step and no accepted L exceeds 4.  Run into the rounding regime
    (|grad phi|^2 ~ 1e-19: the required decrease |grad|^2/(2L) is below the fp64 rounding of
    phi itself),
    the strict test (allowance 0) rejects steps on rounding noise alone and doubles L past the
    bound (to 2^12 and beyond on these instances); with the 1e-13 max(1,|phi|) allowance every
    accepted L stays <= 4 and the value is unchanged."""
    prob, xi, zeta, _ = _small_factored(seed, n, m, r, eps=eps)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    a, b = a / a.sum(), b / b.sum()
    strict = O.accelerated_sinkhorn_factored(xi, zeta, a, b, eps, T=4000, allowance=0.0)
    k = int(np.argmax(strict["L_trace"] > 4.0))
    assert strict["L_trace"].max() > 4.0 * 2 ** 8                  # the bound is violated ...
    phi_k = abs(strict["F_trace"][k]) / eps                        # ... only in the rounding regime
    assert strict["grad_norms"][k].sum() / 2.0 < 4.0 * 2.0 ** -52 * max(1.0, phi_k)
    kept = O.accelerated_sinkhorn_factored(xi, zeta, a, b, eps, T=4000)
    assert kept["L_trace"].max() <= 4.0
    assert abs(kept["F"] - strict["F"]) <= 1e-14 * abs(kept["F"])
