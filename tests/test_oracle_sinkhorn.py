"""Oracle pins for Alg. 1 on K_theta = xi^T zeta and the dual read-out (steps a4-a9)."""
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


# ---------------- P8: factored == dense on the materialised K_theta -----------------------
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_factored_equals_dense(seed):
    prob, xi, zeta, eps = _small_factored(seed)
    K = xi.T @ zeta                         # K_theta = xi^T zeta
    f = O.sinkhorn_factored(xi, zeta, prob["a"], prob["b"], T=25, record_err=True)
    g = O.sinkhorn_dense(K, prob["a"], prob["b"], T=25, record_err=True)
    assert np.allclose(f["u"], g["u"], rtol=1e-12, atol=0)
    assert np.allclose(f["v"], g["v"], rtol=1e-12, atol=0)
    assert abs(O.dual_estimate(f["u"], f["v"], prob["a"], prob["b"], eps)
               - O.dual_estimate(g["u"], g["v"], prob["a"], prob["b"], eps)) < 1e-12
    # explicit K^T u / K v vs elementwise sums (no matmul reordering question at all)
    u = np.linspace(0.5, 2, K.shape[0])
    ktu = np.array([sum(K[i, j] * u[i] for i in range(K.shape[0])) for j in range(K.shape[1])])
    assert np.allclose(zeta.T @ (xi @ u), ktu, rtol=1e-13)


# ---------------- P9: single point, W_hat = c_theta(x,y) --------------------
@pytest.mark.parametrize("T", [1, 5])
def test_single_point(T):
    eps, d, r = 0.7, 3, 64
    rng = np.random.default_rng(3)
    x, y = rng.normal(size=(1, d)) * 0.3, rng.normal(size=(1, d)) * 0.3
    R = O.max_norm(x, y)
    p = O.gaussian_params(eps, d, r, R)
    U = O.draw_anchors(r, d, p["sigma"], 5)
    xi = O.feature_matrix(x, U, eps, p["q"])
    zeta = O.feature_matrix(y, U, eps, p["q"])
    s = O.sinkhorn_factored(xi, zeta, [1.0], [1.0], T=T)
    k_theta = float(xi[:, 0] @ zeta[:, 0])
    # c_theta = -eps log phi_theta(x)^T phi_theta(y)  (eq. cost)
    assert abs(O.dual_estimate(s["u"], s["v"], [1.0], [1.0], eps) - (-eps * math.log(k_theta))) < 1e-14


# ---------------- P10: 2x2 closed form ---------------------------------------------------
def test_two_by_two_closed_form():
    """a=b=(1/2,1/2), C=[[0,1],[1,0]], eps=1: by symmetry u=v=c 1 with c^2(1+e^-1)=1/2, so
    W = eps*(a^T ln u + b^T ln v) = ln c^2 = -ln 2 - ln(1+e^-1)."""
    K = np.exp(-np.array([[0.0, 1.0], [1.0, 0.0]]))
    expect = -math.log(2.0) - math.log(1.0 + math.exp(-1.0))
    a = b = np.array([0.5, 0.5])
    g = O.sinkhorn_dense(K, a, b, T=50)
    assert abs(O.dual_estimate(g["u"], g["v"], a, b, 1.0) - expect) < 1e-14
    # same K as a factorisation xi^T zeta with zeta = I, xi = K (r = 2)
    f = O.sinkhorn_factored(K.T.copy(), np.eye(2), a, b, T=50)
    assert abs(O.dual_estimate(f["u"], f["v"], a, b, 1.0) - expect) < 1e-14


# ---------------- P11: rank-one closed form -----------------------------------------------
def test_rank_one_closed_form():
    """K = alpha beta^T (r=1): after one iteration P = a b^T and
    W/eps = sum a ln a + sum b ln b - sum a ln alpha - sum b ln beta (Sum a = Sum b = 1)."""
    rng = np.random.default_rng(7)
    n, m = 40, 55
    alpha, beta = rng.uniform(0.1, 2, n), rng.uniform(0.1, 2, m)
    a = rng.uniform(0.5, 1.5, n); a /= a.sum()
    b = rng.uniform(0.5, 1.5, m); b /= b.sum()
    eps = 0.3
    expect = eps * (a @ np.log(a) + b @ np.log(b) - a @ np.log(alpha) - b @ np.log(beta))
    for T in (1, 3):
        s = O.sinkhorn_factored(alpha[None, :], beta[None, :], a, b, T=T)
        assert abs(O.dual_estimate(s["u"], s["v"], a, b, eps) - expect) < 1e-13
        P = s["u"][:, None] * np.outer(alpha, beta) * s["v"][None, :]
        assert np.allclose(P, np.outer(a, b), rtol=1e-13)


def test_identical_points_closed_form():
    """All x_i equal and all y_j equal => K_theta = kappa 1 1^T (rank one with alpha = 1_n,
    beta = kappa 1_m).  One Sinkhorn loop gives, for any positive a, b:
    W/eps = sum a ln a + sum b ln b - (sum b) ln kappa + (sum a - sum b) ln n
            - (sum a) ln(sum b); with uniform weights W = eps(-ln n - ln m) + c_theta(x,y).
    This is the full-size GPU pin of P11."""
    cfg = synth.get_config(5)
    prob = synth.make_problem(cfg, n=300, m=200, identical_points=True)
    r = 256
    res = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, r, 9, T=3)
    kappa = float(res["xi"][:, 0] @ res["zeta"][:, 0])
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    expect = cfg.eps * (a @ np.log(a) + b @ np.log(b) - b.sum() * math.log(kappa)
                        + (a.sum() - b.sum()) * math.log(300) - a.sum() * math.log(b.sum()))
    assert abs(res["rot"] - expect) < 1e-12
    assert abs(expect - (cfg.eps * (-math.log(300) - math.log(200)) - cfg.eps * math.log(kappa))) < 1e-6


# ---------------- P12: marginal identities after every iteration -----------
def test_marginal_identities():
    prob, xi, zeta, eps = _small_factored(4, n=40, m=33, r=9)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    for T in (1, 2, 7):
        s = O.sinkhorn_factored(xi, zeta, a, b, T=T)
        Kv = xi.T @ (zeta @ s["v"])
        assert np.allclose(s["u"] * Kv, a, rtol=1e-14)        # row marginal exact
        assert abs(s["u"] @ Kv - a.sum()) < 1e-14              # u^T K v = 1
        Ktu = zeta.T @ (xi @ s["u"])
        err = O.marginal_error(s["u"], s["v"], Ktu, b)
        assert err >= 0


# ---------------- P13: convergence (Thm cvg-sink) ----------
def test_convergence_config1():
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    res = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed,
                T=cfg.T, record_err=True)
    errs = res["errs"]
    assert errs[-1] < 1e-6 * max(1.0, errs[0])
    assert np.all(np.diff(errs[:20]) <= 1e-12)       # monotone early phase
    # tolerance mode stops at the first t with err_t < tol and agrees with fixed-T
    tol = 1e-6
    t = O.sinkhorn_factored(res["xi"], res["zeta"], prob["a"], prob["b"], tol=tol)
    assert t["converged"] and t["errs"][-1] < tol and (len(t["errs"]) == 1 or t["errs"][-2] >= tol)
    it = t["iters"]
    assert abs(it - (np.argmax(errs < tol) + 1)) == 0


# ---------------- P14: primal == dual at convergence --------------
def test_primal_equals_dual():
    prob, xi, zeta, eps = _small_factored(5, n=30, m=26, r=12, eps=0.5)
    # the identity needs sum a = sum b = 1 exactly (the +eps cancels u^T K v = 1, C7);
    # fp32 weights miss it by ~1e-7, so renormalise in fp64 here.
    prob["a"] = prob["a"].astype(np.float64) / prob["a"].astype(np.float64).sum()
    prob["b"] = prob["b"].astype(np.float64) / prob["b"].astype(np.float64).sum()
    s = O.sinkhorn_factored(xi, zeta, prob["a"], prob["b"], tol=1e-14)
    K = xi.T @ zeta
    P = s["u"][:, None] * K * s["v"][None, :]
    C = -eps * np.log(K)                       # c_theta (eq. cost)
    primal = O.primal_objective(P, C, eps)
    dual = O.dual_estimate(s["u"], s["v"], prob["a"], prob["b"], eps)
    assert abs(primal - dual) < 1e-10


# ---------------- P15: gauge invariance --------------------------------
def test_gauge_invariance():
    prob, xi, zeta, eps = _small_factored(6)
    a = prob["a"].astype(np.float64); a /= a.sum()
    b = prob["b"].astype(np.float64); b /= b.sum()
    s = O.sinkhorn_factored(xi, zeta, a, b, T=10)
    w0 = O.dual_estimate(s["u"], s["v"], a, b, eps)
    for t in (1e-3, 2.5, 1e4):
        assert abs(O.dual_estimate(t * s["u"], s["v"] / t, a, b, eps) - w0) < 1e-12


# ---------------- P17: dual range (Lemma gene_control_dual) ------------
def test_dual_range_bound():
    prob, xi, zeta, eps = _small_factored(8, n=24, m=24, r=10)
    s = O.sinkhorn_factored(xi, zeta, prob["a"], prob["b"], tol=1e-13)
    K = xi.T @ zeta
    iota = min(prob["a"].min(), prob["b"].min())
    RK = -math.log(iota * K.min() / K.max())
    alpha, beta = eps * np.log(s["u"]), eps * np.log(s["v"])
    assert alpha.max() - alpha.min() <= eps * RK
    assert beta.max() - beta.min() <= eps * RK


# ---------------- P16: the paper's RE behaviour on its illustration setup ------------------
def test_relative_error_behaviour():
    """RF is accurate at eps=0.5 and 0.1 and improves with r.  The paper
    prints no numbers (figures are placeholders), so only the trends are asserted: |RE| is
    small (< 5%) and falls from r=100 to r=2000 (mean over seeds).  RE := (W_hat - W)/|W|
    (reading C16).  W is the dense exact-Gaussian ROT at tight tolerance."""
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=700, m=700)
    X, Y, a, b = prob["X"], prob["Y"], prob["a"], prob["b"]
    for eps in (0.5, 0.1):
        K = O.gaussian_kernel_dense(X, Y, eps)
        g = O.sinkhorn_dense(K, a, b, tol=1e-12)
        W = O.dual_estimate(g["u"], g["v"], a, b, eps)
        res = {}
        for r in (100, 2000):
            res[r] = np.mean([abs(O.rot(X, Y, a, b, eps, r, s, tol=1e-10)["rot"] - W) / abs(W)
                              for s in range(4)])
        assert res[100] < 0.05 and res[2000] < res[100], (eps, res)


# ---------------- NEXT f1: Sinkhorn divergence (eq. reg-sdiv) -------------------
def test_divergence_pins():
    """W_bar(mu,mu) = 0 exactly (the three solves coincide); at convergence
    W_bar(mu,nu) = W_bar(nu,mu) (the transposed problem has the same optimum); the value is
    the formula applied to three independent dual estimates."""
    prob = synth.random_small(21, 60, 45, 2)
    X, Y = prob["X"], prob["Y"]
    # exact balance sum a = sum b = 1 (fp32 weights miss it by ~1e-7, which breaks the exact
    # (mu,nu) <-> (nu,mu) symmetry at the 1e-9 level)
    a = prob["a"].astype(np.float64) / prob["a"].astype(np.float64).sum()
    b = prob["b"].astype(np.float64) / prob["b"].astype(np.float64).sum()
    eps, r = 0.5, 32
    same = O.sinkhorn_divergence(X, X, a, a, eps, r, 3, T=30)
    assert same["div"] == 0.0
    d1 = O.sinkhorn_divergence(X, Y, a, b, eps, r, 3, tol=1e-13)
    d2 = O.sinkhorn_divergence(Y, X, b, a, eps, r, 3, tol=1e-13)
    assert abs(d1["div"] - d2["div"]) < 1e-10
    res = O.rot(X, Y, a, b, eps, r, 3, tol=1e-13, R=d1["R"])
    assert abs(res["rot"] - d1["xy"]) < 1e-12
    # the Gram kernel k_theta = phi^T phi is positive semi-definite: W_bar >= 0 (Feydy et al.
    # 2019, Thm 1) — checked as a sanity property on these inputs only
    assert d1["div"] > -1e-10


# ---------------- NEXT f2: envelope gradients, pinned by finite differences ---------------------
def test_envelope_gradients_finite_differences():
    """dW/dx_i, dW/dy_j, dW/du_k from Prop. diff-gene + chain rule vs
    central finite differences of W_hat at tight convergence, theta = U and R (so q) fixed."""
    prob = synth.random_small(31, 14, 11, 2)
    X, Y = prob["X"].astype(np.float64), prob["Y"].astype(np.float64)
    a = prob["a"].astype(np.float64); a /= a.sum()
    b = prob["b"].astype(np.float64); b /= b.sum()
    eps, r, R = 0.6, 24, 2.0
    prm = O.gaussian_params(eps, 2, r, R)
    U = O.draw_anchors(r, 2, prm["sigma"], 4)

    def W(X_, Y_, U_):
        return O.rot(X_, Y_, a, b, eps, r, 0, tol=1e-14, R=R, U=U_)["rot"]

    res = O.rot(X, Y, a, b, eps, r, 0, tol=1e-14, R=R, U=U)
    g = O.envelope_gradients(X, Y, U, res["xi"], res["zeta"], res["u"], res["v"], eps, prm["q"])
    h = 1e-5
    for name, arr, grad in (("X", X, g["gX"]), ("Y", Y, g["gY"]), ("U", U, g["gU"])):
        for (i, c) in [(0, 0), (3, 1), (arr.shape[0] - 1, 0)]:
            P, M = arr.copy(), arr.copy()
            P[i, c] += h
            M[i, c] -= h
            args_p = dict(X=X, Y=Y, U=U)
            args_m = dict(X=X, Y=Y, U=U)
            args_p[name], args_m[name] = P, M
            fd = (W(args_p["X"], args_p["Y"], args_p["U"]) - W(args_m["X"], args_m["Y"], args_m["U"])) / (2 * h)
            assert abs(fd - grad[i, c]) <= 1e-6 * max(1.0, abs(fd)), (name, i, c, fd, grad[i, c])


# ---------------- hand-computed pins of the two helpers ---------------------------------------
def test_max_norm_hand_computed():
    """R = max over BOTH clouds of |p|_2 (reading C3), with Pythagorean triples (exact in fp32
    and fp64): the maximum in Y, then in X, then with negative coordinates and d = 3."""
    X = np.array([[3.0, 4.0], [0.0, 1.0]], np.float32)            # norms 5, 1
    Y = np.array([[6.0, 8.0], [-1.0, 0.0]], np.float32)           # norms 10, 1
    assert O.max_norm(X, Y) == 10.0
    assert O.max_norm(Y[1:], X) == 5.0
    X3 = np.array([[-3.0, 4.0, 12.0], [1.0, 2.0, 2.0]], np.float32)   # 13, 3
    Y3 = np.array([[2.0, -3.0, 6.0]], np.float32)                      # 7
    assert O.max_norm(X3, Y3) == 13.0
    assert O.max_norm(Y3, X3[1:]) == 7.0


def test_marginal_error_hand_computed():
    """|v o K^T u - b|_1 on a 2 x 2 case worked by hand:
    K = [[1,2],[3,4]], u = (1,2): K^T u = (7, 10); v = (1/2, 1/4): v o K^T u = (3.5, 2.5);
    b = (0.4, 0.6): |(3.1, 1.9)|_1 = 5.0.  A v with the opposite sign of error: v = (0, 0.1)
    gives |(-0.4, 0.4)|_1 = 0.8."""
    K = np.array([[1.0, 2.0], [3.0, 4.0]])
    u = np.array([1.0, 2.0])
    b = np.array([0.4, 0.6])
    assert abs(O.marginal_error(u, np.array([0.5, 0.25]), K.T @ u, b) - 5.0) < 1e-15
    assert abs(O.marginal_error(u, np.array([0.0, 0.1]), K.T @ u, b) - 0.8) < 1e-15
    # and the oracle's recorded err_t is this quantity of its own iterates
    res = O.sinkhorn_dense(K, [0.5, 0.5], [0.4, 0.6], T=3, record_err=True)
    assert abs(res["errs"][-1] - O.marginal_error(res["u"], res["v"], K.T @ res["u"], [0.4, 0.6])) == 0.0
