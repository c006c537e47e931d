"""Oracle pins for steps a1-a3 (feature parameters, anchors, Gaussian positive features).

Each test pins an oracle function to something other than itself: a library routine, a
published known-answer vector, a closed form or an exact identity of PAPER.md.
"""
import math
import os

import numpy as np
import pytest
import scipy.special

import oracle as O


def _read_golden(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------- P1: Lambert W_0 ------------------
def test_lambert_golden(golden_dir):
    for x, w in _read_golden(os.path.join(golden_dir, "lambert_w0.txt")):
        assert abs(O.lambert_w0(float(x)) - float(w)) <= 1e-15 * max(1.0, abs(float(w)))


def test_lambert_vs_scipy_and_residual():
    xs = np.logspace(-12, 8, 4000)
    for x in xs:
        w = O.lambert_w0(float(x))
        ref = float(np.real(scipy.special.lambertw(x, 0)))
        assert abs(w - ref) <= 1e-13 * max(1.0, abs(ref))
        assert abs(w * math.exp(w) - x) <= 1e-12 * max(1.0, x)


def test_lambert_domain():
    with pytest.raises(ValueError):
        O.lambert_w0(-1.0)


# ---------------- P2: q and sigma -------------------------------
@pytest.mark.parametrize("eps,d,R", [(0.5, 2, 1.24), (0.1, 2, 1.55), (0.2, 16, 1.0),
                                     (1.0, 128, 1.33), (0.05, 3, 1.0), (3.0, 1, 0.2)])
def test_q_identities(eps, d, R):
    p = O.gaussian_params(eps, d, 100, R)
    z = R * R / (eps * d)
    # q W_0(z) 2 eps d = R^2   (definition)
    assert abs(p["q"] * p["W"] * 2 * eps * d - R * R) <= 1e-12 * R * R
    # W e^W = z  =>  q = e^{W}/2 > 1/2
    assert abs(p["q"] - math.exp(float(np.real(scipy.special.lambertw(z)))) / 2) <= 1e-12 * p["q"]
    assert p["q"] > 0.5
    assert abs(p["sigma"] ** 2 - p["q"] * eps / 4) <= 1e-14 * p["sigma"] ** 2
    assert abs(p["log_scale"] - (d / 4 * math.log(2 * p["q"]) - 0.5 * math.log(100))) < 1e-14 * 10


# ---------------- P3: phi(0,0) = (2q)^{d/4} ------------------
@pytest.mark.parametrize("d,q", [(1, 0.7), (2, 1.3), (3, 2.2), (16, 0.64)])
def test_phi_origin(d, q):
    val = O.gaussian_phi(np.zeros(d), np.zeros(d), 0.3, q)
    assert abs(val - (2 * q) ** (d / 4)) <= 1e-15 * (2 * q) ** (d / 4)


# ---------------- P4: kernel identity by Gauss-Hermite quadrature ------------------------
# k(x,y) = int phi(x,u) phi(y,u) d rho(u) = exp(-|x-y|^2/eps)  (Lemma decomp-RBF)
# rho = N(0, sigma^2 I): E f(sigma Z) = sum_j w_j f(sigma t_j) / sqrt(2 pi) (probabilists'
# Hermite nodes, numpy.polynomial.hermite_e.hermegauss).  A dropped constant, a wrong sign in
# an exponent or the main-text exponent (reading C1) all fail this.
@pytest.mark.parametrize("d,eps,R,x,y", [
    (1, 0.5, 1.0, [0.3], [-0.4]),
    (1, 0.1, 1.0, [0.1], [0.25]),
    (2, 0.5, 1.0, [0.1, 0.0], [0.0, 0.2]),
    (2, 0.05, 0.5, [0.1, -0.05], [0.02, 0.1]),
])
def test_kernel_identity_gauss_hermite(d, eps, R, x, y):
    p = O.gaussian_params(eps, d, 1, R)
    t, w = np.polynomial.hermite_e.hermegauss(200)
    w = w / math.sqrt(2 * math.pi)
    grids = np.meshgrid(*([t] * d), indexing="ij")
    wts = np.ones_like(grids[0])
    for g in np.meshgrid(*([w] * d), indexing="ij"):
        wts = wts * g
    U = p["sigma"] * np.stack([g.ravel() for g in grids], axis=1)
    vals = O.gaussian_phi(np.array(x), U, eps, p["q"]) * O.gaussian_phi(np.array(y), U, eps, p["q"])
    integral = float((vals * wts.ravel()).sum())
    exact = math.exp(-float(((np.array(x) - np.array(y)) ** 2).sum()) / eps)
    assert abs(integral / exact - 1) < 1e-10


def test_main_text_exponent_is_biased():
    """Reading C1: the main-text factor exp(eps^-1|u|^2/(1/2+eps^-1 R^2)) does
    not reproduce k; the appendix factor exp(eps^-1|u|^2/q) does (above)."""
    d, eps, R = 1, 0.5, 1.0
    p = O.gaussian_params(eps, d, 1, R)
    t, w = np.polynomial.hermite_e.hermegauss(200)
    w = w / math.sqrt(2 * math.pi)
    u = p["sigma"] * t
    x, y = 0.3, -0.1

    def phi_main(xx):
        return (2 * p["q"]) ** (d / 4) * np.exp(-2 / eps * (xx - u) ** 2) * \
            np.exp(u * u / eps / (0.5 + R * R / eps))
    integral = float((phi_main(x) * phi_main(y) * w).sum())
    exact = math.exp(-(x - y) ** 2 / eps)
    assert abs(integral / exact - 1) > 1e-2


# ---------------- P6 (corrected, reading C20): sup over u of phi phi / k ------------------
# Appendix derivation: phi(x,u)phi(y,u)/k = (2q)^{d/2}
#   exp(-4 eps^-1 (1-1/2q)|u - (1-1/2q)^{-1} m|^2) exp(4 eps^-1 |m|^2/(2q-1)),  m = (x+y)/2,
# so sup_u = (2q)^{d/2} exp(4|m|^2/(eps(2q-1))).  The stated bound 2(2q)^{d/2} (PAPER.md:393,
# 930) does not follow from it (C20); we pin the exact supremum instead.
@pytest.mark.parametrize("eps,R,ang", [(0.5, 1.24, 0.3), (0.1, 1.0, 1.0), (1.0, 0.5, 2.0)])
def test_ratio_supremum_closed_form(eps, R, ang):
    d = 2
    p = O.gaussian_params(eps, d, 1, R)
    q = p["q"]
    x = 0.8 * R * np.array([math.cos(ang), math.sin(ang)])
    y = 0.5 * R * np.array([math.cos(ang + 0.4), math.sin(ang + 0.4)])
    m = (x + y) / 2
    k = math.exp(-float(((x - y) ** 2).sum()) / eps)
    sup_formula = (2 * q) ** (d / 2) * math.exp(4 * float(m @ m) / (eps * (2 * q - 1)))
    ustar = m / (1 - 1 / (2 * q))
    ratio = lambda u: O.gaussian_phi(x, u, eps, q) * O.gaussian_phi(y, u, eps, q) / k
    assert abs(ratio(ustar) / sup_formula - 1) < 1e-12
    rng = np.random.default_rng(0)
    pert = ustar + rng.normal(0, 0.05, size=(2000, 2))
    assert np.all(ratio(pert) <= sup_formula * (1 + 1e-12))


# ---------------- P7: positivity of every fp64 feature ---------------
def test_feature_positivity_and_definition():
    import synth
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=600, m=600)
    R = O.max_norm(prob["X"], prob["Y"])
    p = O.gaussian_params(cfg.eps, 2, 257, R)
    U = O.draw_anchors(257, 2, p["sigma"], 11)
    xi = O.feature_matrix(prob["X"], U, cfg.eps, p["q"])
    assert xi.shape == (257, 600)
    assert np.all(xi > 0)
    # feature_matrix entry == phi(x_i,u_k)/sqrt(r) computed one by one
    rng = np.random.default_rng(1)
    rows = rng.integers(0, 600, 50)
    cols = rng.integers(0, 257, 50)
    one = O.feature_entries_scaled(prob["X"], U, cfg.eps, p["q"], 257, rows, cols)
    assert np.allclose(xi[cols, rows], one, rtol=1e-13, atol=0)


# ---------------- P5: Monte-Carlo rate (north_star) ---------------------
def test_monte_carlo_rate():
    """(1/r) sum_k phi(x,u_k)phi(y,u_k) -> k(x,y) with RMS error ~ r^{-1/2}."""
    eps, d, R = 0.5, 2, 1.0
    p = O.gaussian_params(eps, d, 1, R)
    x, y = np.array([0.1, 0.0]), np.array([0.0, 0.2])
    exact = math.exp(-float(((x - y) ** 2).sum()) / eps)
    rs = np.array([64, 256, 1024, 4096, 16384])
    rms = []
    for r in rs:
        errs = []
        for s in range(40):
            U = O.draw_anchors(int(r), d, p["sigma"], 1000 + s)
            est = float(np.mean(O.gaussian_phi(x, U, eps, p["q"]) * O.gaussian_phi(y, U, eps, p["q"])))
            errs.append(est / exact - 1)
        rms.append(math.sqrt(np.mean(np.square(errs))))
    slope = np.polyfit(np.log(rs), np.log(rms), 1)[0]
    assert -0.6 < slope < -0.4, (slope, rms)


# ---------------- Anchors: Philox KAT, Box-Muller, moments (reading C5) -------------------
def test_philox_known_answers(golden_dir):
    for row in _read_golden(os.path.join(golden_dir, "philox_kat.txt")):
        vals = [int(v, 16) for v in row]
        out = O.philox4x32_10(np.array([vals[:4]], dtype=np.uint32), vals[4:6])
        assert [int(v) for v in out[0]] == vals[6:10]


def test_box_muller_closed_form():
    """standard_normals applies z=sqrt(-2 ln u1)(cos,sin)(2 pi u2) to the Philox words."""
    w = O.philox_words(3, 5, 99)
    z = O.standard_normals(3, 5, 99)
    for k in range(3):
        for c in range(5):
            p, j = divmod(c, 4)
            pair = j // 2
            w1 = float(w[k, p, 2 * pair]) + 1.0
            w2 = float(w[k, p, 2 * pair + 1])
            rad = math.sqrt(-2.0 * math.log(w1 / 2 ** 32))
            ang = 2 * math.pi * w2 / 2 ** 32
            expect = rad * (math.cos(ang) if j % 2 == 0 else math.sin(ang))
            assert abs(z[k, c] - expect) < 1e-14


def test_anchor_moments_and_prefix():
    z = O.standard_normals(20000, 4, 5)
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.02
    assert abs(np.mean(z ** 4) - 3) < 0.1
    U1 = O.draw_anchors(100, 3, 0.4, 77)
    U2 = O.draw_anchors(300, 3, 0.4, 77)
    assert np.array_equal(U1, U2[:100])          # prefix property
    assert not np.array_equal(U1, O.draw_anchors(100, 3, 0.4, 78))
    assert abs(U2.std() / 0.4 - 1) < 0.05


# ---------------- NEXT f3: arc-cosine perturbed features (reading C21) ---------
@pytest.mark.parametrize("s", [0, 1, 2])
def test_arccos_kernel_identity_quadrature(s):
    """int phi(x,u)^T phi(y,u) d rho(u) = k_s(x,y) + kappa with rho = N(0, sigma^2 I), sigma > 1
    (Lemma decomp-arccos), k_s the closed-form arc-cosine kernel (Cho & Saul).  The map is
    integrated as written (arccos_phi) in polar coordinates, d = 2: Gauss-Legendre over the
    exact arc where both u^T x > 0 and u^T y > 0 (elsewhere the first slot is 0 and only the
    kappa slot contributes kappa * rho-mass), Gauss-Legendre over the radius in [0, 12 sigma]."""
    sigma, kappa = 1.5, 0.1
    x, y = np.array([0.8, 0.3]), np.array([-0.2, 0.9])
    ax, ay = math.atan2(x[1], x[0]), math.atan2(y[1], y[0])
    # u^T x > 0  <=>  angle in (ax - pi/2, ax + pi/2); intersect with the arc for y
    lo, hi = max(ax, ay) - math.pi / 2, min(ax, ay) + math.pi / 2
    tn, tw = np.polynomial.legendre.leggauss(200)
    t = 0.5 * (hi - lo) * tn + 0.5 * (hi + lo)
    tw = 0.5 * (hi - lo) * tw
    rn, rw = np.polynomial.legendre.leggauss(400)
    L = 12 * sigma
    rho = 0.5 * L * (rn + 1)
    rw = 0.5 * L * rw
    T, Rr = np.meshgrid(t, rho, indexing="ij")
    W = np.outer(tw, rw) * Rr * np.exp(-Rr ** 2 / (2 * sigma ** 2)) / (2 * math.pi * sigma ** 2)
    U = np.stack([Rr * np.cos(T), Rr * np.sin(T)], axis=-1)
    first = O.arccos_phi(x, U, sigma, s, kappa)[..., 0] * O.arccos_phi(y, U, sigma, s, kappa)[..., 0]
    integral = float((first * W).sum()) + kappa
    exact = O.arccos_kernel(x, y, s) + kappa
    assert abs(integral / exact - 1) < 1e-10, (integral, exact)


def test_arccos_kernel_closed_form_special_cases():
    """k_0(x,x) = 1, k_1(x,x) = |x|^2, k_1(x,-x) = 0, orthogonal k_1 = |x||y|/pi."""
    x = np.array([0.6, 0.8])
    assert abs(O.arccos_kernel(x, x, 0) - 1.0) < 1e-15
    assert abs(O.arccos_kernel(x, x, 1) - 1.0) < 1e-15
    assert abs(O.arccos_kernel(x, -x, 1)) < 1e-7
    assert abs(O.arccos_kernel(np.array([2.0, 0.0]), np.array([0.0, 3.0]), 1) - 6 / math.pi) < 1e-14


def test_arccos_feature_matrix_and_mc():
    sigma, kappa, s, r = 1.5, 0.1, 1, 20000
    U = O.draw_anchors(r, 3, sigma, 5)
    rng = np.random.default_rng(2)
    X = rng.normal(size=(4, 3)) * 0.5
    F = O.feature_matrix_arccos(X, U, sigma, s, kappa)
    assert F.shape == (r + 1, 4) and np.all(F >= 0)
    Kt = F.T @ F
    for i in range(4):
        for j in range(4):
            exact = O.arccos_kernel(X[i], X[j], s) + kappa
            assert abs(Kt[i, j] / exact - 1) < 0.05
            assert Kt[i, j] >= kappa
