"""GPU parity of the resident small-problem kernel (lsk_resident.cu, DESIGN.md §6 K10): both
factors in the shared memory of one thread-block cluster of G = 1, 2, 4 or 8 CTAs.  Every case
is compared with the fp64 oracle (PAPER.md:232-244 Alg. 1, :261 read-out) at the north_star
tolerances (ROT <= 1e-5 relative, u and v <= 1e-4), and with the persistent grid kernels
(LSK_SOLVE_NO_RESIDENT) on the same inputs."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

ROT_TOL = 1e-5
UV_TOL = 1e-4
EWEIGHTS, EBREAKDOWN = -4, -5


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2006_07057_b200 as lib
    return lib


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _maxrel(gpu, ref):
    g = gpu.detach().cpu().double().numpy()
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - ref) / np.abs(ref)))


def _run(L, prob, T, variant="stream", tol=0.0, want_err=False, resident=True):
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    return L.rot(X, Y, a, b, prob["eps"], prob["r"], prob["seed"], iters=T, tol=tol,
                 variant=variant, want_err=want_err, resident=resident)


def _check(res, ref):
    rot_err = abs(res["rot"] - ref["rot"]) / abs(ref["rot"])
    u_err = _maxrel(res["u"], ref["u"])
    v_err = _maxrel(res["v"], ref["v"])
    assert rot_err <= ROT_TOL and u_err <= UV_TOL and v_err <= UV_TOL, (rot_err, u_err, v_err)


def _problem(n, m, d, r, eps, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, 0.3, size=(n, d))
    y = rng.normal(0.2, 0.4, size=(m, d))
    a = rng.uniform(0.5, 1.5, n); a /= a.sum()
    b = rng.uniform(0.5, 1.5, m); b /= b.sum()
    return dict(X=x.astype(np.float32), Y=y.astype(np.float32), a=a.astype(np.float32),
                b=b.astype(np.float32), eps=eps, r=r, seed=seed)


@pytest.mark.parametrize("n,m,r,G", [(500, 500, 100, 8), (37, 53, 8, 1), (100, 97, 100, 2),
                                     (150, 140, 100, 4), (300, 257, 100, 8), (1031, 997, 128, 8),
                                     (600, 650, 256, 8), (200, 150, 512, 8), (1000, 900, 196, 8),
                                     (1, 1, 4, 1), (701, 803, 256, 0), (1300, 1300, 196, 0),
                                     (40000, 40000, 1000, 0), (500, 500, 1024, 0),
                                     (20000, 20000, 100, 0)])
def test_resident_plan(L, n, m, r, G):
    """The planner: the smallest cluster that holds both factors (<= 227 KB of shared memory per
    CTA), grown while half the warps keep a row batch; 0 (grid kernels) past r = 512 or 8 CTAs."""
    assert L.lsk_resident_plan(n, m, r) == G


@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_config1_full_resident_vs_oracle_and_grid(L, variant):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=cfg.T)
    res = _run(L, prob, cfg.T, variant=variant)
    _check(res, ref)
    assert res["report"]["iters"] == cfg.T
    grid = _run(L, prob, cfg.T, variant=variant, resident=False)
    _check(grid, ref)
    assert abs(res["rot"] - grid["rot"]) <= 2e-6 * abs(grid["rot"])


# (n, m, d, r): cluster sizes 1 (tiny), 2, 4, 8 (row counts), ragged n != m, r with 1, 2
# and 4 float4 column groups per lane (r <= 128, <= 256, <= 512)
@pytest.mark.parametrize("n,m,d,r", [
    (37, 53, 2, 8),        # G = 1, padded lanes
    (100, 97, 3, 100),     # G = 2
    (150, 140, 2, 100),    # G = 4
    (300, 257, 2, 100),    # G = 8, 33-38 rows per CTA
    (1031, 997, 2, 128),   # G = 8, every lane one group
    (600, 650, 3, 256),    # NG = 2
    (200, 150, 2, 512),    # NG = 4, the largest r (needs G = 8)
    (1000, 900, 2, 196),   # the factors need G = 8 (1.5 MB)
])
def test_resident_shapes_vs_oracle(L, n, m, d, r):
    prob = _problem(n, m, d, r, 0.5, 17 + n)
    T = 60
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], prob["eps"], r, prob["seed"], T=T)
    for variant in ("stream", "implicit"):
        _check(_run(L, prob, T, variant=variant), ref)


def test_resident_tolerance_mode_and_error(L):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    tol = 1e-5
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, tol=tol)
    for variant in ("stream", "implicit"):
        res = _run(L, prob, 500, variant=variant, tol=tol)
        rep = res["report"]
        assert rep["converged"] == 1 and rep["marginal_err"] < tol
        assert abs(rep["iters"] - ref["iters"]) <= 1, (rep["iters"], ref["iters"])
        if rep["iters"] == ref["iters"]:
            _check(res, ref)
    T = 7
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T,
                record_err=True)
    res = _run(L, prob, T, want_err=True)
    err = res["report"]["marginal_err"]
    assert abs(err - ref["errs"][-1]) <= 1e-3 * ref["errs"][-1] + 1e-7, (err, ref["errs"][-1])
    # at T = 7 the error (~6e-8) is at the fp32 rounding level of v_j t_j - b_j: the grid
    # kernels agree with it to the oracle tolerance, not bit for bit
    grid = _run(L, prob, T, want_err=True, resident=False)
    assert abs(err - grid["report"]["marginal_err"]) <= 1e-3 * err + 1e-7


def test_resident_deterministic(L):
    prob = _problem(1031, 997, 2, 128, 0.5, 3)
    r1 = _run(L, prob, 40)
    r2 = _run(L, prob, 40)
    assert r1["rot"] == r2["rot"]
    assert bool((r1["u"] == r2["u"]).all()) and bool((r1["v"] == r2["v"]).all())


def test_resident_bad_weights_and_breakdown(L):
    import torch
    prob = _problem(300, 257, 2, 100, 0.5, 9)
    bad = dict(prob)
    bad["a"] = prob["a"].copy()
    bad["a"][17] = 0.0
    with pytest.raises(L.LskError) as ei:
        _run(L, bad, 10)
    assert ei.value.status == EWEIGHTS
    # report-less solve: the sticky status carries it to the next synchronising call
    X, Y, a, b = (_dev(bad[k]) for k in ("X", "Y", "a", "b"))
    p = L.lsk_feature_params_init(0.5, 2, 100, 0.0, 9, X, Y)
    U = torch.empty((100, 2), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(300, device="cuda"); v = torch.empty(257, device="cuda")
    L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, L.make_opts(10), u, v, report=False)
    with pytest.raises(L.LskError) as ei:
        L.lsk_stream_status()
    assert ei.value.status == EWEIGHTS
    # far-apart clouds at small eps: the features underflow, a row dot is 0 -> breakdown
    far = _problem(300, 257, 2, 100, 0.5, 9)
    far["Y"] = (far["Y"] + 40.0).astype(np.float32)
    far["eps"] = 0.05
    with pytest.raises(L.LskError) as ei:
        _run(L, far, 10)
    assert ei.value.status in (EBREAKDOWN, EWEIGHTS)


@pytest.mark.parametrize("B,n,m,r", [(7, 300, 257, 100), (64, 500, 500, 100)])
def test_resident_batched(L, B, n, m, r):
    """Batches of small problems: one cluster per problem (B x G CTAs; 64 x 8 = 512 CTAs is more
    than one wave of clusters).  Both batched APIs against the oracle (a sample of the problems
    for B = 64) and against the grid kernels for every problem."""
    import torch
    rng = np.random.default_rng(B)
    d, eps, seed = 2, 0.5, 21
    X = (rng.normal(0.0, 0.3, size=(B, n, d))).astype(np.float32)
    Y = (rng.normal(0.2, 0.4, size=(B, m, d))).astype(np.float32)
    a = rng.uniform(0.5, 1.5, size=(B, n)); a /= a.sum(1, keepdims=True)
    b = rng.uniform(0.5, 1.5, size=(B, m)); b /= b.sum(1, keepdims=True)
    a, b = a.astype(np.float32), b.astype(np.float32)
    R = max(O.max_norm(X[q], Y[q]) for q in range(B))
    Xd, Yd, ad, bd = _dev(X), _dev(Y), _dev(a), _dev(b)
    p = L.lsk_feature_params_init(eps, d, r, R, seed)
    U = torch.empty((r, d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    T = 50
    out = {}
    for res in (True, False):
        u = torch.empty((B, n), dtype=torch.float32, device="cuda")
        v = torch.empty((B, m), dtype=torch.float32, device="cuda")
        reps = L.lsk_factored_sinkhorn_implicit_batched(p, U, Xd, Yd, ad, bd,
                                                        L.make_opts(T, resident=res), u, v)
        Xi = torch.empty((B, n, r), dtype=torch.float32, device="cuda")
        Ze = torch.empty((B, m, r), dtype=torch.float32, device="cuda")
        L.lsk_feature_map_batched(p, U, Xd, Xi)
        L.lsk_feature_map_batched(p, U, Yd, Ze)
        u2 = torch.empty((B, n), dtype=torch.float32, device="cuda")
        v2 = torch.empty((B, m), dtype=torch.float32, device="cuda")
        reps2 = L.lsk_factored_sinkhorn_batched(Xi, Ze, ad, bd, eps, L.make_opts(T, resident=res),
                                                u2, v2)
        out[res] = (u, v, reps, u2, v2, reps2)
    sample = range(B) if B <= 8 else (0, 1, B // 2, B - 1)
    for q in sample:
        ref = O.rot(X[q], Y[q], a[q], b[q], eps, r, seed, T=T, R=R)
        for (u, v, reps) in ((out[True][0], out[True][1], out[True][2]),
                             (out[True][3], out[True][4], out[True][5])):
            rot_err = abs(reps[q].rot - ref["rot"]) / abs(ref["rot"])
            assert rot_err <= ROT_TOL, rot_err
            assert _maxrel(u[q], ref["u"]) <= UV_TOL and _maxrel(v[q], ref["v"]) <= UV_TOL
    for k in (0, 3):   # resident vs grid, every problem
        for q in range(B):
            g, h = out[False][k + 2][q].rot, out[True][k + 2][q].rot
            assert abs(g - h) <= 2e-6 * abs(g), (q, g, h)
            assert out[True][k + 2][q].iters == T


@pytest.mark.parametrize("n,m", [(16, 7), (17, 40), (40, 90), (300, 129), (1, 33)])
def test_two_team_pingpong_tile_counts(L, n, m):
    """The implicit grid kernel's two-team configuration (32 < r/4 <= 256, d <= 3) with its
    ping-pong hand-over between the teams (DESIGN.md §6 K5): shapes whose CTAs hold 0, 1, 2 or 3
    tiles of each side, i.e. equal and unequal team tile counts and a team with no tile, so the
    end-of-pass balancing of the hand-over barriers is exercised on both sides.  Forced onto the
    grid kernels (these shapes would otherwise run resident) and compared with the oracle."""
    prob = _problem(n, m, 2, 256, 0.5, 5 + n + m)
    T = 30
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], prob["eps"], 256, prob["seed"], T=T)
    _check(_run(L, prob, T, variant="implicit", resident=False), ref)
    res_t = _run(L, prob, 400, variant="implicit", tol=1e-6, resident=False)
    ref_t = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], prob["eps"], 256, prob["seed"], tol=1e-6)
    assert res_t["report"]["converged"] == 1
    assert abs(res_t["report"]["iters"] - ref_t["iters"]) <= 1
