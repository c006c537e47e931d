"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  Tolerances (north_star, BASELINE.json): ROT relative error <= 1e-5; u, v max
relative error <= 1e-4 after the same iteration count; features <= 3e-5 relative (entries
above 1e-30); integer work (Philox words) bit-exact.
"""
import math

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

ROT_TOL = 1e-5
UV_TOL = 1e-4


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
    g = gpu.detach().cpu().double().numpy() if hasattr(gpu, "detach") else np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - ref) / np.abs(ref)))


def _run_gpu(L, prob, T, variant="stream", tol=0.0, want_err=False, ctas_per_sm=0):
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    return L.rot(X, Y, a, b, prob["eps"], prob["r"], prob["seed"], iters=T, tol=tol,
                 variant=variant, want_err=want_err, ctas_per_sm=ctas_per_sm)


def _check_parity(res, ref, rot_tol=ROT_TOL, uv_tol=UV_TOL):
    rot_err = abs(res["rot"] - ref["rot"]) / abs(ref["rot"])
    u_err = _maxrel(res["u"], ref["u"])
    v_err = _maxrel(res["v"], ref["v"])
    print("parity: rot %.3e u %.3e v %.3e" % (rot_err, u_err, v_err))   # shown with pytest -s
    assert rot_err <= rot_tol and u_err <= uv_tol and v_err <= uv_tol, (rot_err, u_err, v_err)
    return rot_err, u_err, v_err


# ------------------------------------------------------------------ a2: generator --------
def test_philox_words_bit_exact(L):
    import torch
    for seed, r, d in [(7058, 100, 2), (2 ** 40 + 17, 333, 5), (0, 4096, 3), (7061, 512, 128)]:
        out = torch.zeros((r, (d + 3) // 4, 4), dtype=torch.int32, device="cuda")
        L.lsk_philox_words(seed, r, d, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, O.philox_words(r, d, seed))


@pytest.mark.parametrize("cfg_key", [1, 2, 3, 4, 5])
def test_anchors_match_oracle(L, cfg_key):
    import torch
    cfg = synth.get_config(cfg_key)
    R = 1.0 + 0.1 * cfg_key
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, R, cfg.anchor_seed)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    ref = O.draw_anchors(cfg.r, cfg.d, O.gaussian_params(cfg.eps, cfg.d, cfg.r, R)["sigma"],
                         cfg.anchor_seed).astype(np.float32)
    got = U.cpu().numpy()
    ulps = np.abs(got.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1, ulps.max()
    assert (ulps == 0).mean() > 0.999


# ------------------------------------------------------------------ a1 auto R ------------
def test_auto_R_matches_oracle(L):
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=5000, m=4000)
    p = L.lsk_feature_params_init(cfg.eps, 2, cfg.r, 0.0, 1, _dev(prob["X"]), _dev(prob["Y"]))
    assert abs(p.R - O.max_norm(prob["X"], prob["Y"])) <= 1e-15 * p.R
    with pytest.raises(L.LskError) as e:
        L.lsk_feature_params_init(cfg.eps, 2, cfg.r, 0.5 * p.R, 1, _dev(prob["X"]), _dev(prob["Y"]))
    assert e.value.status == -3


# ------------------------------------------------------------------ a3: feature map ------
@pytest.mark.parametrize("cfg_key,n", [(1, 500), (2, 3001), (3, 1001), (4, 777), (5, 2049)])
def test_feature_map_matches_oracle(L, cfg_key, n):
    import torch
    cfg = synth.get_config(cfg_key)
    prob = synth.make_problem(cfg, n=n, m=n)
    R = O.max_norm(prob["X"], prob["Y"])
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, R, cfg.anchor_seed)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map(p, U, _dev(prob["X"]), Xi)
    torch.cuda.synchronize()
    prm = O.gaussian_params(cfg.eps, cfg.d, cfg.r, R)     # the oracle's own a1, a2
    Uo = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
    ref = O.feature_matrix(prob["X"], Uo, cfg.eps, prm["q"]).T
    got = Xi.cpu().double().numpy()
    mask = ref > 1e-30
    rel = np.abs(got[mask] - ref[mask]) / ref[mask]
    tol = 3e-5 if cfg.d <= 16 else 1e-4
    assert rel.max() <= tol, rel.max()
    assert np.all(got[~mask] < 1e-29)
    assert np.all(got >= 0)


@pytest.mark.parametrize("d,r,n", [(4, 132, 33), (7, 100, 65), (8, 132, 1), (8, 2052, 127), (9, 100, 128),
                                   (12, 1028, 129), (16, 132, 300), (16, 2052, 257)])
def test_feature_map_direct_shapes(L, d, r, n):
    """The FFMA direct-form map (d <= 16, DESIGN.md §6 K2): both row-block sizes (32 rows for
    d < 8, 128 for d >= 8) with one row, one row short of a block, a full block, one row over;
    the float4 (4 | d) and the scalar anchor loads; threads with no, one and three column groups."""
    import torch
    rng = np.random.default_rng(d * 1000 + r + n)
    X = (rng.normal(size=(n, d)) / math.sqrt(d)).astype(np.float32)
    R = float(np.max(np.linalg.norm(X.astype(np.float64), axis=1)))
    eps = 0.5
    p = L.lsk_feature_params_init(eps, d, r, R, 777)
    U = torch.empty((r, d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.full((n + 1, r), -1.0, dtype=torch.float32, device="cuda")   # guard row
    L.lsk_feature_map(p, U, _dev(X), Xi[:n])
    torch.cuda.synchronize()
    assert bool((Xi[n] == -1.0).all())                     # nothing written past row n
    prm = O.gaussian_params(eps, d, r, R)
    Uo = O.draw_anchors(r, d, prm["sigma"], 777)
    ref = O.feature_matrix(X, Uo, eps, prm["q"]).T
    got = Xi[:n].cpu().double().numpy()
    mask = ref > 1e-30
    assert mask.mean() > 0.5
    rel = np.abs(got[mask] - ref[mask]) / ref[mask]
    assert rel.max() <= 3e-5, rel.max()
    assert np.all(got[~mask] < 1e-29) and np.all(got >= 0)


@pytest.mark.parametrize("d,r,n", [(40, 100, 1000), (100, 640, 129), (127, 256, 300),
                                   (128, 512, 4099), (17, 132, 257), (128, 1000, 513)])
def test_feature_map_tensor_core_shapes(L, d, r, n):
    """The persistent tcgen05 feature map (d <= 128, DESIGN.md §6 K3): partial k chunks
    (d % 32 != 0), the scalar load path (d % 4 != 0), partial anchor blocks (r % 128 != 0),
    more anchor blocks than a cluster of SMs divides evenly (r = 640, 1000), ragged row tiles."""
    import torch
    rng = np.random.default_rng(d * 1000 + r)
    X = (rng.normal(size=(n, d)) / math.sqrt(d)).astype(np.float32)
    R = float(np.max(np.linalg.norm(X.astype(np.float64), axis=1)))
    eps = 1.0
    p = L.lsk_feature_params_init(eps, d, r, R, 4242)
    U = torch.empty((r, d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((n, r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map(p, U, _dev(X), Xi)
    torch.cuda.synchronize()
    prm = O.gaussian_params(eps, d, r, R)
    Uo = O.draw_anchors(r, d, prm["sigma"], 4242)
    ref = O.feature_matrix(X, Uo, eps, prm["q"]).T
    got = Xi.cpu().double().numpy()
    mask = ref > 1e-30
    assert mask.mean() > 0.5
    rel = np.abs(got[mask] - ref[mask]) / ref[mask]
    assert rel.max() <= 1e-4, rel.max()
    assert np.all(got[~mask] < 1e-29) and np.all(got >= 0)


# ------------------------------------------------------------------ Sinkhorn parity ------
def test_config1_full_streaming(L):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=cfg.T)
    res = _run_gpu(L, prob, cfg.T)
    _check_parity(res, ref)
    assert res["report"]["iters"] == cfg.T


def test_config1_full_implicit(L):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=cfg.T)
    res = _run_gpu(L, prob, cfg.T, variant="implicit")
    _check_parity(res, ref)


@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_config2_reduced_ragged(L, variant):
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=4099, m=3907)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=cfg.T)
    res = _run_gpu(L, prob, cfg.T, variant=variant)
    _check_parity(res, ref)


@pytest.mark.parametrize("cfg_key,n,m,T,R,eps", [
    (2, 4099, 3907, 200, 0.0, 0.1),   # team kernel (128,2,2,16), factored exponent (auto R)
    (2, 4099, 3907, 60, 2.0, 0.09),   # expanded exponent: (log2e/eps) R^2 = 64.1 > 60
    (5, 6151, 6143, 40, 0.0, 0.05),   # team kernel (256,1,4,8), factored
    (5, 6151, 6143, 40, 1.6, 0.05),   # expanded: 73.9 > 60
    (1, 500, 500, 200, 0.0, 0.5),
    (1, 500, 500, 200, 5.0, 0.5)])    # expanded: 72.1 > 60
def test_implicit_exponent_forms(L, cfg_key, n, m, T, R, eps):
    """The implicit kernel's two exponent forms (DESIGN.md §6 K5): the factored one
    (F = h_j G_jk, used when (log2e/eps) R^2 <= 60) and the plain expanded one (used above it),
    selected by the data through an explicit R >= max |p| (the map is valid for any such R,
    PAPER.md:385-391), against the oracle with the same R (ragged n, m: tail tiles).  The
    tuning-build alternatives (warp-private, hybrid, pipelined) are checked by
    tests/tools/tuning_parity.py against the tuning library."""
    cfg = synth.get_config(cfg_key)
    if R > 0.0:
        assert 1.4426950408889634 / eps * R * R > 60.0
    prob = synth.make_problem(cfg, n=n, m=m)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], eps, cfg.r, cfg.anchor_seed, T=T,
                R=(R if R > 0.0 else None))
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    res = L.rot(X, Y, a, b, eps, cfg.r, cfg.anchor_seed, iters=T, R=R, variant="implicit")
    _check_parity(res, ref)


def test_config3_reduced_dirichlet(L):
    cfg = synth.get_config(3)
    prob = synth.make_problem(cfg, n=3001, m=2999)
    T = 300
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
    res = _run_gpu(L, prob, T)
    _check_parity(res, ref)


@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_config5_reduced(L, variant):
    cfg = synth.get_config(5)
    prob = synth.make_problem(cfg, n=6151, m=6143)
    T = 60
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
    res = _run_gpu(L, prob, T, variant=variant)
    _check_parity(res, ref)


def test_config4_batched_matches_oracle_and_single(L):
    import torch
    cfg = synth.get_config(4)
    B, T = 3, cfg.T
    bp = synth.make_batched(cfg, batch=B, n=1031, m=1029)
    X, Y, a, b = (_dev(bp[k]) for k in ("X", "Y", "a", "b"))
    R = O.max_norm(bp["X"].reshape(-1, cfg.d), bp["Y"].reshape(-1, cfg.d))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, R, cfg.anchor_seed)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((B, 1031, cfg.r), dtype=torch.float32, device="cuda")
    Ze = torch.empty((B, 1029, cfg.r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map_batched(p, U, X, Xi)
    L.lsk_feature_map_batched(p, U, Y, Ze)
    u = torch.empty((B, 1031), device="cuda")
    v = torch.empty((B, 1029), device="cuda")
    reps = L.lsk_factored_sinkhorn_batched(Xi, Ze, a, b, cfg.eps, L.make_opts(T), u, v)
    rots = L.lsk_rot_value_batched(u, v, a, b, cfg.eps)
    for k in range(B):
        ref = O.rot(bp["X"][k], bp["Y"][k], bp["a"][k], bp["b"][k], cfg.eps, cfg.r,
                    cfg.anchor_seed, T=T, R=R)
        _check_parity(dict(rot=reps[k].rot, u=u[k], v=v[k]), ref)
        assert abs(rots[k] - reps[k].rot) <= 1e-12 * abs(reps[k].rot)
        # batched == single solve of the same pair (same kernels, bit-identical)
        u1 = torch.empty(1031, device="cuda")
        v1 = torch.empty(1029, device="cuda")
        rep1 = L.lsk_factored_sinkhorn(Xi[k], Ze[k], a[k], b[k], cfg.eps, L.make_opts(T), u1, v1)
        assert abs(rep1.rot - reps[k].rot) <= 1e-6 * abs(rep1.rot)
        assert _maxrel(u1, u[k].cpu().double().numpy()) <= 1e-5


# ------------------------------------------------------------------ modes & properties ----
@pytest.mark.parametrize("cfg_key,B,n,m,r", [(1, 5, 500, 487, 100), (5, 3, 2049, 1999, 512)])
def test_implicit_batched_matches_oracle_and_single(L, cfg_key, B, n, m, r):
    """B independent recompute solves in one launch (one CTA per problem): each equals the
    oracle and the single-problem implicit solve of the same pair."""
    import torch
    cfg = synth.get_config(cfg_key)
    probs = [synth.make_problem(cfg, n=n, m=m) if k == 0 else synth.random_small(k, n, m, cfg.d, 0.3)
             for k in range(B)]
    X = _dev(np.stack([q["X"] for q in probs])); Y = _dev(np.stack([q["Y"] for q in probs]))
    a = _dev(np.stack([q["a"] for q in probs])); b = _dev(np.stack([q["b"] for q in probs]))
    R = max(O.max_norm(q["X"], q["Y"]) for q in probs)
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, r, R, cfg.anchor_seed)
    U = torch.empty((r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    T = 60
    u = torch.empty((B, n), device="cuda"); v = torch.empty((B, m), device="cuda")
    reps = L.lsk_factored_sinkhorn_implicit_batched(p, U, X, Y, a, b, L.make_opts(T), u, v)
    for k in range(B):
        q = probs[k]
        ref = O.rot(q["X"], q["Y"], q["a"], q["b"], cfg.eps, r, cfg.anchor_seed, T=T, R=R)
        _check_parity(dict(rot=reps[k].rot, u=u[k], v=v[k]), ref)
        u1 = torch.empty(n, device="cuda"); v1 = torch.empty(m, device="cuda")
        rep1 = L.lsk_factored_sinkhorn_implicit(p, U, X[k], Y[k], a[k], b[k], L.make_opts(T), u1, v1)
        assert abs(rep1.rot - reps[k].rot) <= 1e-6 * abs(rep1.rot)


def test_tolerance_mode(L):
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    tol = 1e-5
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, tol=tol)
    for variant in ("stream", "implicit"):
        res = _run_gpu(L, prob, 500, variant=variant, tol=tol)
        rep = res["report"]
        assert rep["converged"] == 1 and rep["marginal_err"] < tol
        assert abs(rep["iters"] - ref["iters"]) <= 1, (rep["iters"], ref["iters"])
        if rep["iters"] == ref["iters"]:
            _check_parity(res, ref)


def test_fixed_T_marginal_error(L):
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=2000, m=2000)
    T = 7
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T,
                record_err=True)
    res = _run_gpu(L, prob, T, want_err=True)
    err = res["report"]["marginal_err"]
    assert abs(err - ref["errs"][-1]) <= 1e-3 * ref["errs"][-1] + 1e-7, (err, ref["errs"][-1])


def test_deterministic(L):
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=20000, m=20000)
    r1 = _run_gpu(L, prob, 50)
    r2 = _run_gpu(L, prob, 50)
    assert r1["rot"] == r2["rot"]
    assert bool((r1["u"] == r2["u"]).all()) and bool((r1["v"] == r2["v"]).all())


def test_single_point_and_tiny(L):
    """n = m = 1: W_hat = c_theta(x, y) (P9); r = 4 minimal; more CTAs than rows."""
    rng = np.random.default_rng(5)
    x = (rng.normal(size=(1, 3)) * 0.3).astype(np.float32)
    y = (rng.normal(size=(1, 3)) * 0.3).astype(np.float32)
    one = np.ones(1, np.float32)
    for r in (4, 64):
        prob = dict(X=x, Y=y, a=one, b=one, eps=0.7, r=r, seed=5)
        res = _run_gpu(L, prob, 3)
        ref = O.rot(x, y, one, one, 0.7, r, 5, T=3)
        kappa = float(ref["xi"][:, 0] @ ref["zeta"][:, 0])
        assert abs(res["rot"] - (-0.7 * math.log(kappa))) <= 1e-5 * abs(res["rot"]) + 1e-6
    prob = synth.random_small(3, 37, 5, 2)
    prob.update(eps=0.5, r=8, seed=1)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], 0.5, 8, 1, T=40)
    for variant in ("stream", "implicit"):
        _check_parity(_run_gpu(L, prob, 40, variant=variant), ref)


@pytest.mark.parametrize("variant,d,r", [("stream", 2, 8192), ("implicit", 8, 4096),
                                         ("implicit", 3, 4096), ("stream", 16, 2048)])
def test_largest_supported_shapes(L, variant, d, r):
    """The largest r each kernel instantiates (stream: 8 float4 groups per consumer thread,
    r = 8192; implicit: r = 4096 at the largest d = 8 and at d = 3) on a ragged small n."""
    rng = np.random.default_rng(11)
    n, m = 1031, 997
    x = rng.normal(0.0, 0.3, size=(n, d))
    y = rng.normal(0.2, 0.3, size=(m, d))
    a = rng.uniform(0.5, 1.5, n); a /= a.sum()
    b = rng.uniform(0.5, 1.5, m); b /= b.sum()
    prob = dict(X=x.astype(np.float32), Y=y.astype(np.float32), a=a.astype(np.float32),
                b=b.astype(np.float32), eps=0.5, r=r, seed=13)
    T = 30
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], 0.5, r, 13, T=T)
    _check_parity(_run_gpu(L, prob, T, variant=variant), ref)


def test_invalid_arguments_fail_loudly(L):
    """Empty inputs, r not a multiple of 4, eps <= 0 and d beyond a kernel's range are
    rejected with the documented status codes (no silent fallback)."""
    import torch
    X = torch.zeros((0, 2), device="cuda")
    Y = torch.zeros((5, 2), device="cuda")
    a = torch.ones(0, device="cuda")
    b = torch.ones(5, device="cuda") / 5
    with pytest.raises(L.LskError) as e:
        L.rot(X, Y, a, b, 0.5, 8, 1, iters=3)
    assert e.value.status in (-1,)
    Xn = torch.rand((4, 2), device="cuda")
    an = torch.ones(4, device="cuda") / 4
    for r in (6, 0):
        with pytest.raises(L.LskError) as e:
            L.rot(Xn, Y, an, b, 0.5, r, 1, iters=3)
        assert e.value.status == -1
    with pytest.raises(L.LskError) as e:
        L.rot(Xn, Y, an, b, -1.0, 8, 1, iters=3)
    assert e.value.status == -1
    X9 = torch.rand((4, 9), device="cuda") * 0.1
    Y9 = torch.rand((5, 9), device="cuda") * 0.1
    with pytest.raises(L.LskError) as e:
        L.rot(X9, Y9, an, b, 0.5, 8, 1, iters=3, variant="implicit")
    assert e.value.status == -2   # LSK_EDIM: the implicit kernels take d <= 8


def test_rank_one_full_size_closed_form(L):
    """Config 5 at FULL size with identical points: K_theta = kappa 11^T, so one loop gives
    W = eps(sum a ln a + sum b ln b - (sum b) ln kappa + (sum a - sum b) ln n
    - (sum a) ln sum b) (P11).  Exercises every row of the full launch configuration."""
    cfg = synth.get_config(5)
    prob = synth.make_problem(cfg, identical_points=True)
    res = _run_gpu(L, prob, 2, variant="implicit")
    prm = O.gaussian_params(cfg.eps, cfg.d, cfg.r, O.max_norm(prob["X"], prob["Y"]))
    U = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)   # the oracle's own anchors
    q = prm["q"]
    xi0 = O.feature_entries_scaled(prob["X"][:1], U, cfg.eps, q, cfg.r, np.zeros(cfg.r, int), np.arange(cfg.r))
    ze0 = O.feature_entries_scaled(prob["Y"][:1], U, cfg.eps, q, cfg.r, np.zeros(cfg.r, int), np.arange(cfg.r))
    kappa = float(xi0 @ ze0)
    a, b = prob["a"].astype(np.float64), prob["b"].astype(np.float64)
    n = len(a)
    expect = cfg.eps * (a @ np.log(a) + b @ np.log(b) - b.sum() * math.log(kappa)
                        + (a.sum() - b.sum()) * math.log(n) - a.sum() * math.log(b.sum()))
    assert abs(res["rot"] - expect) <= 1e-5 * abs(expect), (res["rot"], expect)


def test_rot_value_matches_oracle(L):
    rng = np.random.default_rng(11)
    n, m = 100003, 77777
    u = rng.uniform(0.1, 10, n).astype(np.float32)
    v = rng.uniform(0.1, 10, m).astype(np.float32)
    a = rng.uniform(0.5, 1.5, n).astype(np.float32)
    b = rng.uniform(0.5, 1.5, m).astype(np.float32)
    got = L.lsk_rot_value(_dev(u), _dev(v), _dev(a), _dev(b), 0.3)
    ref = O.dual_estimate(u.astype(np.float64), v.astype(np.float64), a, b, 0.3)
    assert abs(got - ref) <= 1e-12 * abs(ref)


def test_host_entry_point_matches_device_path(L):
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=3000, m=3000)
    dev = _run_gpu(L, prob, 100)
    u = np.empty(3000, np.float32)
    v = np.empty(3000, np.float32)
    rep = L.lsk_rot_host(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r,
                         cfg.anchor_seed, L.make_opts(100), variant=1, u_out=u, v_out=v)
    assert rep.rot == dev["rot"]
    assert np.array_equal(u, dev["u"].cpu().numpy())


@pytest.mark.slow
def test_config2_full_size(L):
    """Config 2 at its full size (n=m=40000, r=1000, T=500) in the bench's launch config."""
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=cfg.T)
    for variant in ("stream", "implicit"):
        _check_parity(_run_gpu(L, prob, cfg.T, variant=variant), ref)


# ------------------------------------------------------------------ multi-GPU code path ---
@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_nccl_multilaunch_one_rank(L, variant):
    """The row-sharded multi-GPU path (one pass per launch, NCCL fp64 all-reduce of the
    r-vector between launches, all-reduced read-out) exercised on one GPU with a 1-rank NCCL
    communicator: same result as the single-launch path and the oracle."""
    import torch
    uid = L.lsk_comm_get_unique_id()
    comm = L.lsk_comm_init(1, 0, uid, torch.cuda.current_device())
    try:
        cfg = synth.get_config(2)
        prob = synth.make_problem(cfg, n=3001, m=2999)
        T = 40
        ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
        X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
        res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant=variant, comm=comm)
        _check_parity(res, ref)
        single = _run_gpu(L, prob, T, variant=variant)
        assert abs(res["rot"] - single["rot"]) <= 1e-6 * abs(single["rot"])
        # tolerance mode (early stop inside the multi-launch sequence)
        tol = 1e-4
        res_t = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, max_iters=300, tol=tol,
                      variant=variant, comm=comm)
        ref_t = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, tol=tol)
        assert res_t["report"]["converged"] == 1 and res_t["report"]["marginal_err"] < tol
        assert abs(res_t["report"]["iters"] - ref_t["iters"]) <= 1
    finally:
        L.lsk_comm_destroy(comm)


@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_p2p_exchange_one_rank(L, variant):
    """The in-kernel cross-GPU exchange (lsk_comm_enable_p2p: one persistent launch per GPU,
    every column's all-rank total formed by its owner CTA through the peer inboxes) on one GPU
    with a 1-rank communicator: the whole protocol runs (store to every inbox, sentinel polls,
    rank-order sum, re-arm) and, with one rank, the total is 0.0 + local — so u, v and W_hat are
    bit-identical to the single-GPU launch, in fixed-T and tolerance mode, solve after solve."""
    import torch
    uid = L.lsk_comm_get_unique_id()
    comm = L.lsk_comm_init(1, 0, uid, torch.cuda.current_device())
    try:
        L.lsk_comm_enable_p2p(comm, 1024)
        cfg = synth.get_config(2)
        prob = synth.make_problem(cfg, n=3001, m=2999)
        X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
        for T in (40, 41):   # both parities of the last pass
            res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant=variant,
                        comm=comm)
            single = _run_gpu(L, prob, T, variant=variant)
            assert torch.equal(res["u"], single["u"]) and torch.equal(res["v"], single["v"])
            assert res["rot"] == single["rot"]
        res_t = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, max_iters=300, tol=1e-4,
                      variant=variant, comm=comm)
        single_t = _run_gpu(L, prob, 300, variant=variant, tol=1e-4)
        assert res_t["report"]["iters"] == single_t["report"]["iters"]
        assert res_t["rot"] == single_t["rot"]
    finally:
        L.lsk_comm_destroy(comm)


def test_smoke_entry_point(L):
    import importlib, sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    ge = importlib.import_module("__graft_entry__")
    ge.smoke()


# ------------------------------------------------------------------ NEXT f1: divergence ----
@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_sinkhorn_divergence(L, variant):
    """W_bar(mu,nu) = W(mu,nu) - (W(mu,mu) + W(nu,nu))/2 vs the oracle; each W to
    1e-5 relative; W_bar (a difference) to 1e-5 of the sum of magnitudes; W_bar(mu,mu) = 0
    exactly (the three solves are the same computation)."""
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=3001, m=2503)
    T = 200
    ref = O.sinkhorn_divergence(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r,
                                cfg.anchor_seed, T=T)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    got = L.sinkhorn_divergence(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T,
                                variant=variant)
    for k in ("xy", "xx", "yy"):
        assert abs(got[k] - ref[k]) <= ROT_TOL * abs(ref[k]), (k, got[k], ref[k])
    scale = abs(ref["xy"]) + abs(ref["xx"]) + abs(ref["yy"])
    assert abs(got["div"] - ref["div"]) <= ROT_TOL * scale, (got["div"], ref["div"])
    same = L.sinkhorn_divergence(X, X, a, a, cfg.eps, cfg.r, cfg.anchor_seed, iters=50,
                                 variant=variant)
    assert same["div"] == 0.0


# ------------------------------------------------------------------ NEXT f2: gradients -----
@pytest.mark.parametrize("cfg_key,n,m", [(1, 500, 500), (2, 2049, 1531), (5, 3001, 2999)])
def test_envelope_gradients(L, cfg_key, n, m):
    """dW/dX, dW/dY, dW/dU from the GPU solve vs the oracle's chain rule
    (itself pinned by finite differences) on the oracle's own scalings after the same T;
    max abs error <= 2e-4 of the largest gradient entry (sums with sign cancellation)."""
    cfg = synth.get_config(cfg_key)
    prob = synth.make_problem(cfg, n=n, m=m)
    T = 100
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
    gref = O.envelope_gradients(prob["X"], prob["Y"], ref["U"], ref["xi"], ref["zeta"], ref["u"],
                                ref["v"], cfg.eps, ref["params"]["q"])
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T)
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    g = L.lsk_rot_gradient(p, res["U"], X, Y, res["Xi"], res["Zeta"], res["u"], res["v"])
    for k, key in (("X", "gX"), ("Y", "gY"), ("U", "gU")):
        got = g[k].cpu().double().numpy()
        want = gref[key]
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err <= 2e-4, (k, err)


# ------------------------------------------------------------------ NEXT f3: arc-cosine ----
@pytest.mark.parametrize("d,s_deg,n", [(3, 1, 1031), (2, 0, 777), (16, 2, 513), (128, 1, 700)])
def test_arccos_features_and_solve(L, d, s_deg, n):
    """Arc-cosine features (Lemma decomp-arccos) vs the oracle entry by entry,
    then Alg. 1 on those factors (rank r + 1, padded to r + 4) vs the oracle's Sinkhorn."""
    import torch
    r, sigma, kappa, eps, T = 256, 1.5, 0.1, 0.5, 150
    rng = np.random.default_rng(100 + d)
    X = (rng.normal(size=(n, d)) / math.sqrt(d)).astype(np.float32)
    Y = (rng.normal(0.2, 1.0, size=(n + 7, d)) / math.sqrt(d)).astype(np.float32)
    a = np.full(n, 1.0 / n, np.float32)
    b = np.full(n + 7, 1.0 / (n + 7), np.float32)
    p = L.arccos_params(d, r, sigma, 77, eps)
    U = torch.empty((r, d), device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((n, r + 4), device="cuda")
    Ze = torch.empty((n + 7, r + 4), device="cuda")
    L.lsk_feature_map_arccos(p, s_deg, kappa, U, _dev(X), Xi)
    L.lsk_feature_map_arccos(p, s_deg, kappa, U, _dev(Y), Ze)
    Uo = O.draw_anchors(r, d, sigma, 77)
    fx = O.feature_matrix_arccos(X, Uo, sigma, s_deg, kappa)       # (r+1) x n, paper layout
    fy = O.feature_matrix_arccos(Y, Uo, sigma, s_deg, kappa)
    got = Xi.cpu().double().numpy()
    assert np.all(got[:, r + 1:] == 0)
    ref = fx.T
    tol = 1e-5 if d <= 16 else 2e-4
    err = np.abs(got[:, :r + 1] - ref) / (np.abs(ref) + 1e-3 * ref.max())
    assert err.max() <= tol, err.max()
    u = torch.empty(n, device="cuda")
    v = torch.empty(n + 7, device="cuda")
    rep = L.lsk_factored_sinkhorn(Xi, Ze, _dev(a), _dev(b), eps, L.make_opts(T), u, v)
    sol = O.sinkhorn_factored(fx, fy, a, b, T=T)
    rot_ref = O.dual_estimate(sol["u"], sol["v"], a, b, eps)
    assert abs(rep.rot - rot_ref) <= ROT_TOL * abs(rot_ref)
    assert _maxrel(u, sol["u"]) <= UV_TOL and _maxrel(v, sol["v"]) <= UV_TOL


# ------------------------------------------------------------------ NEXT f4: Alg. 2 -------
def _accel_pair(L, cfg_key, n, m, T):
    import torch
    cfg = synth.get_config(cfg_key)
    prob = synth.make_problem(cfg, n=n, m=m)
    R = O.max_norm(prob["X"], prob["Y"])
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, R, cfg.anchor_seed)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
    Ze = torch.empty((m, cfg.r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map(p, U, _dev(prob["X"]), Xi)
    L.lsk_feature_map(p, U, _dev(prob["Y"]), Ze)
    gpu = L.lsk_accelerated_sinkhorn(Xi, Ze, _dev(prob["a"]), _dev(prob["b"]), cfg.eps, T,
                                     traces=True)
    prm = O.gaussian_params(cfg.eps, cfg.d, cfg.r, R)      # the oracle's own a1, a2
    Uo = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
    xi = O.feature_matrix(prob["X"], Uo, cfg.eps, prm["q"])
    zeta = O.feature_matrix(prob["Y"], Uo, cfg.eps, prm["q"])
    ref = O.accelerated_sinkhorn_factored(xi, zeta, prob["a"], prob["b"], cfg.eps, T=T)
    return gpu, ref, (xi, zeta, prob, cfg)


@pytest.mark.parametrize("cfg_key,n,m,T", [(1, 500, 500, 60), (2, 4099, 3907, 60),
                                           (3, 3001, 2999, 40)])
def test_accelerated_matches_oracle(L, cfg_key, n, m, T):
    """Alg. 2 through the C ABI vs the oracle on the same seeded inputs.  The line search's
    decisions (block i_k = argmax |grad_i phi|, accepted L) are floating-point decisions taken
    on gradients g = e^lambda o K e^lambda' / c - a: fp32 factors perturb each entry by
    ~1e-7 a_i, i.e. |g|^2 by ~2e-7 |a| |g| — they must agree exactly while the oracle's margin
    |n1 - n2| / (n1 + n2) exceeds 100x that noise; beyond the first such near-tie the paths
    may part, and only F (whose changes are O(|g|^2) there) is compared.  F per iteration
    within 1e-5; the dual point (gauge-fixed: eta1 - eta1[0], eta2 + eta1[0]) within 1e-4
    when no near-tie occurred."""
    gpu, ref, (xi, zeta, prob, cfg) = _accel_pair(L, cfg_key, n, m, T)
    assert gpu["iters"] == T
    g = ref["grad_norms"]
    a = prob["a"].astype(np.float64); a /= a.sum()
    b = prob["b"].astype(np.float64); b /= b.sum()
    noise = 2e-7 * np.maximum(np.linalg.norm(a) / np.sqrt(g[:, 0]), np.linalg.norm(b) / np.sqrt(g[:, 1]))
    ties = np.nonzero(np.abs(g[:, 0] - g[:, 1]) <= 100 * noise * (g[:, 0] + g[:, 1]))[0]
    k = int(ties[0]) if ties.size else T
    assert k >= 5, "instance too close to a tie from the start"
    assert np.array_equal(gpu["blocks"][:k], ref["blocks"][:k])
    assert np.array_equal(gpu["L_trace"][:k], ref["L_trace"][:k])
    assert np.max(np.abs(gpu["F_trace"] - ref["F_trace"]) / np.abs(ref["F_trace"])) <= 1e-5
    if k == T:
        e1 = gpu["eta1"].cpu().numpy()
        e2 = gpu["eta2"].cpu().numpy()
        g0, r0 = e1[0], ref["eta1"][0]
        assert np.max(np.abs((e1 - g0) - (ref["eta1"] - r0))) <= 1e-4
        assert np.max(np.abs((e2 + g0) - (ref["eta2"] + r0))) <= 1e-4


def test_accelerated_converges_to_alg1(L):
    """Tolerance mode on config 1: the accelerated solver's F reaches Alg. 1's converged
    value (oracle, fp64) to 1e-5 relative, and stops on the plan-marginal tolerance."""
    import torch
    gpu, ref, (xi, zeta, prob, cfg) = _accel_pair(L, 1, 500, 500, 5)
    a = prob["a"].astype(np.float64); a /= a.sum()
    b = prob["b"].astype(np.float64); b /= b.sum()
    s1 = O.sinkhorn_factored(xi, zeta, a, b, tol=1e-13, max_iter=100000)
    W = O.dual_estimate(s1["u"], s1["v"], a, b, cfg.eps)
    Xi = torch.from_numpy(xi.T.astype(np.float32).copy()).cuda()
    Ze = torch.from_numpy(zeta.T.astype(np.float32).copy()).cuda()
    res = L.lsk_accelerated_sinkhorn(Xi, Ze, _dev(prob["a"]), _dev(prob["b"]), cfg.eps, 20000,
                                     tol=1e-4)
    assert res["converged"] == 1 and res["plan_err"] < 1e-4
    assert abs(res["F"] - W) <= 1e-5 * abs(W), (res["F"], W)


# ------------------------------------------------------------------ NEXT f4: stabilisation -
@pytest.mark.parametrize("eps", [0.1, 0.01])
def test_stabilized_feature_map_matches_oracle(L, eps):
    """Row-normalised features and their fp64 log offsets (reading C30) vs the oracle."""
    import torch
    cfg = synth.get_config(2)
    n = 3001
    prob = synth.make_problem(cfg, n=n, m=n)
    R = O.max_norm(prob["X"], prob["Y"])
    p = L.lsk_feature_params_init(eps, cfg.d, cfg.r, R, cfg.anchor_seed)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
    A = torch.empty(n, dtype=torch.float64, device="cuda")
    L.lsk_feature_map_stabilized(p, U, _dev(prob["X"]), Xi, A)
    torch.cuda.synchronize()
    prm = O.gaussian_params(eps, cfg.d, cfg.r, R)
    ref, Aref = O.feature_matrix_stabilized(
        prob["X"], O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed), eps, prm["q"])
    got = Xi.cpu().double().numpy()
    assert np.all(got.max(axis=1) == 1.0)                      # every row's largest entry
    mask = ref.T > 1e-30
    rel = np.abs(got[mask] - ref.T[mask]) / ref.T[mask]
    assert rel.max() <= 3e-5, rel.max()
    assert np.max(np.abs(A.cpu().numpy() - Aref) / np.maximum(1.0, np.abs(Aref))) <= 1e-5


@pytest.mark.parametrize("variant", ["stream", "implicit"])
@pytest.mark.parametrize("eps", [0.02, 0.01])
def test_stabilized_small_eps_rot(L, eps, variant):
    """At eps where the plain fp32 paths break down (0.01; the implicit one already at 0.02),
    the stabilised paths (stream: row-normalised stored factors; implicit: per-row exponent
    shift inside the kernel) match the fp64 oracle: W_hat within 1e-5 of the plain oracle's
    value, and the scalings of the normalised problem within 1e-4 of the oracle run of the same
    formulation (C30: Alg. 1 on the row-normalised factors from u~ = 1)."""
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=4000, m=3999)
    T = 300
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], eps, cfg.r, cfg.anchor_seed, T=T)
    res = _run_gpu_stab(L, prob, eps, T, variant)
    assert abs(res["rot"] - ref["rot"]) <= 1e-5 * abs(ref["rot"]), (res["rot"], ref["rot"])
    R = O.max_norm(prob["X"], prob["Y"])
    prm = O.gaussian_params(eps, cfg.d, cfg.r, R)
    Uo = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
    xt, A = O.feature_matrix_stabilized(prob["X"], Uo, eps, prm["q"])
    zt, B = O.feature_matrix_stabilized(prob["Y"], Uo, eps, prm["q"])
    s = O.sinkhorn_factored(xt, zt, prob["a"], prob["b"], T=T)
    assert _maxrel(res["u"], s["u"]) <= 1e-4 and _maxrel(res["v"], s["v"]) <= 1e-4


def _run_gpu_stab(L, prob, eps, T, variant="stream"):
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    cfg = synth.get_config(2)
    return L.rot(X, Y, a, b, eps, cfg.r, cfg.anchor_seed, iters=T, stabilize=True,
                 variant=variant)
