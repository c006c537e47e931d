"""GPU tests of the C-ABI boundary's error behaviour and launch planning (include/lsk.h):
weight validation (LSK_EWEIGHTS), breakdown surfaced without a report (sticky stream status),
the multi-launch (NCCL) path's early stop with many rows per CTA, the solve workspace sized
after planning, and batched solves whose groups loop over several problems — each checked
against the fp64 oracle where a value is produced."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

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
    return float(np.max(np.abs(g - ref) / np.abs(ref)))


def _parity(res_u, res_v, rot, ref, rot_tol=1e-5, uv_tol=1e-4):
    assert abs(rot - ref["rot"]) <= rot_tol * abs(ref["rot"])
    assert _maxrel(res_u, ref["u"]) <= uv_tol and _maxrel(res_v, ref["v"]) <= uv_tol


# ------------------------------------------------------------- weights -----
@pytest.mark.parametrize("variant", ["stream", "implicit"])
@pytest.mark.parametrize("bad", [0.0, -1e-3, float("nan"), float("inf")])
@pytest.mark.parametrize("side", ["a", "b"])
def test_bad_weight_raises_eweights(L, variant, bad, side):
    """mu, nu are probability measures with positive masses: a weight that is
    not finite and > 0 fails the solve with LSK_EWEIGHTS — from the report when one is asked
    for, else from the stream's sticky status (lsk_stream_status, lsk_rot_value)."""
    cfg = synth.get_config(1)
    prob = synth.make_problem(cfg)
    w = prob[side].copy()
    w[137] = bad
    prob[side] = w
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    with pytest.raises(L.LskError) as e:
        L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=20, variant=variant)
    assert e.value.status == EWEIGHTS
    L.lsk_stream_status()   # the report consumed it: clean again
    # report-less: the solve returns asynchronously, the sticky status carries the error
    p = L.lsk_feature_params_init(cfg.eps, 2, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    import torch
    U = torch.empty((cfg.r, 2), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(500, dtype=torch.float32, device="cuda")
    v = torch.empty(500, dtype=torch.float32, device="cuda")
    L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, L.make_opts(20), u, v, report=False)
    with pytest.raises(L.LskError) as e:
        L.lsk_stream_status()
    assert e.value.status == EWEIGHTS
    L.lsk_stream_status()   # cleared
    L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, L.make_opts(20), u, v, report=False)
    with pytest.raises(L.LskError) as e:
        L.lsk_rot_value(u, v, a, b, cfg.eps)
    assert e.value.status == EWEIGHTS


def test_bad_weight_batched(L):
    """Batched: the bad problem's report makes the call fail; the other problems' reports and
    scalings are still written."""
    import torch
    cfg = synth.get_config(1)
    bp = synth.make_batched(synth.get_config(4, d=2), batch=3, n=500, m=500)
    bp["b"][1, 7] = 0.0
    p = L.lsk_feature_params_init(0.5, 2, 100, 0.0, 11, _dev(bp["X"].reshape(-1, 2)),
                                  _dev(bp["Y"].reshape(-1, 2)))
    U = torch.empty((100, 2), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    X, Y, a, b = (_dev(bp[k]) for k in ("X", "Y", "a", "b"))
    u = torch.empty((3, 500), dtype=torch.float32, device="cuda")
    v = torch.empty((3, 500), dtype=torch.float32, device="cuda")
    with pytest.raises(L.LskError) as e:
        L.lsk_factored_sinkhorn_implicit_batched(p, U, X, Y, a, b, L.make_opts(10), u, v)
    assert e.value.status == EWEIGHTS
    L.lsk_stream_status()


# ------------------------------------------------------------- breakdown without a report --
@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_breakdown_surfaces_without_report(L, variant):
    """At eps = 0.004 the un-stabilised fp32 factors of the illustration data underflow (DESIGN.md
    C12/C30): a row dot is 0 and the solve breaks down.  With a report the call returns
    LSK_EBREAKDOWN; without one the sticky status returns it on the next lsk_stream_status."""
    import torch
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=2000, m=2000)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    with pytest.raises(L.LskError) as e:
        L.rot(X, Y, a, b, 0.004, 256, 5, iters=30, variant=variant)
    assert e.value.status == EBREAKDOWN
    L.lsk_stream_status()
    p = L.lsk_feature_params_init(0.004, 2, 256, 0.0, 5, X, Y)
    U = torch.empty((256, 2), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(2000, dtype=torch.float32, device="cuda")
    v = torch.empty(2000, dtype=torch.float32, device="cuda")
    if variant == "implicit":
        L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, L.make_opts(30), u, v, report=False)
    else:
        Xi = torch.empty((2000, 256), dtype=torch.float32, device="cuda")
        Ze = torch.empty((2000, 256), dtype=torch.float32, device="cuda")
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
        L.lsk_factored_sinkhorn(Xi, Ze, a, b, 0.004, L.make_opts(30), u, v, report=False)
    with pytest.raises(L.LskError) as e:
        L.lsk_stream_status()
    assert e.value.status == EBREAKDOWN
    L.lsk_stream_status()


# ------------------------------------------------------------- multi-launch early stop -----
@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_nccl_multilaunch_tolerance_many_rows_per_cta(L, variant):
    """One pass per launch with an NCCL all-reduce between launches, tolerance mode, ~270 rows
    per CTA (config 2 at full size: far more than the stream kernel's ring holds): the launch
    that starts after the stopping iteration must not stream a pass (its producer decides the
    stop with the consumers) — no hang, and the result matches the single-launch solve."""
    import torch
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    uid = L.lsk_comm_get_unique_id()
    comm = L.lsk_comm_init(1, 0, uid, torch.cuda.current_device())
    try:
        res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, max_iters=400, tol=1e-5,
                    variant=variant, comm=comm)
        single = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, max_iters=400, tol=1e-5,
                       variant=variant)
        torch.cuda.synchronize()
        assert res["report"]["converged"] == 1 and res["report"]["marginal_err"] < 1e-5
        assert res["report"]["iters"] == single["report"]["iters"] < 400
        assert abs(res["rot"] - single["rot"]) <= 1e-7 * abs(single["rot"])
    finally:
        L.lsk_comm_destroy(comm)


# ------------------------------------------------------------- workspace sized after planning
def test_workspace_many_ctas_batch_of_one(L):
    """lsk_factored_sinkhorn_batched with batch = 1 plans one CTA group over the whole device
    (gpp up to 148): its fp64 partials (r = 4096) need far more than a fixed 64-CTA
    workspace — sized after planning, the result equals the single solve and the oracle."""
    import torch
    n = m = 2000
    r = 4096
    gpp, grid = L.lsk_solve_plan(n, m, r, 1, 1, "stream")
    assert gpp > 64
    cfg = synth.get_config(5)
    prob = synth.make_problem(cfg, n=n, m=m)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    T = 30
    single = L.rot(X, Y, a, b, cfg.eps, r, 3, iters=T)
    Xi, Ze = single["Xi"], single["Zeta"]
    u = torch.empty((1, n), dtype=torch.float32, device="cuda")
    v = torch.empty((1, m), dtype=torch.float32, device="cuda")
    reps = L.lsk_factored_sinkhorn_batched(Xi[None], Ze[None], a[None], b[None], cfg.eps,
                                           L.make_opts(T), u, v)
    assert torch.equal(u[0], single["u"]) and torch.equal(v[0], single["v"])
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, r, 3, T=T)
    _parity(u[0], v[0], reps[0].rot, ref)


def test_workspace_more_ctas_per_sm(L):
    """ctas_per_sm above the old fixed 2-per-SM reservation (small r, many rows)."""
    cfg = synth.get_config(2)
    prob = synth.make_problem(cfg, n=60001, m=59999)
    r, T = 64, 40
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    res = L.rot(X, Y, a, b, cfg.eps, r, 9, iters=T, ctas_per_sm=4)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, r, 9, T=T)
    _parity(res["u"], res["v"], res["rot"], ref)


# ------------------------------------------------------------- batch > groups --------------
def test_batched_groups_loop_over_problems(L):
    """40 config-4 problems (n = m = 4096, r = 512, d = 128): the planner picks groups of
    gpp > 1 CTAs and fewer groups than problems, so each group runs several problems in turn
    (per-problem barrier counters, partials and ring phases carried across problems).  Every
    problem matches the oracle."""
    import torch
    cfg = synth.get_config(4)
    B, T = 40, 40
    gpp, grid = L.lsk_solve_plan(cfg.n, cfg.m, cfg.r, 1, B, "stream")
    assert gpp > 1 and grid // gpp < B, (gpp, grid)
    bp = synth.make_batched(cfg, batch=B)
    X, Y, a, b = (_dev(bp[k]) for k in ("X", "Y", "a", "b"))
    R = max(O.max_norm(bp["X"][p], bp["Y"][p]) for p in range(B))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, R, cfg.anchor_seed)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((B, cfg.n, cfg.r), dtype=torch.float32, device="cuda")
    Ze = torch.empty((B, cfg.m, cfg.r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map_batched(p, U, X, Xi)
    L.lsk_feature_map_batched(p, U, Y, Ze)
    u = torch.empty((B, cfg.n), dtype=torch.float32, device="cuda")
    v = torch.empty((B, cfg.m), dtype=torch.float32, device="cuda")
    reps = L.lsk_factored_sinkhorn_batched(Xi, Ze, a, b, cfg.eps, L.make_opts(T), u, v)
    for q in range(B):   # the oracle draws its own anchors (same seed, same R)
        ref = O.rot(bp["X"][q], bp["Y"][q], bp["a"][q], bp["b"][q], cfg.eps, cfg.r,
                    cfg.anchor_seed, T=T, R=R)
        _parity(u[q], v[q], reps[q].rot, ref)


# ------------------------------------------------------------- cluster pass boundary --------
@pytest.mark.parametrize("variant", ["stream", "implicit"])
@pytest.mark.parametrize("n,m,T", [(500, 500, 200), (1001, 777, 61), (130, 257, 40)])
def test_cluster_mode_small_problems(L, variant, n, m, T):
    """Small problems run as one thread-block cluster of 2..8 CTAs whose per-pass r-vector
    reduction goes over DSMEM (lsk_sink_common.cuh cx_*): the plan says so, and u, v, W_hat
    match the oracle (config-1 distribution, ragged n != m, both parities of T)."""
    cfg = synth.get_config(1)
    gpp, grid, cx = L.lsk_solve_plan(n, m, cfg.r, cfg.d, 1, variant, cluster=True)
    assert cx == 1 and 2 <= gpp <= 8 and grid == gpp, (gpp, grid, cx)
    prob = synth.make_problem(cfg, n=n, m=m)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    # resident=False: these shapes would otherwise run on the resident kernel (test_gpu_resident)
    res = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, iters=T, variant=variant,
                resident=False)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
    _parity(res["u"], res["v"], res["rot"], ref)
    # tolerance mode: the stop decision from the cluster totals
    res_t = L.rot(X, Y, a, b, cfg.eps, cfg.r, cfg.anchor_seed, max_iters=500, tol=1e-6,
                  variant=variant, resident=False)
    ref_t = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, tol=1e-6)
    assert res_t["report"]["converged"] == 1 and abs(res_t["report"]["iters"] - ref_t["iters"]) <= 1


def test_cluster_mode_batched(L):
    """A batch smaller than the device: each problem is a cluster of CTAs (implicit), or groups
    of cluster CTAs loop over problems (stream)."""
    import torch
    cfg = synth.get_config(1)
    B, n, T = 5, 500, 50
    for variant in ("stream", "implicit"):
        gpp, grid, cx = L.lsk_solve_plan(n, n, cfg.r, cfg.d, B, variant, cluster=True)
        assert cx == 1 and gpp >= 2
    bp = synth.make_batched(synth.get_config(4, d=2, r=100, eps=0.5), batch=B, n=n, m=n)
    X, Y, a, b = (_dev(bp[k]) for k in ("X", "Y", "a", "b"))
    R = max(O.max_norm(bp["X"][q], bp["Y"][q]) for q in range(B))
    p = L.lsk_feature_params_init(0.5, 2, 100, R, 11)
    U = torch.empty((100, 2), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty((B, n), dtype=torch.float32, device="cuda")
    v = torch.empty((B, n), dtype=torch.float32, device="cuda")
    reps = L.lsk_factored_sinkhorn_implicit_batched(p, U, X, Y, a, b, L.make_opts(T), u, v)
    Xi = torch.empty((B, n, 100), dtype=torch.float32, device="cuda")
    Ze = torch.empty((B, n, 100), dtype=torch.float32, device="cuda")
    L.lsk_feature_map_batched(p, U, X, Xi)
    L.lsk_feature_map_batched(p, U, Y, Ze)
    u2 = torch.empty((B, n), dtype=torch.float32, device="cuda")
    v2 = torch.empty((B, n), dtype=torch.float32, device="cuda")
    reps2 = L.lsk_factored_sinkhorn_batched(Xi, Ze, a, b, 0.5, L.make_opts(T), u2, v2)
    # the same batch on the grid kernels (these shapes otherwise run resident, one cluster per
    # problem: test_gpu_resident.py)
    u3 = torch.empty((B, n), dtype=torch.float32, device="cuda")
    v3 = torch.empty((B, n), dtype=torch.float32, device="cuda")
    reps3 = L.lsk_factored_sinkhorn_implicit_batched(p, U, X, Y, a, b,
                                                     L.make_opts(T, resident=False), u3, v3)
    u4 = torch.empty((B, n), dtype=torch.float32, device="cuda")
    v4 = torch.empty((B, n), dtype=torch.float32, device="cuda")
    reps4 = L.lsk_factored_sinkhorn_batched(Xi, Ze, a, b, 0.5, L.make_opts(T, resident=False), u4, v4)
    for q in range(B):
        ref = O.rot(bp["X"][q], bp["Y"][q], bp["a"][q], bp["b"][q], 0.5, 100, 11, T=T, R=R)
        _parity(u[q], v[q], reps[q].rot, ref)
        _parity(u2[q], v2[q], reps2[q].rot, ref)
        _parity(u3[q], v3[q], reps3[q].rot, ref)
        _parity(u4[q], v4[q], reps4[q].rot, ref)
