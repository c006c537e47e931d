"""The multi-GPU row-sharded path's in-kernel exchange (lsk_comm_enable_p2p protocol,
lsk_sink_common.cuh xrank_total) with N = 2, 4 and 8 ranks emulated inside ONE cooperative
launch on one GPU (lsk_*_emulated; B200_PROFILING.md: ranks that wait on one another must not
be separate launches on one GPU).  Every rank stores its fp64 totals into every rank's inbox,
polls its own, sums in rank order and re-arms — per half-iteration (the
r-vector is the only datum the shards share).  Checked: the global u, v and W_hat against the
fp64 oracle of the UNSHARDED problem; all ranks' reports bit-identical; tolerance mode stops
on the same iteration on every rank."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


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
    return float(np.max(np.abs(gpu.cpu().double().numpy() - ref) / np.abs(ref)))


@pytest.mark.parametrize("variant", ["stream", "implicit"])
@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("T", [40, 41])   # both parities of the last pass
def test_emulated_ranks_match_oracle(L, variant, N, T):
    import torch
    cfg = synth.get_config(2)
    n, m = 8000, 7992                     # divisible by 2, 4, 8; n != m
    prob = synth.make_problem(cfg, n=n, m=m)
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, T=T)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    v = torch.empty(m, dtype=torch.float32, device="cuda")
    opts = L.make_opts(T)
    if variant == "stream":
        Xi = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
        Ze = torch.empty((m, cfg.r), dtype=torch.float32, device="cuda")
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
        reps = L.lsk_factored_sinkhorn_emulated(N, Xi, Ze, a, b, cfg.eps, opts, u, v)
    else:
        reps = L.lsk_factored_sinkhorn_implicit_emulated(N, p, U, X, Y, a, b, opts, u, v)
    rots = [rp.rot for rp in reps]
    assert all(x == rots[0] for x in rots)                       # identical on every rank
    assert all(rp.iters == T for rp in reps)
    assert abs(rots[0] - ref["rot"]) <= 1e-5 * abs(ref["rot"])
    assert _maxrel(u, ref["u"]) <= 1e-4 and _maxrel(v, ref["v"]) <= 1e-4
    # the rank-order all-rank sum reproduces the read-out of the returned scalings
    assert abs(L.lsk_rot_value(u, v, a, b, cfg.eps) - rots[0]) <= 1e-12 * abs(rots[0])


@pytest.mark.parametrize("variant", ["stream", "implicit"])
def test_emulated_ranks_tolerance_mode(L, variant):
    import torch
    cfg = synth.get_config(1)
    n = m = 500
    prob = synth.make_problem(cfg)
    tol = 1e-6
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, cfg.r, cfg.anchor_seed, tol=tol)
    X, Y, a, b = (_dev(prob[k]) for k in ("X", "Y", "a", "b"))
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    v = torch.empty(m, dtype=torch.float32, device="cuda")
    opts = L.make_opts(1000, tol=tol)
    if variant == "stream":
        Xi = torch.empty((n, cfg.r), dtype=torch.float32, device="cuda")
        Ze = torch.empty((m, cfg.r), dtype=torch.float32, device="cuda")
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
        reps = L.lsk_factored_sinkhorn_emulated(4, Xi, Ze, a, b, cfg.eps, opts, u, v)
    else:
        reps = L.lsk_factored_sinkhorn_implicit_emulated(4, p, U, X, Y, a, b, opts, u, v)
    its = {rp.iters for rp in reps}
    assert len(its) == 1 and all(rp.converged == 1 for rp in reps)
    assert abs(reps[0].iters - ref["iters"]) <= 1 and reps[0].marginal_err < tol
