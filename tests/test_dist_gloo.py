"""N>1 path on CPU: world_size-2 gloo processes run the row-sharded protocol of the
multi-GPU solver — rows partitioned by the library's lsk_shard_range, one fp64 all-reduce
of the r-vector partial per half-iteration, all-reduced read-out — with the oracle's
arithmetic standing in for the local GPU pass.  The gathered result must equal the
unsharded oracle solve (same fp64 math, only the summation split differs).

exchange="rank_order" models the in-kernel NVLink exchange (lsk_comm_enable_p2p): every rank
receives every rank's fp64 partial (the peer inboxes; here an all-gather) and adds them in
rank order starting from 0.0 — every rank must end with bit-identical vectors, and so with
identical stopping decisions and read-out."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, T, q, exchange="allreduce"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle as O
    import paper_2006_07057_b200 as L
    import synth
    cfg = synth.get_config(3)
    prob = synth.make_problem(cfg, n=1003, m=997)
    r = 64
    nb, ne = L.lsk_shard_range(1003, ws, rank)
    mb, me = L.lsk_shard_range(997, ws, rank)
    # a1: global R = all-reduce(max) of the local max norms
    Rl = torch.tensor([O.max_norm(prob["X"][nb:ne], prob["Y"][mb:me])], dtype=torch.float64)
    dist.all_reduce(Rl, op=dist.ReduceOp.MAX)
    prm = O.gaussian_params(cfg.eps, cfg.d, r, float(Rl))
    U = O.draw_anchors(r, cfg.d, prm["sigma"], cfg.anchor_seed)     # replicated per rank
    xi = O.feature_matrix(prob["X"][nb:ne], U, cfg.eps, prm["q"])   # local shard, r x n_l
    ze = O.feature_matrix(prob["Y"][mb:me], U, cfg.eps, prm["q"])
    a = prob["a"][nb:ne].astype(np.float64)
    b = prob["b"][mb:me].astype(np.float64)

    def allreduce(x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if exchange == "allreduce":
            t = torch.from_numpy(x.copy())
            dist.all_reduce(t)
            return t.numpy()
        parts = [torch.zeros_like(torch.from_numpy(x)) for _ in range(ws)]
        dist.all_gather(parts, torch.from_numpy(x))       # every rank's inbox slots
        tot = np.zeros_like(x)
        for src in range(ws):                            # rank order, from 0.0
            tot = tot + parts[src].numpy()
        return tot

    s_v = allreduce(xi @ np.ones(ne - nb))           # init pass: xi^T 1
    for _ in range(T):
        v = b / (ze.T @ s_v)                          # local v-pass
        s_u = allreduce(ze @ v)                       # r-vector exchange
        u = a / (xi.T @ s_u)                          # local u-pass
        s_v = allreduce(xi @ u)
    parts = allreduce(np.array([a @ np.log(u), b @ np.log(v)]))
    rot = cfg.eps * parts.sum()
    us = [None] * ws
    vs = [None] * ws
    rots = [None] * ws
    dist.all_gather_object(us, u)
    dist.all_gather_object(vs, v)
    dist.all_gather_object(rots, rot)
    if rank == 0:
        q.put((rot, np.concatenate(us), np.concatenate(vs), float(Rl), rots))
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["allreduce", "rank_order"])
@pytest.mark.parametrize("ws", [2])
def test_row_sharded_protocol_matches_unsharded(ws, exchange):
    import oracle as O
    import synth
    T = 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, ws, port, T, q, exchange)) for k in range(ws)]
    for p in procs:
        p.start()
    rot, u, v, R, rots = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.get_config(3)
    prob = synth.make_problem(cfg, n=1003, m=997)
    assert abs(R - O.max_norm(prob["X"], prob["Y"])) == 0.0
    ref = O.rot(prob["X"], prob["Y"], prob["a"], prob["b"], cfg.eps, 64, cfg.anchor_seed, T=T)
    assert abs(rot - ref["rot"]) <= 1e-12 * abs(ref["rot"])
    assert np.allclose(u, ref["u"], rtol=1e-11) and np.allclose(v, ref["v"], rtol=1e-11)
    if exchange == "rank_order":
        assert all(x == rots[0] for x in rots)           # bit-identical on every rank
