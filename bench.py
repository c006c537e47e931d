#!/usr/bin/env python
"""bench.py — factored-Sinkhorn throughput on B200 (BASELINE.json metric).

One *step* = the whole hot path on one synthetic problem of the
workload: feature parameters (auto R), anchors, feature maps (streaming variant), T Sinkhorn
iterations, read-out.  value = iterations/s = (T x steps x problem-units) / device time.

  python bench.py                         # N=1, config 2 (Fig. 1 shape), defaults
  python bench.py --impl reference        # the fp64 oracle on host cores (bounded sample)
  torchrun --nproc-per-node N bench.py --gpus N   # rows of one global problem sharded,
                                                  # N x the per-GPU rows (weak scaling)

Timing: W warm-up steps, then K timed steps; each step is bracketed by CUDA events on the
launching stream, with an L2 flush (256 MiB write) before every step outside the events;
barrier + synchronize on both sides of the timed loop; max over ranks.  nvidia-smi clocks
are sampled during the timed region.  The dominant kernel (the persistent Sinkhorn launch)
is timed separately with its own events for the roofline object.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "factored-Sinkhorn iterations/sec at (n,r)"
UNIT = "iter/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ======================================================================= reference arm ====
def run_reference(args):
    """The fp64 oracle, as it stands, on the host cores: a bounded sample of the workload
    (full-size features + a few iterations), extrapolated to the workload's T."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import oracle as O
    from threadpoolctl import threadpool_info
    cfg = synth.get_config(args.config)
    prob = synth.make_problem(cfg)
    k_iter = args.ref_iters
    # warm-up (untimed): one feature evaluation on a slice
    O.feature_matrix(prob["X"][:1000], np.zeros((cfg.r, cfg.d)), cfg.eps, 1.0)
    step_vals = []
    t_feat_all, t_iter_all = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        R = O.max_norm(prob["X"], prob["Y"])
        prm = O.gaussian_params(cfg.eps, cfg.d, cfg.r, R)
        U = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
        xi = O.feature_matrix(prob["X"], U, cfg.eps, prm["q"])
        zeta = O.feature_matrix(prob["Y"], U, cfg.eps, prm["q"])
        t1 = time.perf_counter()
        sol = O.sinkhorn_factored(xi, zeta, prob["a"], prob["b"], T=k_iter)
        O.dual_estimate(sol["u"], sol["v"], prob["a"], prob["b"], cfg.eps)
        t2 = time.perf_counter()
        t_feat, t_it = t1 - t0, (t2 - t1) / k_iter
        t_feat_all.append(t_feat)
        t_iter_all.append(t_it)
        step_vals.append(cfg.T / (cfg.batch * (t_feat + cfg.T * t_it)))   # B pairs per iteration
    cores = max([int(i.get("num_threads", 0)) for i in threadpool_info()] or [os.cpu_count()])
    value = float(np.median(step_vals))
    sample = ("config %d full size (n=m=%d, r=%d): fp64 features + %d of T=%d iterations per "
              "step, extrapolated to T" % (cfg.key, cfg.n, cfg.r, k_iter, cfg.T))
    if cfg.batch > 1:
        sample += "; one of the %d pairs, x%d" % (cfg.batch, cfg.batch)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.batch * float(np.median([tf + cfg.T * ti for tf, ti in zip(t_feat_all, t_iter_all)])),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "config%d-%s" % (cfg.key, cfg.name), "n": cfg.n, "m": cfg.m,
                   "d": cfg.d, "r": cfg.r, "eps": cfg.eps, "T": cfg.T, "parallelism": "host"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "oracle_seconds": {"features": float(np.median(t_feat_all)),
                           "per_iteration": float(np.median(t_iter_all))},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(cfg, iters=3):
    """Oracle timed on this host's cores on a bounded sample (rank 0, N=1 only)."""
    import oracle as O
    from threadpoolctl import threadpool_info
    prob = synth.make_problem(cfg)
    t0 = time.perf_counter()
    R = O.max_norm(prob["X"], prob["Y"])
    prm = O.gaussian_params(cfg.eps, cfg.d, cfg.r, R)
    U = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
    xi = O.feature_matrix(prob["X"], U, cfg.eps, prm["q"])
    zeta = O.feature_matrix(prob["Y"], U, cfg.eps, prm["q"])
    t1 = time.perf_counter()
    O.sinkhorn_factored(xi, zeta, prob["a"], prob["b"], T=iters)
    t2 = time.perf_counter()
    t_it = (t2 - t1) / iters
    value = cfg.T / (cfg.batch * ((t1 - t0) + cfg.T * t_it))
    cores = max([int(i.get("num_threads", 0)) for i in threadpool_info()] or [os.cpu_count()])
    pairs = (" one of the %d pairs, x%d" % (cfg.batch, cfg.batch)) if cfg.batch > 1 else ""
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "config %d full size%s: fp64 features + %d of T=%d iterations, extrapolated "
                      "to T (features %.2f s, %.3f s/iteration)" % (cfg.key, pairs, iters, cfg.T,
                                                                    t1 - t0, t_it)}


# ======================================================================= lsk arm ==========
def run_lsk(args):
    import torch
    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    import paper_2006_07057_b200 as L
    dist = None
    comm = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [L.lsk_comm_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = L.lsk_comm_init(ws, rank, uid[0], local)
        # in-kernel NVLink exchange: one persistent launch per GPU (NCCL multi-launch fallback)
        exchange = "nccl-multilaunch"
        if os.environ.get("LSK_P2P", "1") != "0":
            try:
                L.lsk_comm_enable_p2p(comm, synth.get_config(args.config).r)
                exchange = "nvlink-p2p-in-kernel"
            except L.LskError as e:
                print("warning: peer exchange unavailable (%s); NCCL path" % e, file=sys.stderr)

    if ws == 1:
        exchange = "none"
    cfg = synth.get_config(args.config)
    if cfg.batch > 1:
        return run_lsk_batched(args, cfg, L, torch, dist, comm, ws, rank, local)
    variant = args.variant
    if variant == "auto":
        # measured: the MUFU-recompute variant is faster where it applies
        # (d <= 8: configs 1, 2, 5); the factor stream elsewhere (configs 3, 4)
        variant = "implicit" if cfg.d <= 8 else "stream"
    n_loc, m_loc = cfg.n, cfg.m
    # weak scaling: the global problem has ws x the per-GPU rows; each rank owns one shard
    full = synth.make_problem(cfg, n=cfg.n * ws, m=cfg.m * ws)
    nb, ne = L.lsk_shard_range(cfg.n * ws, ws, rank)
    mb, me = L.lsk_shard_range(cfg.m * ws, ws, rank)
    dev = torch.device("cuda", local)
    X = torch.from_numpy(full["X"][nb:ne].copy()).to(dev)
    Y = torch.from_numpy(full["Y"][mb:me].copy()).to(dev)
    a = torch.from_numpy(full["a"][nb:ne].copy()).to(dev)
    b = torch.from_numpy(full["b"][mb:me].copy()).to(dev)
    n_loc, m_loc = X.shape[0], Y.shape[0]
    r, d, T, eps = cfg.r, cfg.d, cfg.T, cfg.eps
    U = torch.empty((r, d), dtype=torch.float32, device=dev)
    u = torch.empty(n_loc, dtype=torch.float32, device=dev)
    v = torch.empty(m_loc, dtype=torch.float32, device=dev)
    opts = L.make_opts(T, 0.0, False, args.ctas_per_sm)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    peaks, src = _peaks()

    def measure(var, steps, warmup, sample_clocks):
        Xi = Ze = None
        if var == "stream":
            Xi = torch.empty((n_loc, r), dtype=torch.float32, device=dev)
            Ze = torch.empty((m_loc, r), dtype=torch.float32, device=dev)

        def step(ev_k0=None, ev_k1=None):
            p = L.lsk_feature_params_init(eps, d, r, 0.0, cfg.anchor_seed, X, Y, comm=comm)
            L.lsk_draw_anchors(p, U)
            if var == "stream":
                L.lsk_feature_map(p, U, X, Xi)
                L.lsk_feature_map(p, U, Y, Ze)
                if ev_k0 is not None:
                    ev_k0.record(stream)
                L.lsk_factored_sinkhorn(Xi, Ze, a, b, eps, opts, u, v, report=False, comm=comm)
            else:
                if ev_k0 is not None:
                    ev_k0.record(stream)
                L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=False,
                                                 comm=comm)
            if ev_k1 is not None:
                ev_k1.record(stream)
            # read-out on the host (the step's result): fp64 ROT from the same call's state
            return L.lsk_rot_value(u, v, a, b, eps, comm=comm)

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        if comm is not None:   # surface a cross-GPU exchange failure (the timed steps do not sync)
            p = L.lsk_feature_params_init(eps, d, r, 0.0, cfg.anchor_seed, X, Y, comm=comm)
            L.lsk_draw_anchors(p, U)
            if var == "stream":
                L.lsk_feature_map(p, U, X, Xi)
                L.lsk_feature_map(p, U, Y, Ze)
                L.lsk_factored_sinkhorn(Xi, Ze, a, b, eps, opts, u, v, report=True, comm=comm)
            else:
                L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=True,
                                                 comm=comm)
        clocks = ClockSampler(local) if sample_clocks else None
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        L.launch_count(reset=True)
        step_ms, kern_ms = [], []
        rot_val = None
        for _ in range(steps):
            flush.zero_()                          # L2 flush, outside the timed events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rot_val = step(k0, k1)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            kern_ms.append(k0.elapsed_time(k1))
        launches = L.launch_count()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        clk = clocks.stop() if clocks else None
        tot_ms = float(np.sum(step_ms))
        kmean = float(np.mean(kern_ms))
        if dist is not None:
            t = torch.tensor([tot_ms, kmean], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot_ms, kmean = float(t[0]), float(t[1])
        units = ws                                  # config-sized problem-units per step
        value = units * T * steps / (tot_ms / 1e3)
        # roofline of the dominant kernel (the persistent Sinkhorn launch)
        if var == "stream":
            passes_rows = n_loc + T * (n_loc + m_loc)
            alg_bytes = 4.0 * r * passes_rows + 8.0 * passes_rows + 4.0 * m_loc * (T - 1)
            achieved = alg_bytes / (kmean / 1e3) / 1e9
            peak = float(peaks["hbm_gbs"])
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (%s)" % src,
                    "algorithmic_bytes_per_launch": alg_bytes}
        else:
            ex2 = float(r) * (n_loc + T * (n_loc + m_loc))
            achieved = ex2 / (kmean / 1e3) / 1e9
            peak = 4626.0   # measured, profiles/r01_mufu_microbench.txt (16/clk/SM x 148 x 1.965 GHz = 4653)
            roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gex2/s",
                    "frac": achieved / peak, "traffic": None,
                    "peak_source": "MUFU ex2 measured on B200 (profiles/r01_mufu_microbench.txt)",
                    "algorithmic_ex2_per_launch": ex2}
        tr_path = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr_path):
            try:
                tr = json.load(open(tr_path)).get("config%d-%s" % (cfg.key, var))
                if tr:
                    roof["traffic"] = tr
            except Exception:
                pass
        return {"value": value, "ms_per_step": tot_ms / steps, "kernel_ms": kmean,
                "launches": int(launches), "clocks": clk, "rot": rot_val, "roofline": roof}

    main_m = measure(variant, args.steps, args.warmup, True)
    result = {
        "metric": METRIC, "value": main_m["value"], "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_m["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "config%d-%s" % (cfg.key, cfg.name), "variant": variant,
                   "n_per_gpu": cfg.n, "m_per_gpu": cfg.m, "d": d, "r": r, "eps": eps, "T": T,
                   "global_n": cfg.n * ws, "parallelism": "rows%d" % ws if ws > 1 else "single",
                   "exchange": exchange,
                   "l2": "flushed (256 MiB write) before every timed step"},
        "roofline": main_m["roofline"],
        "kernel_ms": main_m["kernel_ms"],
        "gpu_launches": main_m["launches"],
        "clocks": main_m["clocks"],
        "rot": main_m["rot"],
    }
    # the other variant on the same workload (same timing protocol), for the comparison the
    # variant choice rests on; its roofline is the HBM one when it is the factor stream
    if ws == 1 and not args.no_alt and cfg.d <= 8:
        alt = "stream" if variant == "implicit" else "implicit"
        m = measure(alt, args.steps, args.warmup, False)
        result["alt_variant"] = {"variant": alt, "value": m["value"], "unit": UNIT,
                                 "ms_per_step": m["ms_per_step"], "kernel_ms": m["kernel_ms"],
                                 "roofline": m["roofline"], "rot": m["rot"]}

    # end-to-end through the public host-buffer entry point (N=1 only)
    if ws == 1 and not args.no_e2e:
        Xh = torch.from_numpy(full["X"]).pin_memory()
        Yh = torch.from_numpy(full["Y"]).pin_memory()
        ah = torch.from_numpy(full["a"]).pin_memory()
        bh = torch.from_numpy(full["b"]).pin_memory()
        uh = torch.empty(n_loc, dtype=torch.float32).pin_memory()
        vh = torch.empty(m_loc, dtype=torch.float32).pin_memory()
        vcode = 2 if variant == "implicit" else 1
        for _ in range(max(1, args.warmup)):
            L.lsk_rot_host(Xh, Yh, ah, bh, eps, r, cfg.anchor_seed, opts, variant=vcode, u_out=uh, v_out=vh)
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.lsk_rot_host(Xh, Yh, ah, bh, eps, r, cfg.anchor_seed, opts, variant=vcode, u_out=uh, v_out=vh)
            ts.append(time.perf_counter() - t0)
        h2d = 4 * (n_loc * d + m_loc * d + n_loc + m_loc)
        d2h = 4 * (n_loc + m_loc) + 48
        result["e2e"] = {"value": T * len(ts) / float(np.sum(ts)), "unit": UNIT,
                         "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    else:
        result["e2e"] = None

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, iters=args.ref_iters)
    if comm is not None:
        L.lsk_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))
    return 0


def run_lsk_batched(args, cfg, L, torch, dist, comm, ws, rank, local):
    """Config 4: B independent pairs in one batched solve per step (shared anchor draw, R over
    all pairs; tcgen05 feature maps; one persistent batched Sinkhorn launch; batched read-out).
    An iteration is one Sinkhorn iteration of every pair; weak scaling = B pairs per GPU, no
    cross-GPU exchange (the pairs are independent)."""
    B, n, m, r, d, T, eps = cfg.batch, cfg.n, cfg.m, cfg.r, cfg.d, cfg.T, cfg.eps
    dev = torch.device("cuda", local)
    bp = synth.make_batched(cfg)   # the same B pairs on every rank (independent problems)
    Xh = torch.from_numpy(bp["X"]).pin_memory()
    Yh = torch.from_numpy(bp["Y"]).pin_memory()
    ah = torch.from_numpy(bp["a"]).pin_memory()
    bh = torch.from_numpy(bp["b"]).pin_memory()
    X, Y, a, b = (t.to(dev) for t in (Xh, Yh, ah, bh))
    U = torch.empty((r, d), dtype=torch.float32, device=dev)
    Xi = torch.empty((B, n, r), dtype=torch.float32, device=dev)
    Ze = torch.empty((B, m, r), dtype=torch.float32, device=dev)
    u = torch.empty((B, n), dtype=torch.float32, device=dev)
    v = torch.empty((B, m), dtype=torch.float32, device=dev)
    opts = L.make_opts(T, 0.0, False, args.ctas_per_sm)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    peaks, src = _peaks()

    def step(Xs, Ys, As, Bs, ev_k0=None, ev_k1=None):
        p = L.lsk_feature_params_init(eps, d, r, 0.0, cfg.anchor_seed, Xs.reshape(-1, d), Ys.reshape(-1, d))
        L.lsk_draw_anchors(p, U)
        L.lsk_feature_map_batched(p, U, Xs, Xi)
        L.lsk_feature_map_batched(p, U, Ys, Ze)
        if ev_k0 is not None:
            ev_k0.record(stream)
        L.lsk_factored_sinkhorn_batched(Xi, Ze, As, Bs, eps, opts, u, v, report=False)
        if ev_k1 is not None:
            ev_k1.record(stream)
        return L.lsk_rot_value_batched(u, v, As, Bs, eps)

    for _ in range(args.warmup):
        step(X, Y, a, b)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    L.launch_count(reset=True)
    step_ms, kern_ms, rots = [], [], None
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rots = step(X, Y, a, b, k0, k1)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(k0.elapsed_time(k1))
    launches = L.launch_count()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    tot_ms, kmean = float(np.sum(step_ms)), float(np.mean(kern_ms))
    if dist is not None:
        t = torch.tensor([tot_ms, kmean], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, kmean = float(t[0]), float(t[1])
    value = ws * T * args.steps / (tot_ms / 1e3)
    rows = n + T * (n + m)
    alg_bytes = B * (4.0 * r * rows + 8.0 * rows + 4.0 * m * (T - 1))
    achieved = alg_bytes / (kmean / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (%s)" % src,
            "algorithmic_bytes_per_launch": alg_bytes}
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "config%d-%s" % (cfg.key, cfg.name), "variant": "stream-batched",
                   "batch_per_gpu": B, "n": n, "m": m, "d": d, "r": r, "eps": eps, "T": T,
                   "iteration": "one Sinkhorn iteration of every pair",
                   "pair_iterations_per_s": value * B,
                   "parallelism": "pairs%d" % ws if ws > 1 else "single",
                   "l2": "flushed (256 MiB write) before every timed step"},
        "roofline": roof, "kernel_ms": kmean, "gpu_launches": int(launches), "clocks": clk,
        "rot_pair0": rots[0] if rots else None,
    }
    if ws == 1 and not args.no_e2e:   # host buffers in, ROT values out, copies timed
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Xs, Ys, As, Bs = (t.to(dev, non_blocking=True) for t in (Xh, Yh, ah, bh))
            step(Xs, Ys, As, Bs)   # rot values come back to the host
            ts.append(time.perf_counter() - t0)
        result["e2e"] = {"value": T * len(ts) / float(np.sum(ts)), "unit": UNIT,
                         "h2d_bytes_per_step": 4 * B * (n * d + m * d + n + m),
                         "d2h_bytes_per_step": 8 * B}
    else:
        result["e2e"] = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, iters=args.ref_iters)
    if comm is not None:
        L.lsk_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lsk", choices=["lsk", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--variant", default="auto", choices=["auto", "stream", "implicit"])
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--ref-iters", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip timing the other variant")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "lsk":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_lsk(args)


if __name__ == "__main__":
    sys.exit(main())
