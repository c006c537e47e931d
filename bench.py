#!/usr/bin/env python
"""bench.py — factored-Sinkhorn throughput on B200 (BASELINE.json metric).

One *step* = the whole hot path on one synthetic problem of the
workload: feature parameters (auto R), anchors, feature maps (streaming variant), T Sinkhorn
iterations, read-out.  value = iterations/s = (T x steps x problem-units) / device time.

  python bench.py                         # N=1: config 2 (Fig. 1 shape) headline line, plus
                                          # configs 3, 4, 5 at full size under "configs"
  python bench.py --impl reference        # the fp64 oracle on host cores (bounded sample)
  python bench.py --gpus N                # spawns N ranks itself (torch.distributed.run on
                                          # 127.0.0.1) unless launched under torchrun
  torchrun --nproc-per-node N bench.py --gpus N

Scaling: the headline config is weak-scaled (N x its rows, one global problem row-sharded;
--scaling strong splits the config's rows instead); the "configs" lines are strong-scaled
(the config's fixed global rows — or config 4's 256 pairs — split over the N GPUs; config 5
is north_star's sharded largest config), value = global iterations/s.

Timing: W warm-up steps, then K timed steps; each step is bracketed by CUDA events on the
launching stream, with an L2 flush (256 MiB write) before every step outside the events;
barrier + synchronize on both sides of the timed loop; max over ranks.  nvidia-smi clocks
are sampled during each timed region.  The dominant kernel (the persistent Sinkhorn launch)
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


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


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
    sample = ("config %d full size (n=m=%d, r=%d): each step = fp64 features + %d of the T=%d "
              "iterations (measured); value = T / (features + T x per-iteration time) of the "
              "sample, i.e. extrapolated to T" % (cfg.key, cfg.n, cfg.r, k_iter, cfg.T))
    if cfg.batch > 1:
        sample += "; one of the %d pairs, x%d" % (cfg.batch, cfg.batch)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.median([tf + k_iter * ti for tf, ti in zip(t_feat_all, t_iter_all)])),
        "ms_per_step_note": "measured wall time of one sample step (features + %d iterations)" % k_iter,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "config%d-%s" % (cfg.key, cfg.name), "n": cfg.n, "m": cfg.m,
                   "d": cfg.d, "r": cfg.r, "eps": cfg.eps, "T": cfg.T, "parallelism": "host"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "cpu_model": _cpu_model(), "sample": sample},
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
            "cpu_model": _cpu_model(),
            "sample": "config %d full size%s: fp64 features + %d of T=%d iterations, extrapolated "
                      "to T (features %.2f s, %.3f s/iteration)" % (cfg.key, pairs, iters, cfg.T,
                                                                    t1 - t0, t_it)}


# ======================================================================= lsk arm ==========
MUFU_PEAK = 4626.0   # Gex2/s measured, profiles/r01_mufu_microbench.txt (16/clk/SM x 148 x 1.965 GHz = 4653)


SMEM_B_PER_CLK = 128.0   # shared-memory bandwidth per SM (B300_MICROARCH.md: 32 banks x 4 B)


def _roofline(var, cfg_key, r, n_loc, m_loc, T, kmean_ms, batch=1, stream_rows=(0, 0),
              resident=0):
    """Roofline object of the dominant kernel (the persistent Sinkhorn launch): algorithmic
    bytes (factor stream, HBM-bound) or ex2 (recompute, MUFU-bound) per launch over its mean
    CUDA-event duration.  The hybrid (a fraction of the rows streamed, the rest
    recomputed, both units at once) is bounded by the sum of the two entry rates: MUFU ex2/s +
    HBM bytes/s / 4 (factor entries/s)."""
    peaks, src = _peaks()
    ns0, ns1 = stream_rows
    if resident:
        # resident cluster kernel (DESIGN.md §6 K10): every pass reads its side's factor rows
        # once from shared memory; the roof is the G SMs' shared-memory bandwidth (the
        # one-time feature map of the implicit API is inside the timed launch window too)
        rows = n_loc + T * (n_loc + m_loc)
        alg_bytes = 4.0 * r * rows
        achieved = alg_bytes / (kmean_ms / 1e3) / 1e9
        peak = resident * SMEM_B_PER_CLK * float(peaks.get("sm_max_mhz", 1965.0)) / 1e3
        return {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "peak_source": "%d SMs x 128 B/clk x sm_max_mhz (%s)" % (resident, src),
                "algorithmic_bytes_per_launch": alg_bytes, "cluster_ctas": resident,
                "note": "per pass: st.async push of the CTA partials + one mbarrier wait: latency-bound"}
    if var == "implicit" and ns0 + ns1 > 0:
        entries = float(r) * (n_loc + T * (n_loc + m_loc))
        streamed = float(r) * (ns0 + T * (ns0 + ns1))
        achieved = entries / (kmean_ms / 1e3) / 1e9
        hbm = float(peaks["hbm_gbs"])
        peak = MUFU_PEAK + hbm / 4.0
        roof = {"bound": "alu+hbm", "achieved": achieved, "peak": peak, "unit": "Gentries/s",
                "frac": achieved / peak, "traffic": None,
                "peak_source": "MUFU ex2 measured (profiles/r01_mufu_microbench.txt) + "
                               "MEASURED_PEAKS.json hbm_gbs (%s) / 4 B per entry" % src,
                "algorithmic_entries_per_launch": entries,
                "streamed_fraction": streamed / entries,
                "mufu_frac_of_recomputed": (entries - streamed) / (kmean_ms / 1e3) / 1e9 / MUFU_PEAK,
                "hbm_frac_of_streamed": 4.0 * streamed / (kmean_ms / 1e3) / 1e9 / hbm}
        return roof
    if var == "implicit":
        ex2 = float(r) * (n_loc + T * (n_loc + m_loc)) * batch
        achieved = ex2 / (kmean_ms / 1e3) / 1e9
        peak = MUFU_PEAK
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gex2/s",
                "frac": achieved / peak, "traffic": None,
                "peak_source": "MUFU ex2 measured on B200 (profiles/r01_mufu_microbench.txt)",
                "algorithmic_ex2_per_launch": ex2}
    else:
        rows = n_loc + T * (n_loc + m_loc)
        alg_bytes = batch * (4.0 * r * rows + 8.0 * rows + 4.0 * m_loc * (T - 1))
        achieved = alg_bytes / (kmean_ms / 1e3) / 1e9
        peak = float(peaks["hbm_gbs"])
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (%s)" % src,
                "algorithmic_bytes_per_launch": alg_bytes}
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path)).get("config%d-%s" % (cfg_key, var))
            if tr:
                roof["traffic"] = tr
        except Exception:
            pass
    return roof


class Ctx:
    """Per-process state of the lsk arm: library, torch, process group, lsk communicator."""

    def __init__(self, args):
        import torch
        self.torch = torch
        self.ws, self.rank, self.local = _dist_env()
        torch.cuda.set_device(self.local)
        import paper_2006_07057_b200 as L
        self.L = L
        self.dev = torch.device("cuda", self.local)
        self.dist = None
        self.comm = None
        self.exchange = "none"
        if self.ws > 1:
            import torch.distributed as dist
            self.dist = dist
            dist.init_process_group("nccl", device_id=self.dev)
            uid = [L.lsk_comm_get_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            self.comm = L.lsk_comm_init(self.ws, self.rank, uid[0], self.local)
            # in-kernel NVLink exchange: one persistent launch per GPU (NCCL multi-launch fallback)
            self.exchange = "nccl-multilaunch"
            try:
                L.lsk_comm_enable_p2p(self.comm, 4096)
                self.exchange = "nvlink-p2p-in-kernel"
            except L.LskError as e:
                print("warning: peer exchange unavailable (%s); NCCL path" % e, file=sys.stderr)
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=self.dev)

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, *vals):
        if self.dist is None:
            return vals
        t = self.torch.tensor(list(vals), dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return tuple(float(x) for x in t)

    def close(self):
        if self.comm is not None:
            self.L.lsk_comm_destroy(self.comm)
        if self.dist is not None:
            self.dist.destroy_process_group()


def _timed_loop(C, step, steps, warmup, sample_clocks):
    """W untimed warm-up steps, then K steps, each between CUDA events on the launching
    stream with an L2 flush (256 MiB write) before it outside the events; barrier +
    synchronize on both sides; max over ranks.  step(k0, k1) records the dominant kernel's
    events.  Returns (total ms, mean kernel ms, launches, clocks, last step result)."""
    torch, L = C.torch, C.L
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        step(None, None)
    torch.cuda.synchronize()
    L.lsk_stream_status()   # a warm-up solve that broke down fails the bench here
    clocks = ClockSampler(C.local) if sample_clocks else None
    C.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    L.launch_count(reset=True)
    step_ms, kern_ms, res = [], [], None
    for _ in range(steps):
        C.flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step(k0, k1)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(k0.elapsed_time(k1))
    launches = L.launch_count()
    torch.cuda.synchronize()
    C.barrier()
    clk = clocks.stop() if clocks else None
    L.lsk_stream_status()
    tot_ms, kmean = C.max_over_ranks(float(np.sum(step_ms)), float(np.mean(kern_ms)))
    return tot_ms, kmean, int(launches), clk, res


def measure_single(C, cfg, variant, scaling, steps, warmup, sample_clocks=True,
                   stream_fraction=0.0):
    """One problem of config cfg, rows sharded over the ranks: weak scaling (ws x the config's
    rows, each rank holding the config's rows) or strong scaling (the config's rows split).
    value = global iterations/s = T x steps / max-over-ranks device time."""
    torch, L, ws, rank = C.torch, C.L, C.ws, C.rank
    gn, gm = (cfg.n * ws, cfg.m * ws) if scaling == "weak" else (cfg.n, cfg.m)
    full = synth.make_problem(cfg, n=gn, m=gm)
    nb, ne = L.lsk_shard_range(gn, ws, rank)
    mb, me = L.lsk_shard_range(gm, ws, rank)
    X, Y, a, b = (torch.from_numpy(np.ascontiguousarray(full[k][lo:hi])).to(C.dev)
                  for k, lo, hi in (("X", nb, ne), ("Y", mb, me), ("a", nb, ne), ("b", mb, me)))
    n_loc, m_loc = X.shape[0], Y.shape[0]
    r, d, T, eps = cfg.r, cfg.d, cfg.T, cfg.eps
    U = torch.empty((r, d), dtype=torch.float32, device=C.dev)
    u = torch.empty(n_loc, dtype=torch.float32, device=C.dev)
    v = torch.empty(m_loc, dtype=torch.float32, device=C.dev)
    opts = L.make_opts(T, stream_fraction=stream_fraction)
    srows = L.lsk_stream_rows(n_loc, m_loc, r, d, opts) if variant == "implicit" else (0, 0)
    resident = L.lsk_resident_plan(n_loc, m_loc, r) if C.comm is None else 0
    stream = torch.cuda.current_stream()
    Xi = Ze = None
    if variant == "stream":
        Xi = torch.empty((n_loc, r), dtype=torch.float32, device=C.dev)
        Ze = torch.empty((m_loc, r), dtype=torch.float32, device=C.dev)

    def step(ev_k0, ev_k1):
        p = L.lsk_feature_params_init(eps, d, r, 0.0, cfg.anchor_seed, X, Y, comm=C.comm)
        L.lsk_draw_anchors(p, U)
        if variant == "stream":
            L.lsk_feature_map(p, U, X, Xi)
            L.lsk_feature_map(p, U, Y, Ze)
            if ev_k0 is not None:
                ev_k0.record(stream)
            L.lsk_factored_sinkhorn(Xi, Ze, a, b, eps, opts, u, v, report=False, comm=C.comm)
        else:
            if ev_k0 is not None:
                ev_k0.record(stream)
            L.lsk_factored_sinkhorn_implicit(p, U, X, Y, a, b, opts, u, v, report=False,
                                             comm=C.comm)
        if ev_k1 is not None:
            ev_k1.record(stream)
        # read-out on the host (the step's result): fp64 ROT, all-reduced over the ranks
        return L.lsk_rot_value(u, v, a, b, eps, comm=C.comm)

    tot_ms, kmean, launches, clk, rot = _timed_loop(C, step, steps, warmup, sample_clocks)
    out = {"value": T * steps / (tot_ms / 1e3), "unit": UNIT, "ms_per_step": tot_ms / steps,
           "kernel_ms": kmean, "gpu_launches": launches, "clocks": clk, "rot": rot,
           "roofline": _roofline(variant, cfg.key, r, n_loc, m_loc, T, kmean, stream_rows=srows,
                                 resident=resident),
           "config": {"workload": "config%d-%s" % (cfg.key, cfg.name),
                      "variant": variant + ("-hybrid" if srows[0] + srows[1] else "")
                                 + ("-resident%d" % resident if resident else ""),
                      "stream_rows": list(srows),
                      "global_n": gn, "global_m": gm, "n_per_gpu": n_loc, "m_per_gpu": m_loc,
                      "d": d, "r": r, "eps": eps, "T": T, "scaling": scaling,
                      "parallelism": "rows%d" % ws if ws > 1 else "single",
                      "exchange": C.exchange,
                      "l2": "flushed (256 MiB write) before every timed step"},
           "_host": full}
    return out


def measure_batched(C, cfg, scaling, steps, warmup, sample_clocks=True):
    """Config 4: B independent pairs in one batched solve per step (shared anchor draw, R over
    all pairs; tcgen05 feature maps; one persistent batched Sinkhorn launch; batched read-out).
    An iteration is one Sinkhorn iteration of every pair.  Weak scaling: B pairs per GPU;
    strong scaling: the B pairs split over the ranks.  No cross-GPU exchange (independent
    pairs); R is all-reduced (max) so that every rank draws the same anchors."""
    torch, L, ws, rank = C.torch, C.L, C.ws, C.rank
    n, m, r, d, T, eps = cfg.n, cfg.m, cfg.r, cfg.d, cfg.T, cfg.eps
    bp = synth.make_batched(cfg)
    if scaling == "strong" and ws > 1:
        lo, hi = L.lsk_shard_range(cfg.batch, ws, rank)
        bp = {k: (bp[k][lo:hi] if k in ("X", "Y", "a", "b") else bp[k]) for k in bp}
    B = bp["X"].shape[0]
    Xh, Yh, ah, bh = (torch.from_numpy(np.ascontiguousarray(bp[k])).pin_memory()
                      for k in ("X", "Y", "a", "b"))
    X, Y, a, b = (t.to(C.dev) for t in (Xh, Yh, ah, bh))
    U = torch.empty((r, d), dtype=torch.float32, device=C.dev)
    Xi = torch.empty((B, n, r), dtype=torch.float32, device=C.dev)
    Ze = torch.empty((B, m, r), dtype=torch.float32, device=C.dev)
    u = torch.empty((B, n), dtype=torch.float32, device=C.dev)
    v = torch.empty((B, m), dtype=torch.float32, device=C.dev)
    opts = L.make_opts(T)
    stream = torch.cuda.current_stream()

    def step_on(Xs, Ys, As, Bs, ev_k0, ev_k1):
        p = L.lsk_feature_params_init(eps, d, r, 0.0, cfg.anchor_seed, Xs.reshape(-1, d),
                                      Ys.reshape(-1, d), comm=C.comm)
        L.lsk_draw_anchors(p, U)
        L.lsk_feature_map_batched(p, U, Xs, Xi)
        L.lsk_feature_map_batched(p, U, Ys, Ze)
        if ev_k0 is not None:
            ev_k0.record(stream)
        L.lsk_factored_sinkhorn_batched(Xi, Ze, As, Bs, eps, opts, u, v, report=False)
        if ev_k1 is not None:
            ev_k1.record(stream)
        return L.lsk_rot_value_batched(u, v, As, Bs, eps)

    tot_ms, kmean, launches, clk, rots = _timed_loop(
        C, lambda k0, k1: step_on(X, Y, a, b, k0, k1), steps, warmup, sample_clocks)
    value = T * steps / (tot_ms / 1e3) * (ws if scaling == "weak" else 1)
    return {"value": value, "unit": UNIT, "ms_per_step": tot_ms / steps, "kernel_ms": kmean,
            "gpu_launches": launches, "clocks": clk, "rot_pair0": rots[0] if rots else None,
            "roofline": _roofline("stream", cfg.key, r, n, m, T, kmean, batch=B),
            "config": {"workload": "config%d-%s" % (cfg.key, cfg.name),
                       "variant": "stream-batched", "batch_global": B * ws if scaling == "weak" else cfg.batch,
                       "batch_per_gpu": B, "n": n, "m": m, "d": d, "r": r, "eps": eps, "T": T,
                       "iteration": "one Sinkhorn iteration of every pair",
                       "pair_iterations_per_s": value * (B * ws if scaling == "weak" else cfg.batch),
                       "scaling": scaling,
                       "parallelism": "pairs%d" % ws if ws > 1 else "single",
                       "l2": "flushed (256 MiB write) before every timed step"},
            "_step_on": step_on, "_host": (Xh, Yh, ah, bh), "_B": B}


def _e2e_single(C, cfg, variant, host, steps, warmup):
    """The same metric end to end through the public host-buffer entry point lsk_rot_host:
    pinned host inputs copied in, a1-a9 on the device, u, v and the report copied back, all
    inside the timed region (N=1)."""
    torch, L = C.torch, C.L
    Xh, Yh, ah, bh = (torch.from_numpy(host[k]).pin_memory() for k in ("X", "Y", "a", "b"))
    n, m, d = Xh.shape[0], Yh.shape[0], Xh.shape[1]
    uh = torch.empty(n, dtype=torch.float32).pin_memory()
    vh = torch.empty(m, dtype=torch.float32).pin_memory()
    vcode = 2 if variant == "implicit" else 1
    opts = L.make_opts(cfg.T)
    for _ in range(max(1, warmup)):
        L.lsk_rot_host(Xh, Yh, ah, bh, cfg.eps, cfg.r, cfg.anchor_seed, opts, variant=vcode,
                       u_out=uh, v_out=vh)
    ts = []
    for _ in range(steps):
        C.flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.lsk_rot_host(Xh, Yh, ah, bh, cfg.eps, cfg.r, cfg.anchor_seed, opts, variant=vcode,
                       u_out=uh, v_out=vh)
        ts.append(time.perf_counter() - t0)
    return {"value": cfg.T * len(ts) / float(np.sum(ts)), "unit": UNIT,
            "h2d_bytes_per_step": 4 * (n * d + m * d + n + m),
            "d2h_bytes_per_step": 4 * (n + m) + 48}


def _e2e_batched(C, cfg, mb, steps):
    torch = C.torch
    Xh, Yh, ah, bh = mb["_host"]
    B = mb["_B"]
    ts = []
    for _ in range(steps):
        C.flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Xs, Ys, As, Bs = (t.to(C.dev, non_blocking=True) for t in (Xh, Yh, ah, bh))
        mb["_step_on"](Xs, Ys, As, Bs, None, None)   # rot values come back to the host
        ts.append(time.perf_counter() - t0)
    return {"value": cfg.T * len(ts) / float(np.sum(ts)), "unit": UNIT,
            "h2d_bytes_per_step": 4 * B * (cfg.n * cfg.d + cfg.m * cfg.d + cfg.n + cfg.m),
            "d2h_bytes_per_step": 8 * B}


def _public(d):
    return {k: v for k, v in d.items() if not k.startswith("_")}


def run_lsk(args):
    C = Ctx(args)
    ws, rank = C.ws, C.rank
    cfg = synth.get_config(args.config)
    variant = args.variant
    if variant == "auto":
        # measured: the MUFU-recompute variant is faster where it applies
        # (d <= 8: configs 1, 2, 5); the factor stream elsewhere (configs 3, 4)
        variant = "implicit" if cfg.d <= 8 else "stream"
    if cfg.batch > 1:
        main_m = measure_batched(C, cfg, args.scaling, args.steps, args.warmup)
    else:
        main_m = measure_single(C, cfg, variant, args.scaling, args.steps, args.warmup)
    result = {
        "metric": METRIC, "value": main_m["value"], "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_m["ms_per_step"],
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": main_m["config"], "roofline": main_m["roofline"],
        "kernel_ms": main_m["kernel_ms"], "gpu_launches": main_m["gpu_launches"],
        "clocks": main_m["clocks"],
    }
    if "rot" in main_m:
        result["rot"] = main_m["rot"]
    else:
        result["rot_pair0"] = main_m["rot_pair0"]
    # the other variant on the same workload (same protocol), for the comparison the variant
    # choice rests on (d <= 8: both apply)
    if ws == 1 and not args.no_alt and cfg.d <= 8 and cfg.batch == 1:
        alts = []
        if variant == "implicit" and "hybrid" in result["config"]["variant"]:
            alts.append(("implicit", -1.0))   # pure recompute (the hybrid's MUFU-only twin)
        elif variant == "implicit" and cfg.r <= 1024 and cfg.d <= 3:
            alts.append(("implicit", 0.25))   # the opt-in hybrid (MUFU + HBM) on the same workload
        alts.append(("stream" if variant == "implicit" else "implicit", 0.0))
        result["alt_variants"] = []
        for alt, sf in alts:
            m = measure_single(C, cfg, alt, args.scaling, args.steps, args.warmup, False,
                               stream_fraction=sf)
            result["alt_variants"].append({"variant": m["config"]["variant"], "value": m["value"],
                                           "unit": UNIT, "ms_per_step": m["ms_per_step"],
                                           "kernel_ms": m["kernel_ms"], "roofline": m["roofline"],
                                           "rot": m["rot"]})
    # end to end through the public host-buffer entry point (N=1)
    if ws == 1 and not args.no_e2e:
        if cfg.batch > 1:
            result["e2e"] = _e2e_batched(C, cfg, main_m, args.steps)
        else:
            result["e2e"] = _e2e_single(C, cfg, variant, main_m["_host"], args.steps, args.warmup)
    else:
        result["e2e"] = None
    main_m = None
    # the other BASELINE.json configs at full size, strong scaling over the ranks (config 5:
    # north_star's sharded largest config); parity of each: tests/test_gpu_full.py
    if not args.no_extra:
        extra = {}
        for k in args.extra_configs:
            if k == cfg.key:
                continue
            ck = synth.get_config(k)
            ks, kw = min(args.steps, args.extra_steps), max(3, min(args.warmup, 3))
            if ck.batch > 1:
                mk = measure_batched(C, ck, "strong", ks, kw)
            else:
                vk = "implicit" if ck.d <= 8 else "stream"
                mk = measure_single(C, ck, vk, "strong", ks, kw)
            mk["steps"], mk["warmup"] = ks, kw
            extra["config%d" % k] = _public(mk)
            mk = None
            C.torch.cuda.empty_cache()
        result["configs"] = extra
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, iters=args.ref_iters)
    C.close()
    if rank == 0:
        print(json.dumps(result))
    return 0


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks on this node with
    torch.distributed.run (rendezvous on 127.0.0.1) and forward rank 0's line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="headline config: weak = N x the config's rows (pairs), strong = the "
                         "config's rows (pairs) split over the N GPUs")
    ap.add_argument("--extra-configs", type=int, nargs="*", default=[1, 3, 4, 5])
    ap.add_argument("--extra-steps", type=int, default=2)
    ap.add_argument("--no-extra", action="store_true", help="skip the configs 3/4/5 lines")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lsk", choices=["lsk", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--variant", default="auto", choices=["auto", "stream", "implicit"])
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--ref-iters", type=int, default=20,
                    help="oracle iterations timed per sample (reference arm and cpu_baseline)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip timing the other variant")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "lsk":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if ws is not None and int(ws) != args.gpus:
        print("error: WORLD_SIZE=%s but --gpus %d" % (ws, args.gpus), file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_lsk(args)


if __name__ == "__main__":
    sys.exit(main())
