"""Time the a3 feature map (lsk_feature_map; Lemma 1 / eq. (9)) of both clouds of each
BASELINE.json configuration with CUDA events: configs 1-3 on the FFMA path (d <= 16), config 4
on the tcgen05 path (d = 128, 256 pairs batched), config 5 on a 2^20-row slice per cloud (its
full factors, 275 GB, are never materialised: the implicit solver regenerates them).
Timing only; parity of the map against the oracle lives in tests/test_gpu_parity.py."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


KEYS = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]   # optional: the configs to time
for k in KEYS:
    cfg = synth.get_config(k)
    if k == 4:
        bp = synth.make_batched(cfg)
        X, Y = dev(bp["X"]).reshape(-1, cfg.d), dev(bp["Y"]).reshape(-1, cfg.d)
    else:
        prob = synth.make_problem(cfg)
        X, Y = dev(prob["X"]), dev(prob["Y"])
        if k == 5:
            X, Y = X[: 1 << 20].contiguous(), Y[: 1 << 20].contiguous()
    p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 0.0, cfg.anchor_seed, X, Y)
    U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((X.shape[0], cfg.r), dtype=torch.float32, device="cuda")
    Ze = torch.empty((Y.shape[0], cfg.r), dtype=torch.float32, device="cuda")
    for _ in range(3):
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lsk_feature_map(p, U, X, Xi)
        L.lsk_feature_map(p, U, Y, Ze)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    out_bytes = (X.shape[0] + Y.shape[0]) * cfg.r * 4
    print("config %d feature map, both clouds (%d + %d rows x r = %d, d = %d%s): median %.4f ms "
          "(min %.4f); writes %.3f GB -> %.0f GB/s"
          % (k, X.shape[0], Y.shape[0], cfg.r, cfg.d, ", 2^20-row slice" if k == 5 else "",
             ms, min(ts), out_bytes / 1e9, out_bytes / ms / 1e6), flush=True)
    del Xi, Ze, X, Y
    torch.cuda.empty_cache()
