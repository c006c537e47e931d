"""Time the a3 feature map (lsk_feature_map) on config 4's clouds (256 pairs x 4096 rows,
d = 128, r = 512; the tcgen05 3xTF32 path) with CUDA events, and check a sample of rows
against the fp64 oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2006_07057_b200 as L  # noqa: E402
import synth  # noqa: E402

cfg = synth.get_config(4)
B = 256
g = torch.Generator(device="cuda").manual_seed(5)
X = (torch.randn(B * cfg.n, cfg.d, device="cuda", generator=g) / np.sqrt(cfg.d)).float()
Y = (torch.randn(B * cfg.m, cfg.d, device="cuda", generator=g) / np.sqrt(cfg.d)).float()
X /= X.norm(dim=1).max()
Y /= Y.norm(dim=1).max()
p = L.lsk_feature_params_init(cfg.eps, cfg.d, cfg.r, 1.0, cfg.anchor_seed)
U = torch.empty((cfg.r, cfg.d), dtype=torch.float32, device="cuda")
L.lsk_draw_anchors(p, U)
Xi = torch.empty((X.shape[0], cfg.r), dtype=torch.float32, device="cuda")
Zeta = torch.empty((Y.shape[0], cfg.r), dtype=torch.float32, device="cuda")
for _ in range(3):
    L.lsk_feature_map(p, U, X, Xi)
    L.lsk_feature_map(p, U, Y, Zeta)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.lsk_feature_map(p, U, X, Xi)
    L.lsk_feature_map(p, U, Y, Zeta)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
out_bytes = 2 * X.shape[0] * cfg.r * 4
flops = 3 * 2 * 2 * X.shape[0] * cfg.r * cfg.d
print("feature map, both clouds (2 x %d x %d, d = %d): median %.3f ms (min %.3f); writes %.2f GB "
      "-> %.0f GB/s; 3-term split GEMM %.1f TFLOP/s" % (X.shape[0], cfg.r, cfg.d, ms, min(ts), out_bytes / 1e9,
                                            out_bytes / ms / 1e6, flops / ms / 1e9))
# sample check against the oracle (rows spread over the whole cloud, incl. the last tile)
prm = O.gaussian_params(cfg.eps, cfg.d, cfg.r, 1.0)
Uo = O.draw_anchors(cfg.r, cfg.d, prm["sigma"], cfg.anchor_seed)
idx = np.r_[0:7, 12345, 500000:500003, X.shape[0] - 5:X.shape[0]]
ref = O.feature_matrix(X[idx].cpu().numpy(), Uo, cfg.eps, prm["q"]).T
got = Xi[idx].cpu().double().numpy()
mask = ref > 1e-30
print("sampled rows vs oracle: max rel %.2e" % (np.abs(got[mask] - ref[mask]) / ref[mask]).max())
