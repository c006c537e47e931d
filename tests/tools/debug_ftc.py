import os, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O, paper_2006_07057_b200 as L
for (M, r, d) in [(128, 128, 32), (128, 128, 64), (256, 128, 128), (777, 512, 128)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    X = (torch.randn(M, d, device="cuda", generator=g) / np.sqrt(d)).float()
    X /= X.norm(dim=1).max()
    p = L.lsk_feature_params_init(1.0, d, r, 1.0, 7)
    U = torch.empty((r, d), dtype=torch.float32, device="cuda")
    L.lsk_draw_anchors(p, U)
    Xi = torch.empty((M, r), dtype=torch.float32, device="cuda")
    L.lsk_feature_map(p, U, X, Xi)
    torch.cuda.synchronize()
    prm = O.gaussian_params(1.0, d, r, 1.0)
    Uo = O.draw_anchors(r, d, prm["sigma"], 7)
    ref = O.feature_matrix(X.cpu().numpy(), Uo, 1.0, prm["q"]).T
    got = Xi.cpu().double().numpy()
    rel = np.abs(got - ref) / ref
    bad = rel > 1e-3
    print(M, r, d, "max rel %.2e" % rel.max(), "bad rows", np.unique(np.where(bad)[0])[:20], "bad cols", np.unique(np.where(bad)[1])[:10])
    if bad.any():
        i, j = np.argwhere(bad)[0]
        lr = np.log2(got[i, j] / ref[i, j])
        print("  first bad", i, j, got[i, j], ref[i, j], "log2 ratio", lr)
