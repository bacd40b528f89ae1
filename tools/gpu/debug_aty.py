"""Debug aid: rp.apply(adjoint) on fp32 A vs numpy for small structured cases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1412_3510_b200 as rp
np.set_printoptions(precision=3, linewidth=150)
for (m, n, l) in [(128, 128, 16), (32, 128, 16), (64, 256, 8), (777, 300, 1), (4096, 512, 52), (100000, 4096, 52)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float32)
    Y = torch.randn(m, l, generator=g, device="cuda", dtype=torch.float64)
    X = torch.randn(n, l, generator=g, device="cuda", dtype=torch.float64)
    An = A.cpu().numpy().astype(np.float64)
    z = rp.apply(A, Y, adjoint=True).cpu().numpy()
    zr = An.T @ Y.cpu().numpy()
    y = rp.apply(A, X).cpu().numpy()
    yr = An @ X.cpu().numpy()
    e1 = np.abs(z - zr).max() / np.abs(zr).max()
    e2 = np.abs(y - yr).max() / np.abs(yr).max()
    print(m, n, l, "aty rel", e1, "ax rel", e2, flush=True)
    if e1 > 1e-5 and m <= 1000:
        bad = np.argwhere(np.abs(z - zr) > 1e-4 * np.abs(zr).max())
        print(" bad rows", np.unique(bad[:, 0])[:40], "cols", np.unique(bad[:, 1])[:20])
        print(" z[:4,:4]", z[:4, :4], "\n zr[:4,:4]", zr[:4, :4])
