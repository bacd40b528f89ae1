"""Per-kernel times of rp.lu_renorm on the configs' block shapes — LU tuning aid.

  python tools/gpu/lu_micro.py [m:l,m:l,...]
Run once with and once without RPCA_LU_F64_LEAF=1 to compare the fp32
nomination levels against the fp64 ones; also prints max|L| and the span
agreement with the fp64-nomination L (sin of the largest principal angle).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1412_3510_b200 as rp  # noqa: E402

dev = torch.device("cuda", 0)
shapes = [tuple(int(v) for v in s.split(":")) for s in
          (sys.argv[1] if len(sys.argv) > 1 else "100000:22,32768:42,2000000:52,10000000:32,1000000:32").split(",")]
for m, l in shapes:
    g = torch.Generator(device="cuda").manual_seed(m + l)
    # a block with a decaying spectrum, like A·Q in the power rounds
    Y = torch.randn(m, l, generator=g, device=dev, dtype=torch.float64) * torch.logspace(
        0, -3, l, device=dev, dtype=torch.float64)
    for _ in range(3):
        rp.lu_renorm(Y.clone())
    torch.cuda.synchronize()
    Ys = [Y.clone() for _ in range(5)]
    with rp.profile() as p:
        for Yc in Ys:
            rp.lu_renorm(Yc)
        torch.cuda.synchronize()
    agg = {}
    for name, ms in p.records:
        c, s = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, s + ms)
    L = Ys[0]
    if m * l > 1e8:  # torch.linalg on 10M-row blocks: skip the span check
        sin = float("nan")
    else:
        Q = torch.linalg.qr(L)[0]
        Qy = torch.linalg.qr(Y)[0]
        sin = float(torch.linalg.matrix_norm(Qy - Q @ (Q.T @ Qy), 2))
    tot = sum(v[1] for v in agg.values()) / 5
    print(f"m={m:9d} l={l:2d} total {1e3 * tot:8.1f}us  maxL {float(L.abs().max()):.3g} sin(Y,L) {sin:.1e}  " +
          " ".join(f"{k}:{v[0] // 5}x{1e3 * v[1] / 5:.1f}us" for k, v in agg.items()), flush=True)
# per-launch times of one LU (the tree levels in order)
if os.environ.get("LU_LEVELS"):
    for m, l in shapes:
        g = torch.Generator(device="cuda").manual_seed(m + l)
        Y = torch.randn(m, l, generator=g, device=dev, dtype=torch.float64)
        rp.lu_renorm(Y.clone())
        torch.cuda.synchronize()
        with rp.profile() as p:
            rp.lu_renorm(Y.clone())
            torch.cuda.synchronize()
        print(f"m={m} l={l} levels:", " ".join(f"{n}:{1e3 * ms:.0f}" for n, ms in p.records), flush=True)
