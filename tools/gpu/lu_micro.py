"""Per-kernel times of rp.lu_renorm for a sweep of (m, l) — LU tuning aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1412_3510_b200 as rp
dev = torch.device("cuda", 0)
for l in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8,16,22,32,42,52,64").split(",")]:
    for m in [256, 4096, 100000, 2000000]:
        Y = torch.randn(m, l, device=dev, dtype=torch.float64)
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
        print(f"l={l:2d} m={m:8d} " + " ".join(f"{k}:{v[0]//5}x {1e3*v[1]/5:.1f}us" for k, v in agg.items()), flush=True)
