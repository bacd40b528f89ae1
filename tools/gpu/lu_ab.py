"""A/B of two library builds on rp.lu_renorm (one process, interleaved):
   python tools/gpu/lu_ab.py <libA> <libB> [m:l,...]
Checks that both builds choose the same pivots and give bitwise-equal U and
L, then prints per-kernel µs per LU for each build."""
import importlib.util
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
mods = []
for i, lib in enumerate(sys.argv[1:3]):
    os.environ["RPCA_LIB_PATH"] = os.path.abspath(lib)
    spec = importlib.util.spec_from_file_location(f"rpvar{i}", os.path.join(root, "paper_1412_3510_b200", "__init__.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    mods.append(m)
shapes = [tuple(int(v) for v in s.split(":")) for s in
          (sys.argv[3] if len(sys.argv) > 3 else
           "4000:22,100000:22,32768:42,2000000:52,10000000:32,1000000:32,300000:8,300000:16,300000:24,"
           "300000:40,300000:48,300000:64,1000:1,777:5").split(",")]
dev = torch.device("cuda", 0)
for m, l in shapes:
    g = torch.Generator(device="cuda").manual_seed(m + l)
    Y = torch.randn(m, l, generator=g, device=dev, dtype=torch.float64) * torch.logspace(
        0, -3, l, device=dev, dtype=torch.float64)
    outs = [rp.lu_renorm(Y) for rp in mods]
    same = all(torch.equal(a, b) for a, b in zip(outs[0], outs[1]))
    line = f"m={m:9d} l={l:2d} identical={same}"
    if not same:
        line += f" piv_equal={torch.equal(outs[0][2], outs[1][2])} maxdiffL={float((outs[0][0] - outs[1][0]).abs().max()):.3g}"
    for rp in mods:
        for _ in range(2):
            rp.lu_renorm(Y)
        torch.cuda.synchronize()
        with rp.profile() as p:
            for _ in range(5):
                rp.lu_renorm(Y)
            torch.cuda.synchronize()
        agg = {}
        for name, ms in p.records:
            c, s = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, s + ms)
        tot = sum(v[1] for v in agg.values()) / 5
        line += f" | {1e3 * tot:8.1f}us " + " ".join(
            f"{k}:{v[0] // 5}x{1e3 * v[1] / 5:.0f}" for k, v in agg.items() if k.startswith("lu_"))
    print(line, flush=True)
