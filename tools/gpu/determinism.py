"""Run-to-run bitwise determinism of single library calls: the fp32 tcgen05
passes (A·X, Aᵀ·Y, centred and raw), the fp64 DMMA passes and a centred fp32
PCA, each repeated R times on the same inputs.
   python tools/gpu/determinism.py [R]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1412_3510_b200 as rp  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
A32 = torch.randn(400000, 600, generator=g, device=dev, dtype=torch.float32) + 3.0
A64 = torch.randn(300001, 700, generator=g, device=dev, dtype=torch.float64)
cm = A32.double().mean(0)
for l in (22, 32, 40, 52, 64):
    X = torch.randn(600, l, generator=g, device=dev, dtype=torch.float64)
    Q = torch.randn(400000, l, generator=g, device=dev, dtype=torch.float64)
    X64 = torch.randn(700, l, generator=g, device=dev, dtype=torch.float64)
    Q64 = torch.randn(300001, l, generator=g, device=dev, dtype=torch.float64)
    cases = {
        "f32 A·X": lambda: rp.apply(A32, X),
        "f32 Aᵀ·Y": lambda: rp.apply(A32, Q, adjoint=True),
        "f32 Aᵀ·Y centred": lambda: rp.apply(A32, Q, adjoint=True, cmean=cm),
        "f64 A·X": lambda: rp.apply(A64, X64),
        "f64 Aᵀ·Y": lambda: rp.apply(A64, Q64, adjoint=True),
        **({"f64 A·X int8 emu": lambda: rp.apply_int8emu(A64, X64)} if 24 < l <= 48 else {}),
        "f32c pca": lambda: torch.cat([t.flatten().double().cpu() for t in
                                       rp.pca(A32, l - 2, raw=False, its=2, l=l, seed=0)]),
    }
    for name, f in cases.items():
        ref = f().clone()
        nd = 0
        for _ in range(R):
            nd += not torch.equal(f(), ref)
        print(f"l={l:2d} {name:18s} {'deterministic' if nd == 0 else f'DIFFERS in {nd}/{R}'}", flush=True)
