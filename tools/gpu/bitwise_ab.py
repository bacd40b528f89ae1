"""Bitwise comparison of two librpca.so builds on the same inputs (pca over
dense fp64 / fp32-centred / CSR, l across the padded widths):
   python tools/gpu/bitwise_ab.py <libA> <libB> [case name] [repetitions]"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

mods = []
for i, lib in enumerate(sys.argv[1:3]):
    os.environ["RPCA_LIB_PATH"] = os.path.abspath(lib)
    spec = importlib.util.spec_from_file_location(f"rpvar{i}", os.path.join(ROOT, "paper_1412_3510_b200", "__init__.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    mods.append(m)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
cases = []
A64 = torch.randn(300001, 700, generator=g, device=dev, dtype=torch.float64)
A32 = (torch.randn(400000, 600, generator=g, device=dev, dtype=torch.float32) + 3.0)
r, c, v = synth.make_c5(m=2000000, n=100000, seed=3, device=dev, planted_rows=20000, planted_cols=200)
for l in (6, 12, 22, 32, 40, 52, 64):
    cases.append((f"f64 l={l}", lambda rp, l=l: rp.pca(A64, l - 2, raw=True, its=2, l=l, seed=0)))
    cases.append((f"f32c l={l}", lambda rp, l=l: rp.pca(A32, l - 2, raw=False, its=2, l=l, seed=0)))
for l in (12, 32):
    cases.append((f"csr l={l}", lambda rp, l=l: rp.pca(rp.CSR(r, c, v, (2000000, 100000)), l - 2, raw=True, its=2,
                                                      l=l, seed=0)))
only = sys.argv[3] if len(sys.argv) > 3 else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cases = [c for c in cases if only is None or c[0] == only] * reps
bad = 0
for name, f in cases:
    o = [[t.cpu() for t in f(rp)] for rp in mods]
    same = all(torch.equal(a, b) for a, b in zip(o[0], o[1]))
    bad += not same
    print(f"{name:12s} {'bitwise equal' if same else 'DIFFERENT'}", flush=True)
print(f"{len(cases)} cases, {bad} different")
