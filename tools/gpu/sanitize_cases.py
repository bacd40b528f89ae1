"""Small calls of every kernel family of librpca.so, for compute-sanitizer
(memcheck / racecheck / synccheck) — SURVEY.md §4 tier T5.

  compute-sanitizer --tool racecheck python tools/gpu/sanitize_cases.py
Each case is tiny so the instrumented run finishes in minutes; the cases are
chosen so that every kernel the pipelines launch runs at least once: dense fp64
(DMMA passes, tournament LU, LU-Cholesky-QR, Jacobi), the int8-emulated A·X
(l = 30), fp32 (tcgen05 3×TF32 passes), CSR (SpMM, heavy rows, transpose),
Nyström (both variants), reig, diffsnorm, the Householder TSQR and its
fallback, and the finite check.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1412_3510_b200 as rp  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["all"]


def on(name):
    return "all" in which or name in which


g = torch.Generator(device="cuda").manual_seed(0)
if on("dense"):
    A = synth.make_c1(m=1100, n=300, device=dev)
    r = rp.pca(A, 10, its=2, l=12, check_finite=True)
    rp.diffsnorm(A, *r, its=3)
    rp.pca(A, 10, raw=False, its=1, l=12)
    rp.pca(A.T.contiguous(), 8, its=1, l=10)  # m < n
if on("emu"):
    A = synth.make_c1(m=700, n=260, device=dev)
    rp.pca(A, 28, its=2, l=30)
    rp.apply_int8emu(A, torch.randn(260, 30, generator=g, device=dev, dtype=torch.float64))
if on("f32"):
    A = synth.make_c4(m=3000, n=256, device=dev)
    rp.pca(A, 20, raw=False, its=2, l=22)
    rp.apply(A, torch.randn(256, 52, generator=g, device=dev, dtype=torch.float64))
if on("csr"):
    rp_, ci, va = synth.make_c5(m=6000, n=5000, seed=2, device=dev, planted_rows=60, planted_cols=4500)
    A = rp.CSR(rp_, ci, va, (6000, 5000))
    r = rp.pca(A, 10, its=1, l=12)
    rp.diffsnorm(A, *r, its=2)
if on("nystrom"):
    P = synth.make_c3(n=400, device=dev)
    rp.eigens(P, 10, its=1, l=12)
    rp.eigens(P, 10, its=1, l=12, variant="sqrt")
    rp.reig(P, 10, its=1, l=12)
if on("qr"):
    Y = torch.randn(3000, 20, generator=g, device=dev, dtype=torch.float64)
    rp.qr(Y)
    rp.lu_renorm(Y)
    Yw = torch.zeros(600, 40, dtype=torch.float64, device=dev)
    Yw[:40] = torch.tril(-torch.ones(40, 40, dtype=torch.float64, device=dev), -1) + torch.eye(
        40, dtype=torch.float64, device=dev)
    rp.orthonormalize(Yw)  # breakdown → Householder fallback
    rp.small_svd(torch.randn(500, 22, generator=g, device=dev, dtype=torch.float64))
torch.cuda.synchronize()
print("sanitize cases done:", which, "launches", rp.launch_count())
