"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times, against the oracle on the same
bytes with BASELINE north_star's tolerances: leading-k σ relative 1e-10 (fp64)
/ 1e-4 (fp32), largest principal angle (sine form, per σ cluster) < 1e-8 /
1e-3, and diffsnorm within 1% of the oracle's.

* C2 (fp64 100000×4000) is in test_gpu_parity.py (plus its diffsnorm here).
* C3 (Nyström, fp64 32768²): `eigens` and its diffsnorm (V = U, S = λ).
* C4 (centred fp32 2e6×4096): the whole `pca` and diffsnorm against the oracle
  (≈ 4 min of oracle time on 16 cores), plus the pass kernels on sampled rows
  and the properties that hold at any size (orthonormality, A_cᵀU = V·S,
  Rayleigh–Ritz interlacing against the exact σ of the fp64 Gram).
* C5 (CSR 1e7×1e6): the whole `pca` and diffsnorm against the oracle, plus the
  SpMM passes on sampled rows and against cuSPARSE.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1412_3510_b200 as rp
import synth
from tests.helpers import cluster_sin_angle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def dev():
    return torch.device("cuda", 0)


def diffsnorm_pair(A, A_host, res_g, res_o, raw, same_factors=True):
    """GPU diffsnorm of the GPU factors vs the oracle's of its own factors (≤ 1%,
    BASELINE), and both estimators on the SAME factors (same algorithm, same
    start vector: agreement to rounding)."""
    est = rp.diffsnorm(A, *res_g, raw=raw, its=20, seed=1)
    ref = oracle.diffsnorm(A_host, *res_o, raw=raw, its=20, seed=1)
    assert abs(est - ref) <= 0.01 * ref, (est, ref)
    if same_factors:  # fp64 A: the two estimators differ by rounding only
        same = oracle.diffsnorm(A_host, *[t.cpu().numpy() for t in res_g], raw=raw, its=20, seed=1)
        assert abs(est - same) <= 1e-9 * same, (est, same)
    return est, ref


def test_c3_full_vs_oracle():
    cfg = synth.CONFIGS["C3"]
    A = synth.make_c3(device=dev())
    U, lam = rp.eigens(A, cfg.k, its=cfg.its, l=cfg.l, seed=0)
    Ah = A.cpu().numpy()
    Uo, lo = oracle.eigens(Ah, cfg.k, its=cfg.its, l=cfg.l, seed=0)
    lg = lam.cpu().numpy()
    assert np.max(np.abs(lg - lo) / lo) < 1e-10
    assert cluster_sin_angle(Uo, U.cpu().numpy(), lo, cfg.k) < 1e-8
    # Nyström factors: V = U, S = λ (include/rpca.h)
    est = rp.diffsnorm(A, U, lam, U, its=20, seed=1)
    ref = oracle.diffsnorm(Ah, Uo, lo, Uo, its=20, seed=1)
    assert abs(est - ref) <= 0.01 * ref, (est, ref)
    assert est >= 1.0 / (cfg.k + 1) ** 2 * (1 - 1e-2)  # ≥ λ_{k+1} (power method: from below) (Eckart–Young, exact spectrum j^-2)


def test_c2_full_diffsnorm():
    cfg = synth.CONFIGS["C2"]
    A = synth.make_c2(device=dev())
    res = rp.pca(A, cfg.k, raw=True, its=cfg.its, l=cfg.l, seed=0)
    Ah = A.cpu().numpy()
    o = oracle.pca(Ah, cfg.k, its=cfg.its, l=cfg.l, seed=0)
    diffsnorm_pair(A, Ah, res, o, True)


def test_c4_full_vs_oracle():
    """C4 at full size: 2e6×4096 fp32, centred, k=50, l=52, its=4 — the whole
    pipeline against the oracle (fp32 tolerances of BASELINE)."""
    cfg = synth.CONFIGS["C4"]
    A = synth.make_c4(device=dev())
    res = rp.pca(A, cfg.k, raw=False, its=cfg.its, l=cfg.l, seed=0)
    Ah = A.cpu().numpy()
    o = oracle.pca(Ah, cfg.k, raw=False, its=cfg.its, l=cfg.l, seed=0)
    Sg = res[1].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(Sg - o[1]) / o[1]) < 1e-4
    assert cluster_sin_angle(o[0], res[0].cpu().numpy().astype(np.float64), o[1], cfg.k) < 1e-3
    assert cluster_sin_angle(o[2], res[2].cpu().numpy().astype(np.float64), o[1], cfg.k) < 1e-3
    diffsnorm_pair(A, Ah, res, o, False, same_factors=False)  # (≈ 90 s of oracle time per estimate)


def test_c5_full_vs_oracle():
    """C5 at full size: CSR 1e7×1e6 (≈1.2e8 nonzeros), k=30, l=32, its=2 — the whole
    pipeline against the oracle (fp64 tolerances)."""
    cfg = synth.CONFIGS["C5"]
    rowptr, colind, vals = synth.make_c5(device=dev())
    A = rp.CSR(rowptr, colind, vals, (cfg.m, cfg.n))
    res = rp.pca(A, cfg.k, raw=True, its=cfg.its, l=cfg.l, seed=0)
    host = (rowptr.cpu().numpy(), colind.cpu().numpy(), vals.cpu().numpy(), (cfg.m, cfg.n))
    o = oracle.pca(host, cfg.k, raw=True, its=cfg.its, l=cfg.l, seed=0)
    Sg = res[1].cpu().numpy()
    assert np.max(np.abs(Sg - o[1]) / o[1]) < 1e-10
    assert cluster_sin_angle(o[0], res[0].cpu().numpy(), o[1], cfg.k) < 1e-8
    assert cluster_sin_angle(o[2], res[2].cpu().numpy(), o[1], cfg.k) < 1e-8
    diffsnorm_pair(A, host, res, o, True)


def _chunks(m, size=1 << 17):
    for i0 in range(0, m, size):
        yield i0, min(m, i0 + size)


def test_c4_full_properties():
    cfg = synth.CONFIGS["C4"]
    A = synth.make_c4(device=dev())
    m, n = A.shape
    # (a) the fp32 passes at full size on sampled rows: |gpu − exact| within
    # the 3×TF32 + fp32-accumulation bound of test_apply_f32_input
    g = torch.Generator(device="cuda").manual_seed(4)
    X = torch.randn(n, cfg.l, generator=g, device=dev(), dtype=torch.float64)
    Y = rp.apply(A, X)
    rows = torch.randint(0, m, (64,), generator=g, device=dev())
    Ar = A[rows].double()
    exact = Ar @ X
    bound = (3 * 2.0**-21 + 2 * n * 2.0**-24) * (Ar.abs() @ X.abs())
    assert bool(((Y[rows] - exact).abs() <= bound).all())
    Q = torch.randn(m, cfg.l, generator=g, device=dev(), dtype=torch.float64)
    Z = rp.apply(A, Q, adjoint=True)
    cols = torch.randint(0, n, (16,), generator=g, device=dev())
    ex = torch.zeros(16, cfg.l, dtype=torch.float64, device=dev())
    ab = torch.zeros_like(ex)
    for i0, i1 in _chunks(m):
        Ac = A[i0:i1, cols].double()
        ex += Ac.T @ Q[i0:i1]
        ab += Ac.abs().T @ Q[i0:i1].abs()
    bound = (3 * 2.0**-21 + 2 * 4096 * 2.0**-24 + 1e-12) * ab
    assert bool(((Z[cols] - ex).abs() <= bound).all())
    del Y, Q, Z

    # (b) the whole centred PCA: orthonormality, A_cᵀU = V S, interlacing
    U, S, V = rp.pca(A, cfg.k, raw=False, its=cfg.its, l=cfg.l, seed=0)
    Ud, Sd, Vd = U.double(), S.double(), V.double()
    k = cfg.k
    eye = torch.eye(k, dtype=torch.float64, device=dev())
    assert float(torch.linalg.norm(Ud.T @ Ud - eye)) < 1e-4
    assert float(torch.linalg.norm(Vd.T @ Vd - eye)) < 1e-4
    assert bool((Sd[:-1] >= Sd[1:]).all()) and bool((Sd >= 0).all())
    mu = torch.zeros(n, dtype=torch.float64, device=dev())
    for i0, i1 in _chunks(m):
        mu += A[i0:i1].double().sum(0)
    mu /= m
    AtU = torch.zeros(n, k, dtype=torch.float64, device=dev())
    G = torch.zeros(n, n, dtype=torch.float64, device=dev())
    for i0, i1 in _chunks(m):
        Ac = A[i0:i1].double() - mu
        AtU += Ac.T @ Ud[i0:i1]
        G += Ac.T @ Ac
    # fp32 arithmetic on the uncentred A (column means ~U(−5,5) ≫ the data's
    # spread) bounds the identity to ~1e-4·S_0: 3×TF32 products with fp32
    # accumulation over 4096 rows, fp64 across chunks (reading Q15)
    res = float(torch.linalg.norm(AtU - Vd * Sd)) / float(Sd[0])
    assert res < 2e-4, res
    sig = torch.sqrt(torch.clamp(torch.linalg.eigvalsh(G).flip(0)[:k], min=0))
    ratio = (Sd / sig).cpu().numpy()
    assert np.all(ratio <= 1 + 1e-5), ratio
    assert np.all(ratio[:10] >= 1 - 1e-4), ratio


def test_c5_full_properties():
    cfg = synth.CONFIGS["C5"]
    rowptr, colind, vals = synth.make_c5(device=dev())
    m, n = cfg.m, cfg.n
    A = rp.CSR(rowptr, colind, vals, (m, n))
    T = torch.sparse_csr_tensor(rowptr, colind.long(), vals, (m, n))
    g = torch.Generator(device="cuda").manual_seed(5)
    # (a) the SpMM passes: sampled rows of A·X recomputed from their CSR rows
    X = torch.randn(n, cfg.l, generator=g, device=dev(), dtype=torch.float64)
    Y = rp.apply(A, X)
    rp_h, ci_h, va_h = rowptr.cpu().numpy(), colind.cpu().numpy(), vals.cpu().numpy()
    Xh = X.cpu().numpy()
    Yh = Y.cpu().numpy()
    rs = np.random.default_rng(5).choice(m, 64, replace=False)
    for i in rs:
        c, v = ci_h[rp_h[i]:rp_h[i + 1]], va_h[rp_h[i]:rp_h[i + 1]]
        ex = v @ Xh[c]
        bound = 2 * len(c) * 2.0**-53 * (np.abs(v) @ np.abs(Xh[c])) + 1e-300
        assert np.all(np.abs(Yh[i] - ex) <= bound)
    # Aᵀ·Y on CSR(Aᵀ) (heavy rows chunked) against cuSPARSE's fp64 product
    Q = torch.randn(m, cfg.l, generator=g, device=dev(), dtype=torch.float64)
    Z = rp.apply(A, Q, adjoint=True)
    Zr = torch.sparse.mm(T.to_sparse_coo().t(), Q)
    rel = float(torch.linalg.norm(Z - Zr)) / float(torch.linalg.norm(Zr))
    assert rel < 1e-13, rel
    del Y, Q, Z, Zr
    # (b) the whole PCA: orthonormality and AᵀU = V S
    U, S, V = rp.pca(A, cfg.k, raw=True, its=cfg.its, l=cfg.l, seed=0)
    k = cfg.k
    eye = torch.eye(k, dtype=torch.float64, device=dev())
    assert float(torch.linalg.norm(U.T @ U - eye)) < 1e-10
    assert float(torch.linalg.norm(V.T @ V - eye)) < 1e-10
    AtU = torch.sparse.mm(T.to_sparse_coo().t(), U)
    res = float(torch.linalg.norm(AtU - V * S)) / float(S[0])
    assert res < 1e-10, res


def test_c4_scaled_vs_oracle():
    """The C4 recipe at m = 1e5, n = 1024 (SURVEY.md §8(c) c.4's proxy): the whole
    centred fp32 PCA against the oracle — BASELINE's fp32 tolerances (σ 1e-4,
    principal angles 1e-3)."""
    cfg = synth.CONFIGS["C4"]
    A = synth.make_c4(m=100000, n=1024, device=dev())
    U, S, V = rp.pca(A, cfg.k, raw=False, its=cfg.its, l=cfg.l, seed=0)
    Uo, So, Vo = oracle.pca(A.cpu().numpy(), cfg.k, raw=False, its=cfg.its, l=cfg.l, seed=0)
    Sg = S.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(Sg - So) / So) < 1e-4
    assert cluster_sin_angle(Uo, U.cpu().numpy().astype(np.float64), So, cfg.k) < 1e-3
    assert cluster_sin_angle(Vo, V.cpu().numpy().astype(np.float64), So, cfg.k) < 1e-3
