"""A seeded sweep of shapes across every padded width the kernels are
templated on (l rounded up to 8: 8 … 64, both sides of each boundary), dense
fp64 / fp32 and CSR, raw and centred, m ≥ n and m < n — the GPU pipeline
against the oracle at BASELINE's tolerances (fp64 σ rel 1e-10 and principal
angles 1e-8; fp32 1e-4 / 1e-3).  Spectra decay geometrically (0.8^j; 0.95^j
for fp32, a C4-like range) so every compared cluster is separated from the
rest (tests/helpers.cluster_sin_angle)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1412_3510_b200 as rp
import synth
from tests.helpers import cluster_sin_angle

pytestmark = pytest.mark.gpu


def dev():
    return torch.device("cuda", 0)


# (m, n, k, l, its, raw, kind): l spans 8/9, 16/17, 24/25, 31-33, 40/41, 48/49,
# 56/57, 64 — every LP instantiation of the LU, SVD and pass kernels
CASES = [
    (3000, 300, 6, 8, 2, True, "f64"), (3000, 300, 7, 9, 1, False, "f64"),
    (5000, 400, 14, 16, 2, True, "f64"), (600, 5000, 15, 17, 2, True, "f64"),
    (6000, 350, 22, 24, 2, False, "f64"), (6000, 350, 23, 25, 3, True, "f64"),
    (8000, 300, 29, 31, 2, True, "f64"), (8000, 300, 30, 32, 2, False, "f64"),
    (700, 9000, 31, 33, 2, True, "f64"), (9000, 500, 38, 40, 2, True, "f64"),
    (9000, 500, 39, 41, 1, False, "f64"), (20000, 400, 46, 48, 2, True, "f64"),
    (20000, 400, 47, 49, 2, False, "f64"), (30000, 300, 54, 56, 2, True, "f64"),
    (30000, 300, 55, 57, 2, True, "f64"), (40000, 256, 62, 64, 2, False, "f64"),
    (12000, 600, 20, 22, 2, False, "f32"), (12000, 520, 50, 52, 2, False, "f32"),
    (900, 7000, 30, 32, 2, True, "f32"), (60000, 800, 30, 32, 2, True, "csr"),
    (50000, 900, 20, 22, 2, False, "csr"), (50000, 2000, 50, 52, 1, True, "csr"),
]


def make(m, n, l, kind, seed):
    r = min(m, n)
    # fp32 inputs: a spectrum spanning ~15× over the k values compared, like
    # C4's (10·0.9^j): 3×TF32 products carry ~2^-22 of |A||X|, so σ far below
    # σ_1 would be resolved only to that level (BASELINE's 1e-4 is for C4)
    q = 0.95 if kind == "f32" else 0.8
    sig = torch.tensor([q ** j for j in range(r)], dtype=torch.float64)
    if kind == "csr":
        rowptr, colind, vals = synth.make_c5(m=m, n=n, seed=seed, planted_rows=max(1, m // 100),
                                             planted_cols=min(200, n // 2))
        dense = torch.sparse_csr_tensor(rowptr, colind.long(), vals, (m, n)).to_dense()
        A = rp.CSR(rowptr.to(dev()), colind.to(dev()), vals.to(dev()), (m, n))
        return A, dense.numpy()
    A = synth.synth_dense(m, n, sig, seed=seed)
    if kind == "f32":
        A = A.float()
    An = A.double().numpy()
    return A.to(dev()).contiguous(), An


@pytest.mark.parametrize("m,n,k,l,its,raw,kind", CASES)
def test_sweep_vs_oracle(m, n, k, l, its, raw, kind):
    A, An = make(m, n, l, kind, seed=1000 + l)
    U, S, V = rp.pca(A, k, raw=raw, its=its, l=l, seed=3)
    Uo, So, Vo = oracle.pca(An.astype(np.float32).astype(np.float64) if kind == "f32" else An, k, raw=raw, its=its,
                            l=l, seed=3)
    tol_s, tol_a = (1e-4, 1e-3) if kind == "f32" else (1e-10, 1e-8)
    Sg = S.double().cpu().numpy()
    nz = So > 1e-12 * So[0]
    assert np.max(np.abs(Sg[nz] - So[nz]) / So[nz]) < tol_s, (Sg[:4], So[:4])
    assert cluster_sin_angle(Uo, U.double().cpu().numpy(), So, k) < tol_a
    assert cluster_sin_angle(Vo, V.double().cpu().numpy(), So, k) < tol_a


# Nyström (SHIFT_CHOL and SQRT) and reig across the same widths: PSD
# A = V·diag(0.8^j)·Vᵀ, indefinite A = V·diag(±0.85^j)·Vᵀ (alternating signs)
EIG_CASES = [(1500, 6, 8, 2), (1500, 15, 17, 2), (2000, 22, 24, 1), (2000, 31, 33, 2), (2500, 39, 41, 2),
             (2500, 46, 48, 2), (3000, 55, 57, 1), (3000, 62, 64, 2)]


def sym(n, l, signed):
    q = 0.85 if signed else 0.8
    lam = torch.tensor([q ** j for j in range(n)], dtype=torch.float64)
    if signed:
        lam = lam * (-1.0) ** torch.arange(n, dtype=torch.float64)
    V = synth.haar_columns(n, n, 7 * n + l)
    A = (V * lam) @ V.T
    return (0.5 * (A + A.T)).contiguous()


@pytest.mark.parametrize("n,k,l,its", EIG_CASES)
@pytest.mark.parametrize("variant", ["shift_chol", "sqrt"])
def test_sweep_eigens_vs_oracle(n, k, l, its, variant):
    A = sym(n, l, signed=False)
    U, lam = rp.eigens(A.to(dev()), k, its=its, l=l, seed=5, variant=variant)
    Uo, lo = oracle.eigens(A.numpy(), k, its=its, l=l, seed=5,
                           variant=oracle.SHIFT_CHOL if variant == "shift_chol" else oracle.SQRT)
    lg = lam.cpu().numpy()
    assert np.max(np.abs(lg - lo) / lo) < 1e-10, (lg[:4], lo[:4])
    assert cluster_sin_angle(Uo, U.cpu().numpy(), lo, k) < 1e-8


@pytest.mark.parametrize("n,k,l,its", EIG_CASES)
def test_sweep_reig_vs_oracle(n, k, l, its):
    A = sym(n, l, signed=True)
    U, lam = rp.reig(A.to(dev()), k, its=its, l=l, seed=5)
    Uo, lo = oracle.reig(A.numpy(), k, its=its, l=l, seed=5)
    lg = lam.cpu().numpy()
    assert np.all(np.sign(lg) == np.sign(lo))
    assert np.max(np.abs(lg - lo) / np.abs(lo)) < 1e-10, (lg[:4], lo[:4])
    assert cluster_sin_angle(Uo, U.cpu().numpy(), np.abs(lo), k) < 1e-8
