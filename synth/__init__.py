"""Seeded synthetic inputs for the randomized-PCA hot path (arXiv 1412.3510).

This module is shared by BOTH sides of every parity check — the CUDA product
(``paper_1412_3510_b200``) and the CPU oracle (``oracle/``) — and therefore
holds none of the method's arithmetic: it only draws random numbers and builds
test matrices the way the paper (and BASELINE.json's configs) prescribe.
Library calls (torch.randn, torch.linalg.qr, matmul) are used as recipe steps.

Recipes (DESIGN.md §4 "Inputs"):
  * Haar factors: orthonormalise i.i.d. N(0,1) columns via QR, signs fixed by
    diag(R) > 0 — PAPER.md:507-514 (§7).
  * Spectra D1-D6 — PAPER.md:520-553 (§7).  Sign-flipped Gaussian —
    PAPER.md:598-604.  PROPACK hard diagonals — PAPER.md:460-491 (§6).
  * C1-C5 — BASELINE.json ``configs`` with the readings of SURVEY.md §8(c) Q17
    (N(μ, v) means variance v; C5's planted block restricted to 200 columns).

The paper's own experiments use the University of Florida sparse collection
(PAPER.md:656-661), which is not available here: C5 is a synthetic stand-in.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

GEN_SEEDS = {"C1": 1001, "C2": 1002, "C3": 1003, "C4": 1004, "C5": 1005}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def haar_columns(rows: int, cols: int, seed: int, device="cpu", dtype=torch.float64) -> torch.Tensor:
    """rows×cols with orthonormal columns: QR of an i.i.d. N(0,1) matrix."""
    g = _gen(seed, device)
    G = torch.randn(rows, cols, generator=g, device=device, dtype=dtype)
    Q, R = torch.linalg.qr(G, mode="reduced")
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1
    Q *= d
    return Q


def spectrum(dist: int, m: int, n: int, k: int, seed: int = 0) -> torch.Tensor:
    """σ_1..σ_min(m,n) for the six distributions of PAPER.md:520-553 (D1-D6)."""
    p = min(m, n)
    j = torch.arange(1, p + 1, dtype=torch.float64)
    s = torch.empty(p, dtype=torch.float64)
    if dist == 1:
        s = 1.0 / j
    elif dist == 2:
        s[0] = 1.0
        s[1:k] = 2e-5
        s[k:] = 1e-5 * (k + 1) / j[k:]
    elif dist == 3:
        s[:k] = 10.0 ** (-5.0 * (j[:k] - 1) / (k - 1))
        s[k:] = 1e-5 * (k + 1) / j[k:]
    elif dist == 4:
        s[:k] = 10.0 ** (-5.0 * (j[:k] - 1) / (k - 1))
        s[k] = 1e-5
        s[k + 1:] = 0.0
    elif dist == 5:
        s[:k] = 1e-5 + (1 - 1e-5) * (k - j[:k]) / (k - 1)
        s[k:] = 1e-5 * torch.sqrt((k + 1) / j[k:])
    elif dist == 6:
        g = _gen(seed, "cpu")
        s = torch.sort(torch.randn(p, generator=g, dtype=torch.float64).abs(), descending=True).values
    else:
        raise ValueError("dist must be 1..6")
    return s


def synth_dense(m: int, n: int, sigma: torch.Tensor, seed: int, device="cpu") -> torch.Tensor:
    """A = U·diag(σ)·Vᵀ with Haar U (m×p), V (n×p), p = min(m, n)."""
    p = min(m, n)
    U = haar_columns(m, p, seed * 16 + 1, device)
    V = haar_columns(n, p, seed * 16 + 2, device)
    return (U * sigma.to(device)) @ V.T


def propack_diag(n: int) -> torch.Tensor:
    """diag(1, 1, 1, .999 ×17, 0, …) — PAPER.md:460-463 (the 30×30 and 100×100 cases)."""
    d = torch.zeros(n, dtype=torch.float64)
    d[:3] = 1.0
    d[3:20] = 0.999
    return torch.diag(d)


def sign_flipped_gaussian(n: int, seed: int, device="cpu") -> torch.Tensor:
    """i.i.d. N(√(30/n), 1), sign flipped where i·j is odd (1-based) — PAPER.md:598-604."""
    g = _gen(seed, device)
    A = torch.randn(n, n, generator=g, device=device, dtype=torch.float64) + math.sqrt(30.0 / n)
    odd = (torch.arange(1, n + 1, device=device) % 2 == 1)
    flip = odd[:, None] & odd[None, :]
    A[flip] = -A[flip]
    return A


# ---------------------------------------------------------------------------
# BASELINE.json configs C1-C5 (scalable: every recipe takes its sizes).
# ---------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    kind: str          # "dense" | "csr"
    dtype: torch.dtype
    m: int
    n: int
    k: int
    l: int
    its: int
    raw: bool
    op: str            # "pca" | "eigens"
    desc: str


CONFIGS = {
    "C1": Config("C1", "dense", torch.float64, 1000, 500, 10, 12, 2, True, "pca",
                 "dense fp64 1000x500, sigma_j=exp(-(j-1)/5), k=10 l=12 its=2, raw"),
    "C2": Config("C2", "dense", torch.float64, 100000, 4000, 20, 22, 2, True, "pca",
                 "dense fp64 100000x4000 (3.2 GB), sigma_j=1/j + N(0,1e-8) noise, k=20 l=22 its=2, raw"),
    "C3": Config("C3", "dense", torch.float64, 32768, 32768, 40, 42, 2, True, "eigens",
                 "PSD fp64 32768^2 (8.6 GB), lambda_j=j^-2, k=40 l=42 its=2, Nystrom"),
    "C4": Config("C4", "dense", torch.float32, 2000000, 4096, 50, 52, 4, False, "pca",
                 "dense fp32 2e6x4096 (32.8 GB), 60-dim latent + noise + column means, k=50 l=52 its=4, centered"),
    "C5": Config("C5", "csr", torch.float64, 10000000, 1000000, 30, 32, 2, True, "pca",
                 "CSR fp64 1e7x1e6, 10 nnz/row + planted rank-20 on 1% rows, k=30 l=32 its=2, raw"),
}


def make_c1(m=1000, n=500, seed=GEN_SEEDS["C1"], device="cpu"):
    sigma = torch.exp(-torch.arange(min(m, n), dtype=torch.float64) / 5.0)
    return synth_dense(m, n, sigma, seed, device).contiguous()


def make_c2(m=100000, n=4000, seed=GEN_SEEDS["C2"], device="cpu", noise_var=1e-8):
    sigma = 1.0 / torch.arange(1, min(m, n) + 1, dtype=torch.float64)
    A = synth_dense(m, n, sigma, seed, device)
    g = _gen(seed * 16 + 3, device)
    A += math.sqrt(noise_var) * torch.randn(m, n, generator=g, device=device, dtype=torch.float64)
    return A.contiguous()


def make_c3(n=32768, seed=GEN_SEEDS["C3"], device="cpu"):
    lam = 1.0 / torch.arange(1, n + 1, dtype=torch.float64) ** 2
    V = haar_columns(n, n, seed * 16 + 1, device)
    A = (V * lam.to(device)) @ V.T
    del V
    A = 0.5 * (A + A.T)
    return A.contiguous()


def make_c4(m=2000000, n=4096, seed=GEN_SEEDS["C4"], device="cpu", latent=60, chunk=1 << 17):
    """rows = z·L + e + μ in fp64, rounded to fp32 (reading Q17: noise variance 0.01, j = 0..59)."""
    P = haar_columns(latent, latent, seed * 16 + 1, device)
    R = haar_columns(n, latent, seed * 16 + 2, device)
    sv = 10.0 * 0.9 ** torch.arange(latent, dtype=torch.float64, device=device)
    L = (P * sv) @ R.T                                        # latent × n
    g = _gen(seed * 16 + 3, device)
    mu = (torch.rand(n, generator=g, device=device, dtype=torch.float64) * 10.0 - 5.0)
    A = torch.empty(m, n, dtype=torch.float32, device=device)
    gz = _gen(seed * 16 + 4, device)
    ge = _gen(seed * 16 + 5, device)
    for i0 in range(0, m, chunk):
        i1 = min(m, i0 + chunk)
        z = torch.randn(i1 - i0, latent, generator=gz, device=device, dtype=torch.float64)
        e = 0.1 * torch.randn(i1 - i0, n, generator=ge, device=device, dtype=torch.float64)
        A[i0:i1] = (z @ L + e + mu).to(torch.float32)
    return A


def make_c5(m=10000000, n=1000000, seed=GEN_SEEDS["C5"], device="cpu", nnz_row=10,
            planted_rows=None, planted_cols=200, rank=20, weight=5.0):
    """CSR (rowptr int64, colind int32, vals fp64).  Reading Q17(iii)."""
    g = _gen(seed * 16 + 1, device)
    cols = torch.randint(0, n, (m, nnz_row), generator=g, device=device)
    cols = torch.sort(cols, dim=1).values
    for _ in range(100):  # redraw rows with a repeated column until all are distinct
        dup = (cols[:, 1:] == cols[:, :-1]).any(dim=1)
        nd = int(dup.sum())
        if nd == 0:
            break
        cols[dup] = torch.sort(torch.randint(0, n, (nd, nnz_row), generator=g, device=device), dim=1).values
    gv = _gen(seed * 16 + 2, device)
    vals = torch.randn(m, nnz_row, generator=gv, device=device, dtype=torch.float64)
    rows = torch.arange(m, device=device).repeat_interleave(nnz_row)
    keys = [rows * n + cols.reshape(-1)]
    vv = [vals.reshape(-1)]
    del cols, vals, rows
    if planted_rows is None:
        planted_rows = max(1, m // 100)
    gp = _gen(seed * 16 + 3, device)
    S = torch.sort(torch.randperm(m, generator=gp, device=device)[:planted_rows]).values
    T = torch.sort(torch.randperm(n, generator=gp, device=device)[:planted_cols]).values
    G = torch.randn(planted_rows, rank, generator=gp, device=device, dtype=torch.float64)
    H = torch.randn(planted_cols, rank, generator=gp, device=device, dtype=torch.float64) / math.sqrt(planted_cols)
    blk = weight * (G @ H.T)
    keys.append((S[:, None] * n + T[None, :]).reshape(-1))
    vv.append(blk.reshape(-1))
    key = torch.cat(keys)
    val = torch.cat(vv)
    del keys, vv, blk
    key, order = torch.sort(key)
    val = val[order]
    del order
    uniq, inv = torch.unique_consecutive(key, return_inverse=True)
    sval = torch.zeros(uniq.numel(), dtype=torch.float64, device=device)
    sval.index_add_(0, inv, val)   # duplicates summed; ascending key order within a slot
    del key, val, inv
    r = uniq // n
    c = (uniq % n).to(torch.int32)
    counts = torch.bincount(r, minlength=m)
    rowptr = torch.zeros(m + 1, dtype=torch.int64, device=device)
    rowptr[1:] = torch.cumsum(counts, 0)
    return rowptr, c, sval


def make(name: str, device="cpu", **overrides):
    f = {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}[name]
    return f(device=device, **overrides)
