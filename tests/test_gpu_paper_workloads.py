"""The paper's accuracy workloads run through librpca.

* Figure 1 (§7): dense A = U·diag(σ)·Vᵀ with the six
  spectra D1–D6, m = n = 1000, k = 10, oversampling
  l = k+2 … k+32, its = 2 — the GPU pipeline against the oracle on the same
  bits, and the paper's claim that D2–D5 are approximated to within a small
  factor of the optimal error 1e-5 (tests/golden/dense_optimum.json).
* Figure 2: the n×n sign-flipped Gaussian, k = 4, its =
  0 / 2 / 4 — parity against the oracle at n = 1000, and at n = 100000 (an
  80 GB fp64 matrix) the paper's findings measured with the GPU power-method
  estimate (rpca_diffsnorm): the best rank-4 error is about half of ‖A‖
  (PAPER.md:614-616), its = 0 "produces very inaccurate approximations" and,
  at this size only, its = 2 is not yet "very nearly optimal".
Competitor curves (PROPACK, ARPACK, LAPACK) stay out of scope.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1412_3510_b200 as rp
import synth
from tests.helpers import cluster_sin_angle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def dev():
    return torch.device("cuda", 0)


def compare(res_g, res_o, k, tol_s=1e-10, tol_a=1e-8, rel=1e-12):
    Ug, Sg, Vg = [t.cpu().numpy() for t in res_g]
    Uo, So, Vo = res_o
    nz = So > 1e-12 * So[0]
    assert np.max(np.abs(Sg[nz] - So[nz]) / So[nz]) < tol_s, (Sg, So)
    assert cluster_sin_angle(Uo, Ug, So, k, rel=rel) < tol_a
    assert cluster_sin_angle(Vo, Vg, So, k, rel=rel) < tol_a


@pytest.mark.parametrize("dist", [1, 2, 3, 4, 5, 6])
def test_figure1_spectra_vs_oracle(dist):
    """Figure 1's sweep over the oversampling l − k ∈ {2, 8, 16, 32}."""
    m = n = 1000
    k = 10
    sig = synth.spectrum(dist, m, n, k, seed=dist)
    A = synth.synth_dense(m, n, sig, seed=300 + dist, device=dev()).contiguous()
    Ah = A.cpu().numpy()
    # the vectors are compared where the TRUE spectrum separates them from
    # σ_{k+1}: D3 and D4 have σ_k = σ_{k+1} = 1e-5 (the k-th vector is not
    # determined), D2's σ₂…σ_k are equal (one cluster; the computed values
    # agree only to the convergence level, so it is grouped at 1e-3)
    kv = int(np.sum(sig[:k].numpy() > 1.001 * float(sig[k])))
    errs = []
    for l in (k + 2, k + 8, k + 16, k + 32):
        res = rp.pca(A, k, its=2, l=l, seed=l)
        o = oracle.pca(Ah, k, its=2, l=l, seed=l)
        compare([t[..., :kv] for t in res], [t[..., :kv] for t in o], kv, rel=1e-12 if dist != 2 else 1e-3)
        errs.append(rp.diffsnorm(A, *res, its=20, seed=1))
    errs = np.array(errs)
    # never better than optimal (Eckart–Young) — up to the estimator: the
    # power method approaches ‖A − USVᵀ‖ from below, slowly when E's leading
    # singular values cluster (D5: σ_j = 1e-5·√((k+1)/j) beyond k), hence 10%
    assert np.all(errs >= float(sig[k]) * 0.9)
    if dist in (2, 3, 4, 5):
        g = gold("dense_optimum.json")
        assert np.median(errs) <= g["median_error_bound"], errs
    # more oversampling never hurts much: the widest sketch is within 2× the best
    assert errs[-1] <= 2 * errs.min()


@pytest.mark.parametrize("its", [0, 2, 4])
def test_figure2_signflip_vs_oracle(its):
    n, k = 1000, 4
    A = synth.sign_flipped_gaussian(n, seed=200, device=dev())
    res = rp.pca(A, k, its=its, seed=0)
    compare(res, oracle.pca(A.cpu().numpy(), k, its=its, seed=0), k)


@pytest.mark.slow
def test_figure2_signflip_n100000_on_gpu():
    """n = 100000 (80 GB in fp64), the paper's largest size: errors from the
    GPU power method, relative to ‖A‖ estimated the same way (k = 0).
    Measured on one B200: its = 0 / 2 / 4 → 0.9998 / 0.863 / 0.476."""
    n, k = 100000, 4
    import gc
    gc.collect()
    torch.cuda.empty_cache()  # earlier tests' cached blocks
    free = torch.cuda.mem_get_info()[0]
    if free < 90e9:
        pytest.skip(f"needs ~90 GB free HBM, {free / 1e9:.0f} GB free")
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.randn(n, n, generator=g, device=dev(), dtype=torch.float64)
    A += (30.0 / n) ** 0.5
    A.view(n // 2, 2, n // 2, 2)[:, 0, :, 0] *= -1.0  # i·j odd (1-based) ⇔ both 0-based indices even
    nA = rp.diffsnorm(A, torch.zeros(n, 0, dtype=torch.float64, device=dev()),
                      torch.zeros(0, dtype=torch.float64, device=dev()),
                      torch.zeros(n, 0, dtype=torch.float64, device=dev()), its=20)
    ratios = {}
    for its in (0, 2, 4):
        U, S, V = rp.pca(A, k, its=its, seed=1)
        ratios[its] = rp.diffsnorm(A, U, S, V, its=20) / nA
        del U, S, V
    # "except for m = n = 100000, using only its = 2 extra
    # power/subspace iterations yields very nearly optimal accuracy" — at this
    # size its = 4 reaches the optimal ≈ ‖A‖/2 and its = 2
    # does not yet; its = 0 is "very inaccurate"
    gd = gold("signflip.json")
    lo, hi = gd["ratio_its2_range"]
    assert lo <= ratios[4] <= hi, ratios
    assert ratios[2] > ratios[4] * (1 + gd["its0_worse_by_at_least"]), ratios
    assert ratios[0] > ratios[2] and ratios[0] > 0.95, ratios
    print("sign-flip n=1e5 error/‖A‖:", ratios)
