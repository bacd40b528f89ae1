"""Pins for the whole oracle pipelines against what the paper and the
mathematics fix (not against the oracle itself):

pca      — PAPER.md §2 (i1)-(i4) l.116-149, §5 l.382-435; PROPACK diagonals
           §6 l.460-491 (tests/golden/propack_diag.json); exact-rank capture;
           l = min(m,n) ⇒ the exact SVD (a LAPACK case); interlacing and
           Eckart–Young bounds; D2-D5 near-optimality l.549-551
           (golden/dense_optimum.json); sign-flip its=0 vs its=2 l.598-627
           (golden/signflip.json); implicit centring ≡ explicit centring.
eigens   — PAPER.md §3 l.214-282: exact-rank PSD, identity, SHIFT_CHOL vs SQRT,
           Nyström ≥ self-adjoint accuracy.
diffsnorm— PAPER.md §4 l.362-371: diag(3,1), zero, exact truncation → σ_{k+1},
           factor-two reliability.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.helpers import cluster_sin_angle, sin_angle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def spec_norm(M):
    return float(np.linalg.norm(M, 2))


# ------------------------------------------------------------------ PROPACK
def test_propack_30x30_k20_all_seeds():
    case = gold("propack_diag.json")["cases"][0]
    A = synth.propack_diag(30).numpy()
    for seed in range(20):
        U, S, V = oracle.pca(A, case["k"], its=2, seed=seed)
        assert np.max(np.abs(S - np.array(case["expected"]))) < 1e-10, (seed, S)


def test_propack_30x30_k21_zero_tail():
    case = gold("propack_diag.json")["cases"][1]
    A = synth.propack_diag(30).numpy()
    U, S, V = oracle.pca(A, case["k"], its=2, seed=3)
    assert np.max(np.abs(S - np.array(case["expected"]))) < 1e-10


def test_propack_100x100_k50():
    case = gold("propack_diag.json")["cases"][2]
    A = synth.propack_diag(100).numpy()
    U, S, V = oracle.pca(A, case["k"], its=2, seed=1)
    head = np.array(case["expected_head"])
    assert np.max(np.abs(S[:20] - head)) < 1e-10
    assert np.all(np.abs(S[20:]) < 1e-10) and len(S[20:]) == case["expected_tail_zeros"]
    assert np.linalg.norm(U.T @ U - np.eye(50)) < 1e-10
    assert np.linalg.norm(V.T @ V - np.eye(50)) < 1e-10


# ------------------------------------------------------------------ exact cases
@pytest.mark.parametrize("m,n,r,k,l", [(200, 80, 6, 6, 8), (90, 150, 5, 4, 7)])
def test_exact_rank_capture(m, n, r, k, l):
    rng = np.random.default_rng(r)
    A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    U, S, V = oracle.pca(A, r, its=2, l=l, seed=2)
    assert spec_norm(A - U * S @ V.T) <= 1e-10 * spec_norm(A)
    assert np.allclose(S, np.linalg.svd(A, compute_uv=False)[:r], rtol=1e-10)


@pytest.mark.parametrize("m,n", [(60, 25), (25, 60)])
def test_full_width_is_exact_svd(m, n):
    """l = min(m,n): the basis spans everything, so the result IS the SVD (LAPACK)."""
    A = np.random.default_rng(0).standard_normal((m, n))
    p = min(m, n)
    U, S, V = oracle.pca(A, p, its=1, l=p, seed=0)
    Un, Sn, Vtn = np.linalg.svd(A, full_matrices=False)
    assert np.allclose(S, Sn, rtol=1e-12)
    assert sin_angle(Un[:, :5], U[:, :5]) < 1e-10
    assert sin_angle(Vtn.T[:, :5], V[:, :5]) < 1e-10
    assert spec_norm(A - U * S @ V.T) < 1e-12 * Sn[0]


def test_brute_force_small():
    """m, n ≤ 60, l = k+32, its = 6 → top-k within 1e-8."""
    rng = np.random.default_rng(42)
    for t in range(12):
        m, n = rng.integers(41, 61, 2)
        k = int(rng.integers(1, 9))
        A = rng.standard_normal((m, n))
        U, S, V = oracle.pca(A, k, its=6, l=k + 32, seed=t)
        Sn = np.linalg.svd(A, compute_uv=False)
        assert np.allclose(S, Sn[:k], rtol=1e-8)


def test_bounds_orthonormality_interlacing():
    A = synth.make_c1(m=300, n=120, seed=5).numpy()
    k = 10
    U, S, V = oracle.pca(A, k, its=2, l=12, seed=0)
    Sn = np.linalg.svd(A, compute_uv=False)
    assert np.all(S <= Sn[:k] * (1 + 1e-12))                       # interlacing
    assert spec_norm(A - U * S @ V.T) >= Sn[k] - 1e-10            # Eckart–Young
    assert np.linalg.norm(U.T @ U - np.eye(k)) < 1e-12
    assert np.linalg.norm(V.T @ V - np.eye(k)) < 1e-12
    assert np.all(np.diff(S) <= 0) and np.all(S >= 0)
    # sign convention (Q10): largest-|.| entry of each V column is positive
    assert np.all(V[np.argmax(np.abs(V), axis=0), np.arange(k)] > 0)


def test_c1_recipe_known_spectrum():
    """C1: σ_j = e^{-(j-1)/5}; the leading values are pinned tightly (Ritz factor
    (σ13/σ1)^{10} ≈ 3e-11)."""
    A = synth.make_c1().numpy()
    U, S, V = oracle.pca(A, 10, its=2, l=12, seed=0)
    sig = np.exp(-np.arange(10) / 5.0)
    assert abs(S[0] - sig[0]) < 1e-9
    assert np.all(S <= sig * (1 + 1e-12))
    # randomized subspace iteration: relative error of σ_j decays like the Ritz
    # factor (σ_{l+1}/σ_j)^{2(2·its+1)} (HMT §10)
    ritz = (np.exp(-12 / 5.0) / sig) ** 10
    assert np.all(np.abs(S - sig) / sig <= 10 * ritz)


def test_orientation_transpose_is_bitwise_swap():
    """m < n sketches Aᵀ (reading Q6): pca(A) = swap(pca(Aᵀ)) exactly, up to the
    column signs (the sign convention Q10 looks at V, which differs after a swap)."""
    A = np.random.default_rng(9).standard_normal((40, 70))
    U1, S1, V1 = oracle.pca(A, 5, its=2, seed=4)
    U2, S2, V2 = oracle.pca(np.ascontiguousarray(A.T), 5, its=2, seed=4)
    d = np.sign(U1[0] * V2[0])
    assert np.array_equal(S1, S2) and np.array_equal(U1, V2 * d) and np.array_equal(V1, U2 * d)


def test_deterministic():
    A = synth.make_c1(m=200, n=90, seed=3).numpy()
    r1 = oracle.pca(A, 8, its=2, seed=1)
    r2 = oracle.pca(A, 8, its=2, seed=1)
    assert all(np.array_equal(a, b) for a, b in zip(r1, r2))


def test_zero_matrix():
    U, S, V = oracle.pca(np.zeros((30, 20)), 4, its=2, seed=0)
    assert np.all(S == 0)
    assert np.linalg.norm(U.T @ U - np.eye(4)) < 1e-12


def test_argument_errors():
    A = np.ones((10, 8))
    for kw in [dict(k=0), dict(k=5, l=4), dict(k=3, l=9), dict(k=2, its=-1)]:
        k = kw.pop("k")
        with pytest.raises(oracle.OracleError) as e:
            oracle.pca(A, k, **kw)
        assert e.value.code == oracle.E_SHAPE


# ------------------------------------------------------------------ paper's accuracy claims
@pytest.mark.slow
def test_d2_to_d5_near_optimal():
    g = gold("dense_optimum.json")
    m = n = 1000
    k = 10
    for dist in (2, 3, 4, 5):
        sig = synth.spectrum(dist, m, n, k)
        assert abs(sig[0] - g["norm_A"]) < 1e-15 and abs(sig[k] - g["optimal_error"]) < 1e-18
        errs = []
        for t in range(3):
            A = synth.synth_dense(m, n, sig, seed=100 + 10 * dist + t).numpy()
            U, S, V = oracle.pca(A, k, its=2, l=k + 16, seed=t)
            errs.append(spec_norm(A - U * S @ V.T))
            assert errs[-1] >= g["optimal_error"] * (1 - 1e-6)
        assert np.median(errs) <= g["median_error_bound"], (dist, errs)


@pytest.mark.slow
def test_signflip_its_matters():
    g = gold("signflip.json")
    n, k = 1000, g["k"]
    r0, r2 = [], []
    for t in range(3):
        A = synth.sign_flipped_gaussian(n, seed=200 + t).numpy()
        nA = spec_norm(A)
        U, S, V = oracle.pca(A, k, its=2, seed=t)
        r2.append(spec_norm(A - U * S @ V.T) / nA)
        U, S, V = oracle.pca(A, k, its=0, seed=t)
        r0.append(spec_norm(A - U * S @ V.T) / nA)
    lo, hi = g["ratio_its2_range"]
    assert lo <= np.median(r2) <= hi
    assert np.median(r0) >= (1 + g["its0_worse_by_at_least"]) * np.median(r2)


# ------------------------------------------------------------------ centring
def test_centering_matches_explicit_pipeline_and_svd():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((60, 30)) @ np.diag(np.linspace(3, 0.1, 30)) + rng.uniform(-5, 5, 30)
    Ac = A - A.mean(axis=0)
    Uc, Sc, Vc = oracle.pca(A, 4, raw=False, its=2, l=26, seed=0)
    Ue, Se, Ve = oracle.pca(Ac, 4, raw=True, its=2, l=26, seed=0)
    assert np.allclose(Sc, Se, rtol=1e-12)
    assert sin_angle(Ue, Uc) < 1e-10 and sin_angle(Ve, Vc) < 1e-10
    Sn = np.linalg.svd(Ac, compute_uv=False)
    assert np.allclose(Sc, Sn[:4], rtol=1e-8)
    const = np.tile(rng.standard_normal(12), (20, 1))
    U, S, V = oracle.pca(const, 3, raw=False, seed=0)
    assert np.all(S <= 1e-12)


def test_fp32_input_is_upcast():
    A = synth.make_c1(m=200, n=80, seed=2).to(torch.float32).numpy()
    U1, S1, V1 = oracle.pca(A, 6, its=2, seed=0)
    U2, S2, V2 = oracle.pca(A.astype(np.float64), 6, its=2, seed=0)
    # fp32 path consumes fl32(Ω): same A values, Ω perturbed by ≤ 2^-24 relative
    assert np.allclose(S1, S2, rtol=1e-5)
    Sn = np.linalg.svd(A.astype(np.float64), compute_uv=False)
    assert np.all(S1 <= Sn[:6] * (1 + 1e-12))


# ------------------------------------------------------------------ Nyström
def psd(n, lam, seed):
    Q = synth.haar_columns(n, n, seed).numpy()
    A = (Q * lam) @ Q.T
    return 0.5 * (A + A.T)


@pytest.mark.parametrize("variant", [oracle.SHIFT_CHOL, oracle.SQRT])
def test_nystrom_exact_rank(variant):
    rng = np.random.default_rng(1)
    for t in range(5):
        G = rng.standard_normal((30, 8))
        A = G @ G.T
        U, lam = oracle.eigens(A, 8, its=2, l=10, seed=t, variant=variant)
        assert spec_norm(A - U * lam @ U.T) <= 1e-9 * spec_norm(A)
        assert np.all(lam >= 0)


def test_nystrom_identity_and_agreement():
    U, lam = oracle.eigens(np.eye(12), 12, its=1, l=12, seed=0)
    assert np.allclose(lam, 1.0, atol=1e-12)
    lam_true = 1.0 / np.arange(1, 201) ** 2
    A = psd(200, lam_true, 11)
    U1, l1 = oracle.eigens(A, 10, its=2, l=12, seed=0, variant=oracle.SHIFT_CHOL)
    U2, l2 = oracle.eigens(A, 10, its=2, l=12, seed=0, variant=oracle.SQRT)
    assert np.allclose(l1, l2, rtol=1e-9)
    assert np.all(l1 <= lam_true[:10] * (1 + 1e-9) + 1e-13)     # λ̂ ≤ λ + ν
    assert np.allclose(l1[:4], lam_true[:4], rtol=1e-8)
    assert np.linalg.norm(U1.T @ U1 - np.eye(10)) < 1e-10


def test_nystrom_more_accurate_than_rayleigh_ritz():
    """given the same Q, the Nyström approximation 'should be
    better' than formulae (i2)-(i4).  Q is rebuilt from the oracle's primitives
    exactly as the self-adjoint loop of PAPER.md:386-412 does (same bits), and
    the rank-k Rayleigh–Ritz approximation Q·(QᵀAQ)_k·Qᵀ is formed with LAPACK."""
    n, k, l = 200, 10, 12
    lam_true = np.empty(n)
    lam_true[:k] = 10.0 ** (-5 * np.arange(k) / (k - 1))           # D3 head
    lam_true[k:] = 1e-5 * (k + 1) / np.arange(k + 1, n + 1)
    ny, rr = [], []
    for t in range(9):
        A = psd(n, lam_true, 300 + t)
        U, lam = oracle.eigens(A, k, its=2, l=l, seed=t)
        ny.append(spec_norm(A - U * lam @ U.T))
        Q = oracle.lu_renorm(oracle.apply(A, oracle.omega(t, n, l)))[0]
        Q = oracle.lu_renorm(oracle.apply(A, Q))[0]
        Q = oracle.house_qr(oracle.apply(A, Q))[0]
        T = Q.T @ A @ Q
        w, E = np.linalg.eigh(0.5 * (T + T.T))
        E = E[:, ::-1][:, :k]
        w = w[::-1][:k]
        rr.append(spec_norm(A - (Q @ E) * w @ (Q @ E).T))
    assert np.median(ny) <= np.median(rr)


def test_nystrom_rank_deficient_no_crash():
    A = np.zeros((20, 20))
    A[:3, :3] = np.diag([3.0, 2.0, 1.0])
    U, lam = oracle.eigens(A, 5, its=2, l=8, seed=0)
    assert np.allclose(lam[:3], [3, 2, 1], rtol=1e-10) and np.all(np.abs(lam[3:]) < 1e-10)
    U, lam = oracle.eigens(np.zeros((10, 10)), 3, its=1, seed=0)
    assert np.all(lam == 0)


# ------------------------------------------------------------------ diffsnorm
def test_diffsnorm_closed_forms():
    A = np.diag([3.0, 1.0])
    z = np.zeros((2, 0))
    assert abs(oracle.diffsnorm(A, z, np.zeros(0), z, its=20) - 3.0) < 1e-8
    assert oracle.diffsnorm(np.zeros((5, 4)), np.zeros((5, 0)), np.zeros(0), np.zeros((4, 0))) == 0.0
    D = synth.propack_diag(30).numpy()
    U, S, V = np.linalg.svd(D)
    est = oracle.diffsnorm(D, U[:, :20], S[:20], Vt := V.T[:, :20])
    assert est <= 1e-10


def test_diffsnorm_exact_truncation_and_factor_two():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((50, 40))
    U, S, Vt = np.linalg.svd(A, full_matrices=False)
    est = oracle.diffsnorm(A, U[:, :5], S[:5], Vt.T[:, :5], its=100, seed=3)
    assert S[5] / 2 <= est <= S[5] * (1 + 1e-10)
    # the paper's claim (Kuczyński–Woźniakowski Thm 4.1(a)) is
    # "within a factor of two": every one of 100 seeds at its = 20.  Convergence
    # is monotone in its; at its = 50 ≥ 95 of the 100 land within 1% (the square
    # Gaussian has no spectral gap at the top, so its = 20 gets only ~70).
    within = 0
    for t in range(100):
        B = np.random.default_rng(1000 + t).standard_normal((100, 100))
        nb = spec_norm(B)
        z = np.zeros((100, 0))
        e20 = oracle.diffsnorm(B, z, np.zeros(0), z, its=20, seed=t)
        e50 = oracle.diffsnorm(B, z, np.zeros(0), z, its=50, seed=t)
        assert nb / 2 <= e20 <= e50 * (1 + 1e-12) <= nb * (1 + 1e-10)
        within += abs(e50 - nb) <= 0.01 * nb
    assert within >= 95


def test_diffsnorm_centered_and_pca_residual():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((80, 30)) + rng.uniform(-5, 5, 30)
    U, S, V = oracle.pca(A, 5, raw=False, its=3, l=20, seed=0)
    Ac = A - A.mean(axis=0)
    exact = spec_norm(Ac - U * S @ V.T)
    est = oracle.diffsnorm(A, U, S, V, raw=False, its=60, seed=1)
    assert exact / 2 <= est <= exact * (1 + 1e-10)
    assert abs(est - exact) < 0.02 * exact


# ----------------------------------------------------------------- reig (§8(f) N1)
def test_reig_spec_examples():
    """diag(3, −2, 1, 0, …) 10×10, k = 2 → (3, −2) with signs
    kept and eigenvectors e₀, e₁; the identity with k = 1 → 1."""
    A = np.diag([3.0, -2.0, 1.0] + [0.0] * 7)
    U, lam = oracle.reig(A, 2, its=2, l=4, seed=0)
    assert np.allclose(lam, [3.0, -2.0], atol=1e-10, rtol=0)
    assert np.allclose(np.abs(U[:2, :]), np.eye(2), atol=1e-10) and np.allclose(U[2:], 0, atol=1e-10)
    U, lam = oracle.reig(np.eye(20), 1, its=1, l=3, seed=1)
    assert abs(lam[0] - 1.0) < 1e-12 and abs(np.linalg.norm(U[:, 0]) - 1.0) < 1e-12


def test_reig_full_width_is_lapack_eigh():
    """l = n: Q spans everything, so reig is the exact eigendecomposition —
    LAPACK's (numpy eigh) ordered by |λ| (SPEC.md:236's random symmetric 40×40)."""
    rng = np.random.default_rng(40)
    G = rng.standard_normal((40, 40))
    A = (G + G.T) / 2
    U, lam = oracle.reig(A, 6, its=4, l=40, seed=0)
    w, V = np.linalg.eigh(A)
    o = np.argsort(-np.abs(w), kind="stable")[:6]
    assert np.max(np.abs(lam - w[o]) / np.abs(w[o])) < 1e-12
    for j in range(6):  # simple eigenvalues: vectors equal up to sign
        assert min(np.linalg.norm(U[:, j] - V[:, o[j]]), np.linalg.norm(U[:, j] + V[:, o[j]])) < 1e-10
    assert np.linalg.norm(U.T @ U - np.eye(6)) < 1e-13


@pytest.mark.parametrize("n,r,k,l", [(300, 8, 8, 10), (500, 12, 6, 12)])
def test_reig_exact_rank_indefinite(n, r, k, l):
    """A = V diag(λ) Vᵀ of rank r ≤ l with mixed signs: reig recovers the
    eigenpairs of largest |λ| exactly (Q spans range(A) after one application)."""
    rng = np.random.default_rng(n + r)
    V = np.linalg.qr(rng.standard_normal((n, r)))[0]
    lam_true = np.array([(-1.0) ** j * 10.0 * 0.7 ** j for j in range(r)])
    A = (V * lam_true) @ V.T
    A = (A + A.T) / 2
    U, lam = oracle.reig(A, k, its=1, l=l, seed=2)
    o = np.argsort(-np.abs(lam_true), kind="stable")[:k]
    assert np.max(np.abs(lam - lam_true[o]) / np.abs(lam_true[o])) < 1e-11
    assert np.all(np.sign(lam) == np.sign(lam_true[o]))
    assert sin_angle(V[:, o], U) < 1e-10
    Ak = (U * lam) @ U.T
    if k == r:
        assert np.linalg.norm(A - Ak) < 1e-10 * np.linalg.norm(A)


def test_reig_psd_matches_nystrom_and_is_nonnegative():
    """SPEC.md invariants: a nonnegative-definite A gives lam ≥ −1e-10·‖A‖, and
    Rayleigh–Ritz (reig) interlaces below the true λ (λ̂_j ≤ λ_j)."""
    A = synth.make_c3(n=1024).numpy()
    U, lam = oracle.reig(A, 20, its=2, l=22, seed=0)
    true = 1.0 / np.arange(1, 21) ** 2
    assert np.all(lam >= -1e-10 * true[0])
    assert np.all(lam <= true * (1 + 1e-12))
    assert np.max(np.abs(lam[:5] - true[:5]) / true[:5]) < 1e-7  # (λ₂₃/λ_j)^(2·its+2) convergence
    Un, ln = oracle.eigens(A, 20, its=2, l=22, seed=0)
    assert np.max(np.abs(lam[:5] - ln[:5]) / ln[:5]) < 1e-7


# ----------------------------------------------------------------- renorm_odd (§8(f) N2)
def test_renorm_odd_reduces_to_default_without_interior_rounds():
    """its ≤ 1 has no interior round to skip: bitwise the default path."""
    A = synth.make_c1(m=400, n=300).numpy()
    for its in (0, 1):
        a = oracle.pca(A, 8, its=its, l=10, seed=2)
        b = oracle.pca(A, 8, its=its, l=10, seed=2, renorm_odd=True)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("raw", [True, False])
def test_renorm_odd_same_span_when_well_conditioned(raw):
    """Renormalisation does not change the span in exact arithmetic (PAPER.md:
    200-204): on a well-conditioned spectrum the two schedules agree to rounding."""
    A = synth.make_c1(m=800, n=400, seed=5).numpy()
    if not raw:
        A = A + np.linspace(-3, 3, 400)[None, :]
    a = oracle.pca(A, 10, raw=raw, its=3, l=12, seed=1)
    b = oracle.pca(A, 10, raw=raw, its=3, l=12, seed=1, renorm_odd=True)
    assert np.max(np.abs(a[1] - b[1]) / a[1]) < 1e-12
    assert cluster_sin_angle(a[0], b[0], a[1], 10) < 1e-10
    assert cluster_sin_angle(a[2], b[2], a[1], 10) < 1e-10


def test_renorm_odd_loses_accuracy_on_fast_decay():
    """skipping renormalisations "would sacrifice accuracy".
    With σ_j = 10^-j/2 an unrenormalised F·F*·Q has κ ≈ (σ₁/σ_l)² and the trailing
    directions drown in rounding: the default schedule's trailing σ are exact
    to ~1e-13 relative, the odd-only schedule's are not."""
    m, n, k, l = 600, 300, 16, 18
    sig = torch.tensor([10.0 ** (-j / 2) for j in range(n)], dtype=torch.float64)
    A = synth.synth_dense(m, n, sig, seed=9).numpy()
    a = oracle.pca(A, k, its=4, l=l, seed=0)
    b = oracle.pca(A, k, its=4, l=l, seed=0, renorm_odd=True)
    true = sig[:k].numpy()
    err_a = np.max(np.abs(a[1] - true) / true)
    err_b = np.max(np.abs(b[1] - true) / true)
    assert err_a < 1e-10 and err_b > 10 * err_a, (err_a, err_b)
    assert np.max(np.abs(b[1][:4] - true[:4]) / true[:4]) < 1e-10  # the leading values survive
