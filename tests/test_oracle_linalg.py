"""Pins for the oracle's building blocks against LAPACK (numpy/scipy, test-only)
and against the identities that define them.

LU  — PAPER.md:382-404 ("[Q,R] = lu(Q)"), reading Q3.  LAPACK getrf uses the
      same partial-pivoting rule (first index of the largest |·|), so scipy's
      permuted-L factor must agree with the oracle's L in original row order.
QR  — PAPER.md:169-172, 406-425 (unpivoted, reading Q4); unique for full rank
      once diag(R) > 0.
SVD — PAPER.md:133-139 (eq. i3), one-sided Jacobi (reading Q9/Q18).
A·X, Aᵀ·Y, centring — PAPER.md:427-435.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle


def rand(m, n, seed):
    return np.random.default_rng(seed).standard_normal((m, n))


# ----------------------------------------------------------------- LU
@pytest.mark.parametrize("m,l,seed", [(50, 7, 0), (300, 22, 1), (5000, 12, 2), (22, 22, 3)])
def test_lu_matches_lapack(m, l, seed):
    Y = rand(m, l, seed)
    L, U, piv = oracle.lu_renorm(Y)
    PL, Ul = sla.lu(Y, permute_l=True)          # Y = PL·Ul, PL in original row order
    assert np.allclose(U, Ul, rtol=1e-12, atol=1e-12 * np.abs(Y).max())
    assert np.allclose(L, PL, rtol=1e-12, atol=1e-12)
    assert np.abs(L).max() <= 1.0 + 1e-15            # GEPP bound
    assert np.linalg.norm(L @ U - Y) <= 1e-14 * np.linalg.norm(Y) * np.sqrt(m)
    Lp = L[piv]                                      # pivot rows: unit lower triangular
    assert np.array_equal(np.diag(Lp), np.ones(l))
    assert np.all(np.triu(Lp, 1) == 0)


def test_lu_identity_and_scaling():
    I = np.eye(9)[:, :6]
    L, U, piv = oracle.lu_renorm(I)
    assert np.array_equal(L, I) and np.array_equal(U, np.eye(6))
    Y = rand(40, 6, 11)
    L1, _, _ = oracle.lu_renorm(Y)
    L2, _, _ = oracle.lu_renorm(Y * 1e30)
    assert np.allclose(L1, L2, rtol=1e-13, atol=1e-15)
    assert np.abs(L2).max() <= 1.0


def test_lu_span_and_zero_pivot():
    # rank-2 block with 4 columns: two zero pivots (reading Q3)
    Y = np.zeros((10, 4))
    Y[:, 0] = np.arange(1, 11)
    Y[:, 1] = 2 * Y[:, 0]
    Y[3, 2] = 5.0
    L, U, piv = oracle.lu_renorm(Y)
    assert U[1, 1] == 0.0                    # exact zero pivot
    assert np.allclose(L @ U, Y, atol=1e-13)
    assert len(set(piv.tolist())) == 4
    for j in np.nonzero(np.diag(U) == 0)[0]:
        col = L[:, j]
        assert col[piv[j]] == 1.0 and np.count_nonzero(col) == 1
    # full-rank: span(L) = span(Y)
    Y = rand(60, 5, 4)
    L, _, _ = oracle.lu_renorm(Y)
    Qy = np.linalg.qr(Y)[0]
    Ql = np.linalg.qr(L)[0]
    assert np.linalg.norm(Ql - Qy @ (Qy.T @ Ql), 2) < 1e-12


# ----------------------------------------------------------------- QR
@pytest.mark.parametrize("m,l,seed", [(30, 5, 0), (400, 22, 1), (7000, 42, 2), (12, 12, 3)])
def test_qr_matches_lapack(m, l, seed):
    Y = rand(m, l, seed)
    Q, R = oracle.house_qr(Y)
    Qn, Rn = np.linalg.qr(Y)
    d = np.sign(np.diag(Rn))
    Qn, Rn = Qn * d, (Rn.T * d).T
    assert np.allclose(R, Rn, rtol=1e-12, atol=1e-12 * np.linalg.norm(Y))
    assert np.allclose(Q, Qn, atol=1e-12)
    assert np.linalg.norm(Q.T @ Q - np.eye(l)) < 1e-14 * l
    assert np.linalg.norm(Q @ R - Y) < 1e-14 * np.linalg.norm(Y) * np.sqrt(l)
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)


def test_qr_rank_deficient_still_orthonormal():
    Y = np.zeros((50, 6))
    Y[:, :3] = rand(50, 3, 9)
    Y[:, 3] = Y[:, 0] + Y[:, 1]                      # dependent column
    Q, R = oracle.house_qr(Y)                        # cols 4, 5 exactly zero
    assert np.linalg.norm(Q.T @ Q - np.eye(6)) < 1e-13
    assert np.linalg.norm(Q @ R - Y) < 1e-13 * np.linalg.norm(Y)
    Q0, R0 = oracle.house_qr(np.zeros((8, 3)))
    assert np.allclose(Q0.T @ Q0, np.eye(3)) and np.all(R0 == 0)


# ----------------------------------------------------------------- Jacobi
@pytest.mark.parametrize("n,l,seed", [(20, 4, 0), (500, 22, 1), (4000, 12, 2), (42, 42, 3)])
def test_jacobi_svd_matches_lapack(n, l, seed):
    G = rand(n, l, seed) * np.logspace(0, -6, l)
    V, s, W = oracle.jacobi_svd(G)
    sn = np.linalg.svd(G, compute_uv=False)
    assert np.allclose(s, sn, rtol=1e-12)
    assert np.all(np.diff(s) <= 0)
    assert np.linalg.norm(V.T @ V - np.eye(l)) < 1e-13 * l
    assert np.linalg.norm(W.T @ W - np.eye(l)) < 1e-13 * l
    assert np.linalg.norm(V * s @ W.T - G) < 1e-13 * np.linalg.norm(G)


def test_jacobi_closed_forms():
    V, s, W = oracle.jacobi_svd(np.diag([1.0, 3.0, 2.0]))
    assert np.array_equal(s, [3.0, 2.0, 1.0])
    # 2×2: singular values of [[a, b], [0, d]] are sqrt of the eigenvalues of MᵀM
    a, b, d = 3.0, 4.0, 1.0
    V, s, W = oracle.jacobi_svd(np.array([[a, b], [0.0, d]]))
    tr, det = a * a + b * b + d * d, (a * d) ** 2
    ev = np.array([(tr + np.sqrt(tr * tr - 4 * det)) / 2, (tr - np.sqrt(tr * tr - 4 * det)) / 2])
    assert np.allclose(s, np.sqrt(ev), rtol=1e-14)


def test_jacobi_rank_deficient_completion():
    G = np.zeros((10, 4))
    G[:, 0] = np.arange(10.0)
    G[:, 2] = 1.0
    V, s, W = oracle.jacobi_svd(G)
    assert s[2] == 0 and s[3] == 0
    assert np.linalg.norm(V.T @ V - np.eye(4)) < 1e-13
    assert np.linalg.norm(V * s @ W.T - G) < 1e-13 * np.linalg.norm(G)


@pytest.mark.parametrize("scale", [2.0 ** 500, 2.0 ** -500, 1e150])
def test_jacobi_extreme_scales(scale):
    """σ(c·G) = c·σ(G) at magnitudes where a·b and 1 + ζ² overflow or
    underflow in fp64 (column norms 2^±500): the rotation test and tan θ must
    not be formed from those products."""
    G = rand(300, 16, 7) * np.logspace(0, -5, 16)
    sn = np.linalg.svd(G, compute_uv=False)
    V, s, W = oracle.jacobi_svd(G * scale)
    assert np.allclose(s / scale, sn, rtol=1e-12)
    assert np.linalg.norm(V.T @ V - np.eye(16)) < 1e-13 * 16
    M = rand(12, 12, 8)
    S = M @ M.T - np.eye(12)
    mu, E = oracle.jacobi_eig(S * scale)
    ev = np.linalg.eigvalsh(S)[::-1]
    assert np.allclose(mu / scale, ev, rtol=1e-12, atol=1e-12 * np.abs(ev).max())


def test_jacobi_eig_matches_lapack():
    M = rand(30, 30, 5)
    S = M @ M.T - 3 * np.eye(30)
    mu, E = oracle.jacobi_eig(S)
    ev = np.linalg.eigvalsh(S)[::-1]
    assert np.allclose(mu, ev, rtol=1e-12, atol=1e-12 * np.abs(ev).max())
    assert np.linalg.norm(E @ np.diag(mu) @ E.T - S) < 1e-12 * np.linalg.norm(S)
    mu, E = oracle.jacobi_eig(np.diag([4.0, 9.0]))
    assert np.array_equal(mu, [9.0, 4.0])


# ----------------------------------------------------------------- A·X, Aᵀ·Y
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_apply_dense_and_adjoint(dt):
    A = rand(37, 23, 1).astype(dt)
    X, Y = rand(23, 5, 2), rand(37, 5, 3)
    Ad = A.astype(np.float64)
    assert np.allclose(oracle.apply(A, X), Ad @ X, rtol=1e-13, atol=1e-13)
    assert np.allclose(oracle.apply(A, Y, adjoint=True), Ad.T @ Y, rtol=1e-13, atol=1e-13)
    # adjoint identity <AX, Y> = <X, AᵀY>
    lhs = np.sum(oracle.apply(A, X) * Y)
    rhs = np.sum(X * oracle.apply(A, Y, adjoint=True))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Ad) * np.linalg.norm(X) * np.linalg.norm(Y)


def test_centering_equals_explicit():
    A = rand(41, 17, 4) + 3.0
    X, Y = rand(17, 4, 5), rand(41, 4, 6)
    Ac = A - A.mean(axis=0)
    assert np.allclose(oracle.apply(A, X, raw=False), Ac @ X, atol=1e-12)
    assert np.allclose(oracle.apply(A, Y, adjoint=True, raw=False), Ac.T @ Y, atol=1e-12)
    assert np.allclose(oracle.colmeans(np.array([[1.0, 3.0], [3.0, 5.0]])), [2.0, 4.0])
    const = np.tile(rand(1, 6, 7), (9, 1))         # all-equal rows: centring annihilates
    assert np.abs(oracle.apply(const, rand(6, 2, 8), raw=False)).max() < 1e-13


def _csr(A):
    rowptr = [0]
    cols, vals = [], []
    for i in range(A.shape[0]):
        nz = np.nonzero(A[i])[0]
        cols += nz.tolist()
        vals += A[i, nz].tolist()
        rowptr.append(len(cols))
    return (np.array(rowptr), np.array(cols, dtype=np.int32), np.array(vals), A.shape)


def test_csr_equals_dense():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((30, 20)) * (rng.random((30, 20)) < 0.2)
    S = _csr(A)
    X, Y = rand(20, 3, 1), rand(30, 3, 2)
    for raw in (True, False):
        assert np.allclose(oracle.apply(S, X, raw=raw), oracle.apply(A, X, raw=raw), atol=1e-13)
        assert np.allclose(oracle.apply(S, Y, adjoint=True, raw=raw),
                           oracle.apply(A, Y, adjoint=True, raw=raw), atol=1e-13)
    assert np.allclose(oracle.colmeans(S), A.mean(axis=0), atol=1e-15)
