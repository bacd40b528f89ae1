"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerances:

* integer / bit work (Philox stream): bit-exact;
* one application of A (A·X, Aᵀ·Y): both sides are fp64 dot products of
  length K, so |gpu − oracle| ≤ 2·γ_K·(|A||X|), γ_K = K·u/(1−K·u) (Higham);
* whole pipelines (BASELINE.json north_star): leading-k σ relative 1e-10 and
  largest principal angle (sine form, reading Q10) < 1e-8 for fp64;
  diffsnorm within 1% of the oracle's.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1412_3510_b200 as rp
import synth
from tests.helpers import cluster_sin_angle, sin_angle

pytestmark = pytest.mark.gpu
U64 = 2.0**-53


def dev():
    return torch.device("cuda", 0)


def gamma(K):
    return K * U64 / (1 - K * U64)


# ----------------------------------------------------------------- a1: Ω
@pytest.mark.parametrize("rows,cols,seed,sid", [(1000, 12, 0, 0), (4001, 22, 7, 1), (33, 7, 2**40 + 5, 3)])
def test_omega_uniform_bit_exact(rows, cols, seed, sid):
    g = rp.omega(rows, cols, seed=seed, stream_id=sid, dist=rp.UNIFORM).cpu().numpy()
    o = oracle.omega(seed, rows, cols, dist=oracle.UNIFORM, stream=sid)
    assert np.array_equal(g, o)


@pytest.mark.parametrize("rows,cols,seed", [(1000, 12, 0), (4001, 22, 7), (32768, 42, 0)])
def test_omega_gaussian_within_ulps(rows, cols, seed):
    g = rp.omega(rows, cols, seed=seed).cpu().numpy()
    o = oracle.omega(seed, rows, cols)
    # same integer stream; log/cos/sin of two libms differ by a few ulp
    assert np.max(np.abs(g - o) / np.maximum(np.abs(o), 1.0)) <= 8 * U64 * 8
    g32 = rp.omega(rows, cols, seed=seed, round_f32=True).cpu().numpy()
    assert np.array_equal(g32, g32.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(g32 - o)) <= 2.0**-23 * 6


# ----------------------------------------------------------------- a2/a4/a6: A·X, Aᵀ·Y
SHAPES = [(1000, 500), (1003, 518), (257, 129), (4097, 64), (300, 517), (64, 64), (33, 1000)]


@pytest.mark.parametrize("m,n", SHAPES)
@pytest.mark.parametrize("l", [1, 12, 22, 42, 64])
def test_apply_dense_f64(m, n, l):
    g = torch.Generator(device="cuda").manual_seed(m * 131 + n + l)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float64)
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    An, Xn, Yn = A.cpu().numpy(), X.cpu().numpy(), Y.cpu().numpy()
    got = rp.apply(A, X).cpu().numpy()
    ref = oracle.apply(An, Xn)
    assert np.all(np.abs(got - ref) <= 2 * gamma(n) * (np.abs(An) @ np.abs(Xn)) + 1e-300)
    got = rp.apply(A, Y, adjoint=True).cpu().numpy()
    ref = oracle.apply(An, Yn, adjoint=True)
    assert np.all(np.abs(got - ref) <= 2 * gamma(m) * (np.abs(An).T @ np.abs(Yn)) + 1e-300)


@pytest.mark.parametrize("m,n,l", [(1000, 500, 12), (2050, 130, 22), (300, 517, 7)])
def test_apply_centered(m, n, l):
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float64) + 3.0
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    An = A.cpu().numpy()
    c = rp.colmeans(A)
    assert np.allclose(c.cpu().numpy(), oracle.colmeans(An), rtol=1e-14, atol=1e-14)
    Ac = An - An.mean(axis=0)
    tol = 4 * gamma(max(m, n)) * (np.abs(An).max() * max(m, n) * np.abs(X.cpu().numpy()).max())
    assert np.allclose(rp.apply(A, X, cmean=c).cpu().numpy(), oracle.apply(An, X.cpu().numpy(), raw=False),
                       atol=tol, rtol=0)
    assert np.allclose(rp.apply(A, Y, adjoint=True, cmean=c).cpu().numpy(),
                       oracle.apply(An, Y.cpu().numpy(), adjoint=True, raw=False), atol=tol * 4, rtol=0)
    del Ac


@pytest.mark.parametrize("m,n", [(777, 300), (4100, 260), (300, 4096), (1000, 518), (129, 33 * 4)])
@pytest.mark.parametrize("l", [1, 12, 22, 52, 64])
def test_apply_f32_input(m, n, l):
    """fp32 A: tcgen05 3×TF32 (lda·4 ≡ 0 mod 16) or the CUDA-core fallback; the
    3×TF32 product error is ≈ 2^-21·|a||x| per term, fp32 accumulation adds K·2^-24."""
    g = torch.Generator(device="cuda").manual_seed(8 + m + l)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float32)
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    An = A.cpu().numpy().astype(np.float64)
    bound = (3 * 2.0**-21 + 2 * n * 2.0**-24)
    got = rp.apply(A, X).cpu().numpy()
    ref = oracle.apply(A.cpu().numpy(), X.cpu().numpy())
    assert np.all(np.abs(got - ref) <= bound * (np.abs(An) @ np.abs(X.cpu().numpy())) + 1e-300)
    bound = (3 * 2.0**-21 + 2 * m * 2.0**-24)
    got = rp.apply(A, Y, adjoint=True).cpu().numpy()
    ref = oracle.apply(A.cpu().numpy(), Y.cpu().numpy(), adjoint=True)
    assert np.all(np.abs(got - ref) <= bound * (np.abs(An).T @ np.abs(Y.cpu().numpy())) + 1e-300)


# ----------------------------------------------------------------- a2: int8 emulation
# The fp64 A·X of pca/eigens for 24 < l ≤ 48 (dense_ax_emu.cu): against the
# oracle's product, within the scheme's bound — each of the n terms is exact
# to 2^-55·2^E_i·2^G_j (E_i, G_j the row / column exponents, 2^E > max|·|)
@pytest.mark.parametrize("m,n,l", [(1000, 700, 42), (257, 1026, 25), (3001, 96, 48), (128, 32, 30)])
def test_apply_int8emu_vs_oracle(m, n, l):
    g = torch.Generator(device="cuda").manual_seed(m * 11 + n + l)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float64)
    A *= 10.0 ** torch.randint(-30, 30, (m, 1), generator=g, device=dev()).double()  # rows of any scale
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    X[:, 3] *= 1e-80
    Y = rp.apply_int8emu(A, X).cpu().numpy()
    An, Xn = A.cpu().numpy(), X.cpu().numpy()
    ref = oracle.apply(An, Xn)
    rmax = 2.0 ** np.ceil(np.log2(np.abs(An).max(1) * (1 + 2**-52)))
    cmax = 2.0 ** np.ceil(np.log2(np.abs(Xn).max(0) * (1 + 2**-52)))
    bound = n * 2.0**-54 * np.outer(rmax, cmax) + 2.0**-52 * np.abs(ref)
    assert np.all(np.abs(Y - ref) <= bound)
    assert np.max(np.abs(Y - ref) / (np.abs(An) @ np.abs(Xn))) < 1e-13


def test_apply_int8emu_special_values():
    m, n, l = 300, 200, 40
    g = torch.Generator(device="cuda").manual_seed(7)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float64)
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    A[5] = 0.0                      # zero row → zero output row
    A[9, 17] = float("nan")         # non-finite row → NaN output row
    X[:, 2] = 0.0                   # zero column → zero output column
    A[40] *= 1e300                  # near the top of the range
    A[41] *= 1e-300                 # and near the bottom
    Y = rp.apply_int8emu(A, X)
    assert bool((Y[5] == 0).all()) and bool(Y[9].isnan().all())
    assert bool((torch.cat([Y[:9], Y[10:]])[:, 2] == 0).all())
    ok = torch.ones(m, dtype=torch.bool, device=dev())
    ok[9] = False
    ref = torch.tensor(oracle.apply(torch.nan_to_num(A).cpu().numpy(), X.cpu().numpy()), device=dev())
    rel = ((Y - ref).abs() / (A.abs() @ X.abs())).nan_to_num(0.0)[ok]
    assert float(rel.max()) < 1e-13
    with pytest.raises(rp.RPCAError):
        rp.apply_int8emu(A, X[:, :20])  # l ≤ 24: not an emulated shape


# ----------------------------------------------------------------- a3: LU
# the last three run persistent leaves (more leaves than resident CTAs) whose
# last leaf has an odd number of doubles (the bulk copy's 16-byte tail)
@pytest.mark.parametrize("m,l", [(100, 12), (1000, 22), (100000, 22), (70000, 42), (4096, 64), (257, 64), (22, 22),
                                 (300001, 13), (200003, 41), (1000003, 53), (600007, 29), (300005, 32)])
def test_lu_span_and_factorisation(m, l):
    g = torch.Generator(device="cuda").manual_seed(m + l)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    L, U, piv = rp.lu_renorm(Y)
    Yn, Ln, Un, pv = Y.cpu().numpy(), L.cpu().numpy(), U.cpu().numpy(), piv.cpu().numpy()
    assert len(set(pv.tolist())) == l
    Lp = Ln[pv]
    assert np.array_equal(np.diag(Lp), np.ones(l)) and np.all(np.triu(Lp, 1) == 0)
    assert np.linalg.norm(Ln @ Un - Yn) <= 1e-13 * np.linalg.norm(Yn) * np.sqrt(l)
    assert np.all(np.triu(Un) == Un)
    # span(L) = span(Y) = span(oracle's L)
    Lo, _, _ = oracle.lu_renorm(Yn)
    Qo = np.linalg.qr(Lo)[0]
    Qg = np.linalg.qr(Ln)[0]
    assert sin_angle(Qo, Qg) < 1e-11
    assert np.abs(Ln).max() < 50  # tournament pivoting keeps L bounded in practice


def test_lu_zero_pivots():
    Y = np.zeros((600, 6))
    Y[:, 0] = np.arange(1, 601)
    Y[:, 1] = 2 * Y[:, 0]
    Y[5, 2] = 3.0
    Y[400, 4] = -1.0
    L, U, piv = rp.lu_renorm(torch.tensor(Y, device=dev()))
    Ln, Un, pv = L.cpu().numpy(), U.cpu().numpy(), piv.cpu().numpy()
    assert np.allclose(Ln @ Un, Y, atol=1e-12)
    for j in np.nonzero(np.diag(Un) == 0)[0]:
        col = Ln[:, j]
        assert col[pv[j]] == 1.0 and np.count_nonzero(col) == 1


# ----------------------------------------------------------------- a5: QR
@pytest.mark.parametrize("m,l", [(100, 12), (1000, 22), (100000, 22), (70001, 42), (4096, 64), (300, 64), (64, 64)])
def test_qr_matches_oracle(m, l):
    g = torch.Generator(device="cuda").manual_seed(m * 3 + l)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    Q, R = rp.qr(Y)
    Qn, Rn, Yn = Q.cpu().numpy(), R.cpu().numpy(), Y.cpu().numpy()
    assert np.linalg.norm(Qn.T @ Qn - np.eye(l)) < 1e-14 * l * np.sqrt(m / 100 + 1)
    assert np.linalg.norm(Qn @ Rn - Yn) < 1e-14 * np.linalg.norm(Yn) * np.sqrt(l)
    assert np.all(np.tril(Rn, -1) == 0) and np.all(np.diag(Rn) >= 0)
    Qo, Ro = oracle.house_qr(Yn)
    assert np.max(np.abs(Rn - Ro)) <= 1e-12 * np.abs(Ro).max()
    assert np.max(np.abs(Qn - Qo)) <= 1e-11


def test_qr_rank_deficient():
    Y = np.zeros((5000, 8))
    rng = np.random.default_rng(1)
    Y[:, :3] = rng.standard_normal((5000, 3))
    Y[:, 3] = Y[:, 0] - Y[:, 2]
    Q, R = rp.qr(torch.tensor(Y, device=dev()))
    Qn, Rn = Q.cpu().numpy(), R.cpu().numpy()
    assert np.linalg.norm(Qn.T @ Qn - np.eye(8)) < 1e-13
    assert np.linalg.norm(Qn @ Rn - Y) < 1e-13 * np.linalg.norm(Y)


# ----------------------------------------------------------------- a7: small SVD
@pytest.mark.parametrize("n,l", [(500, 12), (4000, 22), (32768, 42), (64, 64), (300, 1), (300, 7), (900, 31),
                                 (900, 32), (900, 33)])
def test_small_svd(n, l):
    g = torch.Generator(device="cuda").manual_seed(n + l)
    G = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64) * torch.logspace(
        0, -4, l, device=dev(), dtype=torch.float64)
    Vt, s, W = rp.small_svd(G)
    Gn = G.cpu().numpy()
    Vo, so, Wo = oracle.jacobi_svd(Gn)
    sn = s.cpu().numpy()
    assert np.allclose(sn, so, rtol=1e-12)
    Vn, Wn = Vt.cpu().numpy(), W.cpu().numpy()
    assert np.linalg.norm(Vn * sn @ Wn.T - Gn) < 1e-13 * np.linalg.norm(Gn)
    assert np.linalg.norm(Vn.T @ Vn - np.eye(l)) < 1e-13 * l
    assert cluster_sin_angle(Vo, Vn, so, l) < 1e-9


@pytest.mark.parametrize("l", [22, 42])
@pytest.mark.parametrize("scale", [2.0 ** 500, 2.0 ** -500, 1e288])
def test_small_svd_extreme_scale(l, scale):
    """σ(c·G) = c·σ(G) where the column norms² over- or underflow fp64 (the
    one-warp kernel at l = 22, the shared-memory one at l = 42)."""
    rng = np.random.default_rng(l)
    Gn = rng.standard_normal((600, l)) * np.exp(-np.arange(l) / 4.0)
    sn = np.linalg.svd(Gn, compute_uv=False)
    Vt, s, W = rp.small_svd(torch.tensor(Gn * scale, device=dev()))
    assert np.allclose(s.cpu().numpy() / scale, sn, rtol=1e-12)
    Vn = Vt.cpu().numpy()
    assert np.linalg.norm(Vn.T @ Vn - np.eye(l)) < 1e-13 * l


@pytest.mark.parametrize("l", [9, 24, 40])
def test_small_svd_rank_deficient(l):
    """Repeated and zero columns: σ = 0 for l − r of them; the zero-σ columns
    of Vt are completed to an orthonormal basis (Gram–Schmidt of e_t)."""
    rng = np.random.default_rng(l)
    r = l // 3
    Gn = np.zeros((700, l))
    Gn[:, :r] = rng.standard_normal((700, r))
    Gn[:, r:2 * r] = Gn[:, :r] * 2.0
    Vt, s, W = rp.small_svd(torch.tensor(Gn, device=dev()))
    sn, Vn, Wn = s.cpu().numpy(), Vt.cpu().numpy(), W.cpu().numpy()
    so = np.linalg.svd(Gn, compute_uv=False)
    assert np.allclose(sn[:r], so[:r], rtol=1e-12)
    assert np.all(sn[r:] <= 1e-13 * so[0])
    assert np.all(np.diff(sn) <= 0)
    assert np.linalg.norm(Vn[:, :r] * sn[:r] @ Wn[:, :r].T - Gn) < 1e-13 * np.linalg.norm(Gn)
    assert np.linalg.norm(Wn.T @ Wn - np.eye(l)) < 1e-13 * l
    # the σ > 0 columns are orthonormal; completed ones are unit vectors
    # orthogonal to them and to each other (when G has l ≤ n rows)
    assert np.linalg.norm(Vn.T @ Vn - np.eye(l)) < 1e-12 * l


# ----------------------------------------------------------------- whole pca
def compare(res_g, res_o, k, tol_s=1e-10, tol_a=1e-8, skip_zero=True):
    Ug, Sg, Vg = [t.cpu().numpy().astype(np.float64) for t in res_g]
    Uo, So, Vo = res_o
    nz = So > 1e-12 * So[0] if skip_zero else np.ones(k, bool)
    assert np.max(np.abs(Sg[nz] - So[nz]) / So[nz]) < tol_s, (Sg, So)
    assert cluster_sin_angle(Uo, Ug, So, k) < tol_a
    assert cluster_sin_angle(Vo, Vg, So, k) < tol_a


def test_pca_c1_full():
    A = synth.make_c1(device=dev())
    An = A.cpu().numpy()
    res = rp.pca(A, 10, raw=True, its=2, l=12, seed=0)
    compare(res, oracle.pca(An, 10, its=2, l=12, seed=0), 10)
    # the same call again is bitwise identical (fixed-order reductions, T6)
    res2 = rp.pca(A, 10, raw=True, its=2, l=12, seed=0)
    assert all(torch.equal(a, b) for a, b in zip(res, res2))


@pytest.mark.parametrize("m,n,k,l,its,raw", [(2000, 700, 8, 10, 0, True), (700, 2000, 8, 10, 2, True),
                                             (3001, 257, 20, 22, 3, False), (513, 1025, 5, 12, 1, False),
                                             (4000, 64, 40, 64, 2, True)])
def test_pca_shapes(m, n, k, l, its, raw):
    g = torch.Generator(device="cuda").manual_seed(m + n)
    sig = torch.exp(-torch.arange(min(m, n), dtype=torch.float64) / 4.0)
    A = synth.synth_dense(m, n, sig, seed=m * 7 + n, device=dev()).contiguous()
    if not raw:
        A += torch.rand(n, generator=g, device=dev(), dtype=torch.float64) * 10 - 5
    An = A.cpu().numpy()
    res = rp.pca(A, k, raw=raw, its=its, l=l, seed=3)
    compare(res, oracle.pca(An, k, raw=raw, its=its, l=l, seed=3), k)


# fp64 dense with l > 24 takes the int8-digit emulation of A·X (dense_ax_emu.cu):
# ragged m and n (not multiples of 128 / 32), centring, the transposed path
# (m < n), and rows whose magnitudes span 10^±150 plus a zero row (the per-row
# exponent of the digit planes)
@pytest.mark.parametrize("m,n,k,l,its,raw,spread", [(3001, 777, 28, 30, 2, True, False),
                                                    (2500, 1200, 40, 48, 1, False, False),
                                                    (1000, 3001, 25, 27, 2, True, False),
                                                    (2049, 513, 30, 32, 2, True, True)])
def test_pca_emu_path(m, n, k, l, its, raw, spread):
    g = torch.Generator(device="cuda").manual_seed(m * 3 + n)
    sig = torch.exp(-torch.arange(min(m, n), dtype=torch.float64) / 6.0)
    A = synth.synth_dense(m, n, sig, seed=m * 5 + n, device=dev()).contiguous()
    if not raw:
        A += torch.rand(n, generator=g, device=dev(), dtype=torch.float64) * 10 - 5
    if spread:
        A *= 10.0 ** torch.linspace(-150, 150, m, device=dev(), dtype=torch.float64)[:, None]
        A[m // 3] = 0.0
    An = A.cpu().numpy()
    res = rp.pca(A, k, raw=raw, its=its, l=l, seed=5)
    compare(res, oracle.pca(An, k, raw=raw, its=its, l=l, seed=5), k)


def test_pca_propack_diagonal():
    """the matrices PROPACK gets wrong; zero pivots on the GPU too."""
    A = synth.propack_diag(30).to(dev())
    for seed in range(5):
        U, S, V = rp.pca(A, 20, its=2, seed=seed)
        exp = np.array([1, 1, 1] + [0.999] * 17)
        assert np.max(np.abs(S.cpu().numpy() - exp)) < 1e-10
    A = synth.propack_diag(100).to(dev())
    U, S, V = rp.pca(A, 50, its=2, seed=1)
    Sn = S.cpu().numpy()
    assert np.max(np.abs(Sn[:20] - np.array([1, 1, 1] + [0.999] * 17))) < 1e-10
    assert np.all(np.abs(Sn[20:]) < 1e-10)
    Un, Vn = U.cpu().numpy(), V.cpu().numpy()
    assert np.linalg.norm(Un.T @ Un - np.eye(50)) < 1e-10
    assert np.linalg.norm(Vn.T @ Vn - np.eye(50)) < 1e-10


def test_pca_fp32_input():
    A32 = synth.make_c1(m=3000, n=400, seed=9, device=dev()).to(torch.float32).contiguous()
    res = rp.pca(A32, 10, its=2, l=12, seed=0)
    assert res[0].dtype == torch.float32
    o = oracle.pca(A32.cpu().numpy(), 10, its=2, l=12, seed=0)
    compare(res, o, 10, tol_s=1e-4, tol_a=1e-3)


def test_pca_host_buffers_e2e():
    A = synth.make_c1(device=dev())
    Ah = A.cpu().pin_memory()
    Ug, Sg, Vg = rp.pca(Ah, 10, its=2, l=12, seed=0)
    assert Ug.device.type == "cpu"
    Ud, Sd, Vd = rp.pca(A, 10, its=2, l=12, seed=0)
    assert torch.equal(Sg, Sd.cpu()) and torch.equal(Ug, Ud.cpu()) and torch.equal(Vg, Vd.cpu())


def test_pca_errors():
    A = torch.ones(10, 8, device=dev(), dtype=torch.float64)
    for k, l, its in [(0, None, 2), (5, 4, 2), (3, 9, 2), (2, None, -1)]:
        with pytest.raises(rp.RPCAError) as e:
            rp.pca(A, k, l=l, its=its)
        assert e.value.code == rp.E_SHAPE


# ----------------------------------------------------------------- eigens, diffsnorm
@pytest.mark.parametrize("variant", ["shift_chol", "sqrt"])
def test_eigens_psd(variant):
    n, k, l = 2048, 40, 42
    A = synth.make_c3(n=n, device=dev())
    U, lam = rp.eigens(A, k, its=2, l=l, seed=0, variant=variant)
    Uo, lo = oracle.eigens(A.cpu().numpy(), k, its=2, l=l, seed=0,
                           variant=oracle.SHIFT_CHOL if variant == "shift_chol" else oracle.SQRT)
    ln = lam.cpu().numpy()
    assert np.max(np.abs(ln - lo) / lo) < 1e-10
    assert cluster_sin_angle(Uo, U.cpu().numpy(), lo, k) < 1e-8
    # the second identical call replays the captured CUDA graph: same bits
    U2, lam2 = rp.eigens(A, k, its=2, l=l, seed=0, variant=variant)
    assert torch.equal(U, U2) and torch.equal(lam, lam2)


def test_diffsnorm_matches_oracle():
    A = synth.make_c1(device=dev())
    U, S, V = rp.pca(A, 10, its=2, l=12, seed=0)
    est = rp.diffsnorm(A, U, S, V, its=20, seed=1)
    An = A.cpu().numpy()
    ref = oracle.diffsnorm(An, U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy(), its=20, seed=1)
    assert abs(est - ref) <= 1e-10 * ref
    exact = np.linalg.norm(An - (U.cpu().numpy() * S.cpu().numpy()) @ V.cpu().numpy().T, 2)
    assert exact / 2 <= est <= exact * (1 + 1e-10)
    Ac = A + 2.0
    U, S, V = rp.pca(Ac, 10, raw=False, its=2, l=12, seed=0)
    est = rp.diffsnorm(Ac, U, S, V, raw=False, its=20, seed=1)
    ref = oracle.diffsnorm(Ac.cpu().numpy(), U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy(), raw=False, its=20,
                           seed=1)
    assert abs(est - ref) <= 1e-9 * ref


# ----------------------------------------------------------------- full-size C2 (BASELINE configs[1])
@pytest.mark.slow
def test_pca_c2_full_size():
    A = synth.make_c2(device=dev())
    res = rp.pca(A, 20, raw=True, its=2, l=22, seed=0)
    o = oracle.pca(A.cpu().numpy(), 20, its=2, l=22, seed=0)
    compare(res, o, 20)


# ----------------------------------------------------------------- a9: sparse CSR
def csr_case(m, n, seed=7, planted_rows=None):
    rp_, ci, va = synth.make_c5(m=m, n=n, seed=seed, device=dev(), planted_rows=planted_rows,
                                planted_cols=min(200, n))
    A = rp.CSR(rp_, ci, va, (m, n))
    host = (rp_.cpu().numpy(), ci.cpu().numpy(), va.cpu().numpy(), (m, n))
    return A, host


def dense_of(host):
    rp_, ci, va, (m, n) = host
    D = np.zeros((m, n))
    for i in range(m):
        D[i, ci[rp_[i]:rp_[i + 1]]] += va[rp_[i]:rp_[i + 1]]
    return D


@pytest.mark.parametrize("m,n,l", [(3000, 700, 32), (1000, 2500, 12), (5000, 300, 64)])
def test_csr_apply_and_colmeans(m, n, l):
    A, host = csr_case(m, n, planted_rows=30)
    g = torch.Generator(device="cuda").manual_seed(11)
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    D = dense_of(host)
    Xn, Yn = X.cpu().numpy(), Y.cpu().numpy()
    got = rp.apply(A, X).cpu().numpy()
    assert np.all(np.abs(got - oracle.apply(host, Xn)) <= 2 * gamma(64) * (np.abs(D) @ np.abs(Xn)) + 1e-300)
    got = rp.apply(A, Y, adjoint=True).cpu().numpy()
    assert np.all(np.abs(got - oracle.apply(host, Yn, adjoint=True)) <= 2 * gamma(64) * (np.abs(D).T @ np.abs(Yn)) + 1e-300)
    c = rp.colmeans(A).cpu().numpy()
    assert np.allclose(c, oracle.colmeans(host), rtol=1e-13, atol=1e-15)
    got = rp.apply(A, Y, adjoint=True, cmean=rp.colmeans(A)).cpu().numpy()
    ref = oracle.apply(host, Yn, adjoint=True, raw=False)
    assert np.allclose(got, ref, atol=1e-11 * np.abs(ref).max())


@pytest.mark.parametrize("m,n,raw", [(10000, 1000, True), (10000, 1000, False), (800, 3000, True)])
def test_pca_csr_scaled_c5(m, n, raw):
    """C5 recipe at m = 1e4, n = 1e3 (scaled C5 pinned vs the oracle)."""
    A, host = csr_case(m, n, planted_rows=max(1, m // 100))
    k, l, its = 30, 32, 2
    res = rp.pca(A, k, raw=raw, its=its, l=l, seed=0)
    o = oracle.pca(host, k, raw=raw, its=its, l=l, seed=0)
    compare(res, o, k)
    est = rp.diffsnorm(A, *res, raw=raw, its=20, seed=1)
    ref = oracle.diffsnorm(host, *[t.cpu().numpy() for t in res], raw=raw, its=20, seed=1)
    assert abs(est - ref) <= 1e-9 * ref


def heavy_csr(m=12000, n=9000, seed=5):
    """CSR with heavy rows in A (three dense rows, n > 4096 nonzeros) and in Aᵀ
    (column 0 in every row): both directions take the chunked heavy-row path."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(m):
        if i in (7, 5000, m - 1):
            cols = np.arange(n)
        else:
            cols = np.unique(np.concatenate([[0], rng.choice(n, 6, replace=False)]))
        rows.append(cols)
    rp_ = np.zeros(m + 1, dtype=np.int64)
    rp_[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows).astype(np.int32)
    va = rng.standard_normal(len(ci))
    A = rp.CSR(torch.tensor(rp_, device=dev()), torch.tensor(ci, device=dev()), torch.tensor(va, device=dev()), (m, n))
    return A, (rp_, ci, va, (m, n))


@pytest.mark.parametrize("l", [1, 32, 52])
def test_csr_heavy_rows(l):
    A, host = heavy_csr()
    D = dense_of(host)
    g = torch.Generator(device="cuda").manual_seed(12)
    X = torch.randn(D.shape[1], l, generator=g, device=dev(), dtype=torch.float64)
    Y = torch.randn(D.shape[0], l, generator=g, device=dev(), dtype=torch.float64)
    Xn, Yn = X.cpu().numpy(), Y.cpu().numpy()
    got = rp.apply(A, X).cpu().numpy()
    assert np.all(np.abs(got - oracle.apply(host, Xn)) <= 2 * gamma(9000) * (np.abs(D) @ np.abs(Xn)) + 1e-300)
    got2 = rp.apply(A, X).cpu().numpy()
    assert np.array_equal(got, got2)  # deterministic chunk order
    got = rp.apply(A, Y, adjoint=True).cpu().numpy()
    assert np.all(np.abs(got - oracle.apply(host, Yn, adjoint=True)) <=
                  2 * gamma(12000) * (np.abs(D).T @ np.abs(Yn)) + 1e-300)


# ----------------------------------------------------------------- reig (§8(f) N1)
@pytest.mark.parametrize("n,k,l,its", [(2048, 20, 22, 2), (3001, 8, 12, 1), (1500, 30, 42, 3)])
def test_reig_indefinite_vs_oracle(n, k, l, its):
    """Symmetric indefinite A = V·diag(λ)·Vᵀ, λ_j = ±j^-1.5 alternating: reig
    against the oracle on the same bits (λ rel 1e-10, angles 1e-8), and
    against the known spectrum (the leading |λ| converge)."""
    lam_t = (-1.0) ** torch.arange(n, dtype=torch.float64) * torch.arange(1, n + 1, dtype=torch.float64) ** -1.5
    V = synth.haar_columns(n, n, n + k, device=dev())
    A = (V * lam_t.to(dev())) @ V.T
    A = 0.5 * (A + A.T)
    U, lam = rp.reig(A, k, its=its, l=l, seed=0)
    Uo, lo = oracle.reig(A.cpu().numpy(), k, its=its, l=l, seed=0)
    lg = lam.cpu().numpy()
    assert np.all(np.sign(lg) == np.sign(lo))
    assert np.max(np.abs(lg - lo) / np.abs(lo)) < 1e-10
    assert cluster_sin_angle(Uo, U.cpu().numpy(), np.abs(lo), k) < 1e-8
    assert abs(lg[0] - 1.0) < 1e-4 and abs(lg[1] + 2.0**-1.5) < 1e-3 * 2.0**-1.5  # (|λ_{l+1}|/|λ_j|)^(2its+2)
    # the error estimate of the rank-k eigen-approximation: ≥ |λ_{k+1}| (Eckart–Young)
    est = rp.diffsnorm(A, U, lam, U, its=20, seed=1)
    ref = oracle.diffsnorm(A.cpu().numpy(), Uo, lo, Uo, its=20, seed=1)
    # (the power method approaches ‖E‖ from below: 1% slack)
    assert abs(est - ref) <= 1e-2 * ref and est >= (k + 1) ** -1.5 * (1 - 1e-2)


def test_reig_spec_examples_gpu():
    """SPEC.md:233-235 on the GPU: diag(3, −2, 1, 0, …) → (3, −2); identity → 1."""
    A = torch.diag(torch.tensor([3.0, -2.0, 1.0] + [0.0] * 61, dtype=torch.float64)).to(dev())
    U, lam = rp.reig(A, 2, its=2, l=4, seed=0)
    assert np.allclose(lam.cpu().numpy(), [3.0, -2.0], atol=1e-12, rtol=0)
    U, lam = rp.reig(torch.eye(40, dtype=torch.float64, device=dev()), 1, its=1, l=3)
    assert abs(float(lam[0]) - 1.0) < 1e-13


# ----------------------------------------------------------------- renorm_odd (§8(f) N2)
@pytest.mark.parametrize("m,n,k,l,its,raw", [(20000, 1000, 20, 22, 3, True), (3001, 257, 20, 22, 4, False),
                                             (700, 2000, 8, 10, 3, True)])
def test_pca_renorm_odd_vs_oracle(m, n, k, l, its, raw):
    """RPCA_FLAG_RENORM_ODD: the interior long-side LUs are
    skipped on both sides; parity at the fp64 tolerances on spectra where the
    unrenormalised block stays well conditioned (σ_j = 1/j)."""
    g = torch.Generator(device="cuda").manual_seed(m + its)
    sig = 1.0 / torch.arange(1, min(m, n) + 1, dtype=torch.float64)
    A = synth.synth_dense(m, n, sig, seed=m + n, device=dev()).contiguous()
    if not raw:
        A += torch.rand(n, generator=g, device=dev(), dtype=torch.float64) * 10 - 5
    res = rp.pca(A, k, raw=raw, its=its, l=l, seed=4, renorm_odd=True)
    # unrenormalised blocks amplify the two sides' different rounding (the
    # accuracy the paper says this variant gives up): 10× the fp64 tolerances
    compare(res, oracle.pca(A.cpu().numpy(), k, raw=raw, its=its, l=l, seed=4, renorm_odd=True), k,
            tol_s=1e-9, tol_a=1e-7)
    # and it launches fewer LU leaves than the default schedule
    with rp.profile() as p1:
        rp.pca(A, k, raw=raw, its=its, l=l, seed=4)
        torch.cuda.synchronize()
    with rp.profile() as p2:
        rp.pca(A, k, raw=raw, its=its, l=l, seed=4, renorm_odd=True)
        torch.cuda.synchronize()
    assert p2.total("lu_leaf")[0] < p1.total("lu_leaf")[0]


def test_csr_large_operand_spmm():
    """A gathered operand X of 102 MB (n = 400000, l = 32, near the L2 size):
    A·X against the oracle elementwise and the whole PCA at the fp64
    tolerances."""
    m, n, l = 600000, 400000, 32
    A, host = csr_case(m, n, seed=13, planted_rows=m // 100)
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    got = rp.apply(A, X).cpu().numpy()
    ref = oracle.apply(host, X.cpu().numpy())
    rp_, ci, va, _ = host
    absA_X = np.zeros_like(ref)
    Xa = np.abs(X.cpu().numpy())
    rows = np.repeat(np.arange(m), np.diff(rp_))
    np.add.at(absA_X, rows, np.abs(va)[:, None] * Xa[ci])
    assert np.all(np.abs(got - ref) <= 2 * gamma(256) * absA_X + 1e-300)
    res = rp.pca(A, 30, its=2, l=32, seed=0)
    compare(res, oracle.pca(host, 30, its=2, l=32, seed=0), 30)


@pytest.mark.parametrize("l", [40, 44, 52, 64])
def test_aty_f32_repeated_calls_bitwise_stable(l):
    """The fp32 tcgen05 Aᵀ·Y pass, called repeatedly on the same inputs, gives
    the same bits every time, within 1e-4 (relative to the largest entry) of
    the fp64 product.  Regression: its split warps released each shared-memory A stage
    before their loads had returned, so the TMA could refill it under them —
    ~1 call in 6 at these shapes came back with some rows of Z off by ~1e-3
    (dense_f32_tc.cu, loads_done16)."""
    g = torch.Generator(device=dev()).manual_seed(7)
    A = torch.randn(400000, 600, generator=g, device=dev(), dtype=torch.float32) + 3.0
    Q = torch.randn(400000, l, generator=g, device=dev(), dtype=torch.float64)
    ref = A.double().T @ Q
    first = rp.apply(A, Q, adjoint=True)
    assert (first - ref).abs().max().item() <= 1e-4 * ref.abs().max().item()
    for _ in range(12):
        assert torch.equal(rp.apply(A, Q, adjoint=True), first)
