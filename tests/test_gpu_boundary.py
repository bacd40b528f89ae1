"""The §8(b) boundary contract on the GPU (include/rpca.h): the CSR(Aᵀ) cache
keyed by contents, host CSR inputs, the caller-owned workspace, the
RPCA_FLAG_CHECK_FINITE domain error, the pipeline's orthonormalisation with
its Householder fallback, and the guard that keeps rows with a wide dynamic
range off the int8-emulated A·X."""
import numpy as np
import pytest
import torch

import oracle
import paper_1412_3510_b200 as rp
import synth
from tests.helpers import cluster_sin_angle

pytestmark = pytest.mark.gpu
U64 = 2.0**-53


def dev():
    return torch.device("cuda", 0)


def compare(res_g, res_o, k, tol_s=1e-10, tol_a=1e-8):
    Ug, Sg, Vg = [t.cpu().numpy().astype(np.float64) for t in res_g]
    Uo, So, Vo = res_o
    assert np.max(np.abs(Sg - So) / So) < tol_s, (Sg, So)
    assert cluster_sin_angle(Uo, Ug, So, k) < tol_a
    assert cluster_sin_angle(Vo, Vg, So, k) < tol_a


def csr_host(A):
    return (A.rowptr.cpu().numpy(), A.colind.cpu().numpy(), A.vals.cpu().numpy(), A.shape)


# ------------------------------------------------- CSR(Aᵀ) cache
def test_csr_cache_detects_new_contents_at_same_addresses():
    """Two different matrices with the same nnz at the SAME device addresses
    (an in-place edit, and a freed-and-reallocated matrix) must each give their
    own result — the transpose cache is keyed by a fingerprint of the contents."""
    m, n, k, l = 6000, 900, 10, 12
    rp_, ci, va = synth.make_c5(m=m, n=n, seed=3, device=dev(), planted_rows=60, planted_cols=150)
    A = rp.CSR(rp_, ci, va, (m, n))
    res1 = rp.pca(A, k, its=2, l=l, seed=0)
    compare(res1, oracle.pca(csr_host(A), k, its=2, l=l, seed=0), k)
    # in place: new values, same pointers, same nnz
    g = torch.Generator(device="cuda").manual_seed(9)
    A.vals.copy_(torch.randn(A.vals.shape, generator=g, device=dev(), dtype=torch.float64))
    res2 = rp.pca(A, k, its=2, l=l, seed=0)
    compare(res2, oracle.pca(csr_host(A), k, its=2, l=l, seed=0), k)
    assert not torch.equal(res1[1], res2[1])
    # column indices changed in place (rows keep their counts; new sorted columns)
    cols = torch.sort(torch.randint(0, n, (m, 10), generator=g, device=dev()), dim=1).values
    ok = bool((cols[:, 1:] != cols[:, :-1]).all())
    if ok and int(A.rowptr[-1]) == m * 10 and bool((A.rowptr.diff() == 10).all()):
        A.colind.copy_(cols.reshape(-1).to(torch.int32))
        res3 = rp.pca(A, k, its=2, l=l, seed=0)
        compare(res3, oracle.pca(csr_host(A), k, its=2, l=l, seed=0), k)
    # a different matrix built after freeing the first: the allocator may hand
    # back the same addresses
    ptrs = (A.rowptr.data_ptr(), A.colind.data_ptr(), A.vals.data_ptr())
    nnz = A.vals.numel()
    del A, rp_, ci, va
    rp2, ci2, va2 = synth.make_c5(m=m, n=n, seed=4, device=dev(), planted_rows=60, planted_cols=150)
    B = rp.CSR(rp2, ci2, va2, (m, n))
    resB = rp.pca(B, k, its=2, l=l, seed=0)
    compare(resB, oracle.pca(csr_host(B), k, its=2, l=l, seed=0), k)
    _ = (ptrs, nnz)


def test_host_csr_end_to_end():
    """location = RPCA_HOST for CSR: the three arrays copied and transposed inside
    the call — the same kernels on the same bytes as the device CSR."""
    m, n = 8000, 1000
    rp_, ci, va = synth.make_c5(m=m, n=n, seed=7, device=dev(), planted_rows=80, planted_cols=200)
    Ad = rp.CSR(rp_, ci, va, (m, n))
    Ah = rp.CSR(rp_.cpu().pin_memory(), ci.cpu().pin_memory(), va.cpu().pin_memory(), (m, n))
    for raw in (True, False):
        Ud, Sd, Vd = rp.pca(Ad, 30, raw=raw, its=2, l=32, seed=0)
        Uh, Sh, Vh = rp.pca(Ah, 30, raw=raw, its=2, l=32, seed=0)
        assert Uh.device.type == "cpu"
        assert torch.equal(Sh, Sd.cpu()) and torch.equal(Uh, Ud.cpu()) and torch.equal(Vh, Vd.cpu())
        est_d = rp.diffsnorm(Ad, Ud, Sd, Vd, raw=raw)
        est_h = rp.diffsnorm(Ah, Ud, Sd, Vd, raw=raw)
        assert est_d == est_h


# ------------------------------------------------- caller-owned workspace
@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_caller_workspace(kind):
    if kind == "dense":
        A = synth.make_c1(m=3000, n=700, device=dev())
        k, l = 10, 12
    else:
        rp_, ci, va = synth.make_c5(m=5000, n=800, seed=2, device=dev(), planted_rows=50, planted_cols=100)
        A = rp.CSR(rp_, ci, va, (5000, 800))
        k, l = 20, 22
    ref = rp.pca(A, k, raw=False, its=2, l=l, seed=1)
    need = rp.workspace_query(rp.OP_PCA, A, k, l, 2)
    need_d = rp.workspace_query(rp.OP_DIFFSNORM, A, k)
    buf = torch.empty(max(need, need_d), dtype=torch.uint8, device=dev())
    rp.set_workspace(buf)
    try:
        got = rp.pca(A, k, raw=False, its=2, l=l, seed=1)
        assert all(torch.equal(a, b) for a, b in zip(ref, got))
        got2 = rp.pca(A, k, raw=False, its=2, l=l, seed=1)  # graph replay inside the caller's memory
        assert all(torch.equal(a, b) for a, b in zip(ref, got2))
        rp.diffsnorm(A, *got, raw=False)
        rp.set_workspace(buf[: need // 2])  # too small: RPCA_E_WORKSPACE, nothing launched
        with pytest.raises(rp.RPCAError) as e:
            rp.pca(A, k, raw=False, its=2, l=l, seed=1)
        assert e.value.code == rp.E_WORKSPACE
    finally:
        rp.set_workspace(None)
    got3 = rp.pca(A, k, raw=False, its=2, l=l, seed=1)
    assert all(torch.equal(a, b) for a, b in zip(ref, got3))


# ------------------------------------------------- RPCA_FLAG_CHECK_FINITE
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_check_finite(bad):
    A = synth.make_c1(m=2000, n=300, device=dev())
    A[1234, 17] = bad
    with pytest.raises(rp.RPCAError) as e:
        rp.pca(A, 10, its=2, l=12, check_finite=True)
    assert e.value.code == rp.E_NONFINITE
    rp.pca(A, 10, its=2, l=12)  # without the flag the call completes (outputs unspecified)
    P = synth.make_c3(n=512, device=dev())
    P[100, 3] = bad
    with pytest.raises(rp.RPCAError) as e:
        rp.eigens(P, 10, l=12, check_finite=True)
    assert e.value.code == rp.E_NONFINITE
    A2 = synth.make_c1(m=2000, n=300, device=dev())
    U, S, V = rp.pca(A2, 10, its=2, l=12)
    A2[5, 5] = bad
    with pytest.raises(rp.RPCAError) as e:
        rp.diffsnorm(A2, U, S, V, check_finite=True)
    assert e.value.code == rp.E_NONFINITE
    rp_, ci, va = synth.make_c5(m=3000, n=500, seed=1, device=dev(), planted_rows=30, planted_cols=100)
    va[77] = bad
    with pytest.raises(rp.RPCAError) as e:
        rp.pca(rp.CSR(rp_, ci, va, (3000, 500)), 10, l=12, check_finite=True)
    assert e.value.code == rp.E_NONFINITE
    # finite inputs pass with the flag on, bit-identical to the flag off
    A3 = synth.make_c1(m=2000, n=300, device=dev())
    r1 = rp.pca(A3, 10, its=2, l=12, check_finite=True)
    r2 = rp.pca(A3, 10, its=2, l=12)
    assert all(torch.equal(a, b) for a, b in zip(r1, r2))


# ------------------------------------------------- a5: the pipeline's orthonormalisation
@pytest.mark.parametrize("m,l,cond", [(50000, 22, 1e10), (20001, 42, 1e12), (4096, 64, 1e8)])
def test_orthonormalize_ill_conditioned(m, l, cond):
    """LU-Cholesky-QR2 on a block with κ up to 1e12: LU's bounded multipliers keep
    L well conditioned, so no fallback is needed and Q is orthonormal to u."""
    g = torch.Generator(device="cuda").manual_seed(m + l)
    U = torch.linalg.qr(torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64))[0]
    W = torch.linalg.qr(torch.randn(l, l, generator=g, device=dev(), dtype=torch.float64))[0]
    s = torch.logspace(0, -np.log10(cond), l, device=dev(), dtype=torch.float64)
    Y = (U * s) @ W.T
    Q, R, used = rp.orthonormalize(Y)
    assert not used
    Qn, Rn, Yn = Q.cpu().numpy(), R.cpu().numpy(), Y.cpu().numpy()
    assert np.linalg.norm(Qn.T @ Qn - np.eye(l)) < 1e-14 * l
    assert np.linalg.norm(Qn @ Rn - Yn) < 1e-14 * np.linalg.norm(Yn) * np.sqrt(l)
    assert np.all(np.tril(Rn, -1) == 0) and np.all(np.diag(Rn) >= 0)
    # |R| agrees with the oracle's Householder R in its well-determined part
    Ro = oracle.house_qr(Yn)[1]
    assert abs(Rn[0, 0] - Ro[0, 0]) <= 1e-13 * Ro[0, 0]


def test_orthonormalize_breakdown_falls_back_to_householder():
    """A block whose partial-pivoting L is the classic unit lower triangle of −1's
    (κ(L) ≈ 2^l): Cholesky of LᵀL breaks down; the call redoes it with TSQR."""
    m, l = 3000, 60
    Y = torch.zeros(m, l, dtype=torch.float64, device=dev())
    Y[:l, :l] = torch.tril(-torch.ones(l, l, dtype=torch.float64, device=dev()), -1) + torch.eye(
        l, dtype=torch.float64, device=dev())
    Q, R, used = rp.orthonormalize(Y)
    assert used
    Qn, Rn, Yn = Q.cpu().numpy(), R.cpu().numpy(), Y.cpu().numpy()
    assert np.linalg.norm(Qn.T @ Qn - np.eye(l)) < 1e-13 * l
    assert np.linalg.norm(Qn @ Rn - Yn) < 1e-13 * np.linalg.norm(Yn)
    Qo, Ro = oracle.house_qr(Yn)
    assert np.max(np.abs(Rn - Ro)) <= 1e-12 * np.abs(Ro).max()


# ------------------------------------------------- a2: fp32 tcgen05 A·X over several K-chunks
@pytest.mark.parametrize("m,n", [(777, 8200), (300, 12301)])
@pytest.mark.parametrize("l", [1, 12, 52])
def test_apply_f32_multi_k_chunk(m, n, l):
    """n > 4096: the fp32 pass accumulates 4096-wide K-chunks in fp32 and adds the
    chunks in fp64 (reading Q15); bound per chunk 3·2^-21 + 2·4096·2^-24."""
    g = torch.Generator(device="cuda").manual_seed(n + l)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float32)
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    An, Xn = A.cpu().numpy(), X.cpu().numpy()
    got = rp.apply(A, X).cpu().numpy()
    ref = oracle.apply(An, Xn)
    bound = (3 * 2.0**-21 + 2 * 4096 * 2.0**-24) * (np.abs(An.astype(np.float64)) @ np.abs(Xn))
    assert np.all(np.abs(got - ref) <= bound + 1e-300)
    # and a centred fp32 PCA at this width against the oracle
    if l == 12:
        A += torch.rand(n, generator=g, device=dev(), dtype=torch.float32) * 6 - 3
        res = rp.pca(A, 10, raw=False, its=2, l=12, seed=0)
        o = oracle.pca(A.cpu().numpy(), 10, raw=False, its=2, l=12, seed=0)
        Sg = res[1].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(Sg - o[1]) / o[1]) < 1e-4


# ------------------------------------------------- a2: the emulation's dynamic-range guard
def _kernels(fn):
    with rp.profile() as p:
        out = fn()
        torch.cuda.synchronize()
    return out, {n for n, _ in p.records}


@pytest.mark.parametrize("spike", [1e12, 1e4])
def test_emulation_guard_intra_row_range(spike):
    """One entry per row scaled by `spike`: the int8 emulation's error
    is relative to the row maximum, so the guard keeps such an A on the fp64 DMMA
    passes and the PCA meets the fp64 tolerances; a plain Gaussian A of the same
    shape takes the emulation."""
    m, n, k, l = 3000, 1000, 40, 42
    g = torch.Generator(device="cuda").manual_seed(int(np.log10(spike)))
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float64)
    res, names = _kernels(lambda: rp.pca(A, k, its=2, l=l, seed=0))
    assert "ax_f64_emu" in names
    cols = torch.randint(0, n, (m,), generator=g, device=dev())
    A[torch.arange(m, device=dev()), cols] *= spike
    res, names = _kernels(lambda: rp.pca(A, k, its=2, l=l, seed=0))
    assert "ax_f64_emu" not in names
    compare(res, oracle.pca(A.cpu().numpy(), k, its=2, l=l, seed=0), k)
    # elementwise fp64-class: the first pass A·Ω of that call against γ_n·|A||Ω|
    Om = rp.omega(n, l, seed=0)
    Y = rp.apply(A, Om).cpu().numpy()
    An, On = A.cpu().numpy(), Om.cpu().numpy()
    gam = n * U64 / (1 - n * U64)
    assert np.all(np.abs(Y - An @ On) <= 2 * gam * (np.abs(An) @ np.abs(On)))
