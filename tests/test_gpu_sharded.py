"""GPU parity of the row-sharded path through the C ABI.

P virtual ranks run on ONE GPU (rp.VirtualGroup: one host thread and one
context per rank, collectives = host-barrier-synchronised device copies and a
fixed-order sum kernel, include/rpca.h), each holding a row shard of A.  The
concatenated shards of U and the replicated S, V are compared with the CPU
oracle under the same tolerances as the single-GPU pipelines
(test_gpu_parity.py): leading-k σ relative 1e-10, largest principal angle
< 1e-8 (fp64).  Sharding changes only the pivot tournament and the order of
the cross-rank sums, never the method.
"""
import threading

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


def run_ranks(P, fn, timeout=300):
    """fn(rank) on P threads attached to one virtual group; returns the results."""
    group = rp.VirtualGroup(P)
    out, err = [None] * P, [None] * P

    def worker(r):
        try:
            torch.cuda.set_device(0)
            group.attach(r)
            out[r] = fn(r)
            torch.cuda.synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e
        finally:
            rp.release_context()

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "virtual ranks hung"
    group.close()
    for e in err:
        if e is not None:
            raise e
    return out


def splits_of(m, P, uneven=True):
    if not uneven:
        return [rp.uniform_shard(m, P, r) for r in range(P)]
    w = np.arange(1, P + 1, dtype=np.float64)  # rank r gets a share ∝ r+1
    b = np.concatenate([[0], np.cumsum(w) / w.sum() * m]).round().astype(int)
    return [(int(b[r]), int(b[r + 1] - b[r])) for r in range(P)]


def compare(U, S, V, res_o, k, tol_s=1e-10, tol_a=1e-8):
    Uo, So, Vo = res_o
    nz = So > 1e-12 * So[0]
    assert np.max(np.abs(S[nz] - So[nz]) / So[nz]) < tol_s, (S, So)
    assert cluster_sin_angle(Uo, U, So, k) < tol_a
    assert cluster_sin_angle(Vo, V, So, k) < tol_a


def sharded_pca(A, P, k, uneven=True, **kw):
    m = A.shape[0]
    sp = splits_of(m, P, uneven)

    def fn(r):
        r0, ml = sp[r]
        Ar = A[r0:r0 + ml].contiguous()
        U, S, V = rp.pca(Ar, k, m_total=m, row0=r0, **kw)
        return U.cpu().double().numpy(), S.cpu().double().numpy(), V.cpu().double().numpy()

    res = run_ranks(P, fn)
    for r in range(1, P):  # S, V replicated bit for bit
        assert np.array_equal(res[r][1], res[0][1]) and np.array_equal(res[r][2], res[0][2])
    return np.concatenate([x[0] for x in res]), res[0][1], res[0][2]


@pytest.mark.parametrize("P", [2, 3, 4])
def test_sharded_pca_c1(P):
    A = synth.make_c1(device=dev())
    U, S, V = sharded_pca(A, P, 10, its=2, l=12, seed=0)
    compare(U, S, V, oracle.pca(A.cpu().numpy(), 10, its=2, l=12, seed=0), 10)


@pytest.mark.parametrize("m,n,k,l,its,raw,P", [(700, 2000, 8, 10, 2, True, 2),     # m < n: sketch Aᵀ
                                               (3001, 257, 20, 22, 3, False, 3),   # centred, ragged
                                               (513, 1025, 5, 12, 1, False, 2),
                                               (4000, 64, 40, 64, 2, True, 2),     # l = 64, P·l = 128
                                               (2000, 700, 8, 10, 0, True, 3),     # its = 0: QR only
                                               (3001, 258, 20, 30, 2, False, 3)])  # l = 30: int8-emulated A·X
def test_sharded_pca_shapes(m, n, k, l, its, raw, P):
    g = torch.Generator(device="cuda").manual_seed(m + n)
    sig = torch.exp(-torch.arange(min(m, n), dtype=torch.float64) / 4.0)
    A = synth.synth_dense(m, n, sig, seed=m * 7 + n, device=dev()).contiguous()
    if not raw:
        A += torch.rand(n, generator=g, device=dev(), dtype=torch.float64) * 10 - 5
    U, S, V = sharded_pca(A, P, k, raw=raw, its=its, l=l, seed=3)
    compare(U, S, V, oracle.pca(A.cpu().numpy(), k, raw=raw, its=its, l=l, seed=3), k)


def test_sharded_pca_many_ranks_wide_sketch():
    """8 ranks × l = 64 candidates = 512 rows: the gathered tournament needs two levels."""
    m, n, k, l = 6000, 300, 60, 64
    sig = torch.exp(-torch.arange(n, dtype=torch.float64) / 8.0)
    A = synth.synth_dense(m, n, sig, seed=17, device=dev()).contiguous()
    U, S, V = sharded_pca(A, 8, k, its=1, l=l, seed=5)
    compare(U, S, V, oracle.pca(A.cpu().numpy(), k, its=1, l=l, seed=5), k)


def test_sharded_pca_fp32():
    A32 = synth.make_c1(m=3000, n=400, seed=9, device=dev()).to(torch.float32).contiguous()
    U, S, V = sharded_pca(A32, 2, 10, its=2, l=12, seed=0)
    o = oracle.pca(A32.cpu().numpy(), 10, its=2, l=12, seed=0)
    compare(U, S, V, o, 10, tol_s=1e-4, tol_a=1e-3)


def test_sharded_pca_matches_single_gpu_closely():
    """Sharding moves only rounding: the factors agree with the 1-GPU call to ~1e-12."""
    A = synth.make_c1(device=dev())
    U1, S1, V1 = [t.cpu().numpy() for t in rp.pca(A, 10, its=2, l=12, seed=0)]
    U, S, V = sharded_pca(A, 2, 10, its=2, l=12, seed=0)
    assert np.max(np.abs(S - S1) / S1) < 1e-12
    assert np.max(np.abs(V - V1)) < 1e-9 and np.max(np.abs(U - U1)) < 1e-9  # same sign convention


def test_sharded_csr_pca_and_diffsnorm():
    m, n, k, l = 10000, 1000, 30, 32
    rp_, ci, va = synth.make_c5(m=m, n=n, seed=7, device=dev(), planted_rows=m // 100, planted_cols=200)
    host = (rp_.cpu().numpy(), ci.cpu().numpy(), va.cpu().numpy(), (m, n))
    P = 3
    sp = splits_of(m, P)

    def fn(r):
        r0, ml = sp[r]
        a, b = int(rp_[r0]), int(rp_[r0 + ml])
        Ar = rp.CSR(rp_[r0:r0 + ml + 1] - a, ci[a:b], va[a:b], (ml, n))
        U, S, V = rp.pca(Ar, k, its=2, l=l, seed=0, m_total=m, row0=r0)
        est = rp.diffsnorm(Ar, U, S, V, its=20, seed=1, m_total=m, row0=r0)
        return U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy(), est

    res = run_ranks(P, fn)
    U = np.concatenate([x[0] for x in res])
    S, V = res[0][1], res[0][2]
    compare(U, S, V, oracle.pca(host, k, its=2, l=l, seed=0), k)
    ref = oracle.diffsnorm(host, U, S, V, its=20, seed=1)
    assert all(abs(x[3] - ref) <= 1e-9 * ref for x in res)


@pytest.mark.parametrize("comm", ["virtual", "nccl"])
def test_sharded_csr_overlapped_allreduce(comm):
    """n·l·8 ≥ 32 MB: the sharded sparse Aᵀ·Y all-reduces CSR(Aᵀ)'s output in 8
    row tiles on a second stream, each overlapping the next tile's SpMM
    (driver.cu csr_aty_allreduce_overlapped) — on virtual ranks (host-barrier
    collectives) and through a 1-rank NCCL communicator inside the captured
    graph (replayed on the second call)."""
    m, n, k, l = 300000, 140000, 30, 32
    rp_, ci, va = synth.make_c5(m=m, n=n, seed=11, device=dev(), planted_rows=m // 100, planted_cols=200)
    host = (rp_.cpu().numpy(), ci.cpu().numpy(), va.cpu().numpy(), (m, n))
    o = oracle.pca(host, k, raw=False, its=2, l=l, seed=0)
    if comm == "virtual":
        P = 2
        sp = splits_of(m, P)

        def fn(r):
            r0, ml = sp[r]
            a, b = int(rp_[r0]), int(rp_[r0 + ml])
            Ar = rp.CSR(rp_[r0:r0 + ml + 1] - a, ci[a:b], va[a:b], (ml, n))
            U, S, V = rp.pca(Ar, k, raw=False, its=2, l=l, seed=0, m_total=m, row0=r0)
            return U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy()

        res = run_ranks(P, fn)
        U = np.concatenate([x[0] for x in res])
        compare(U, res[0][1], res[0][2], o, k)
        return
    out = {}

    def body():
        try:
            torch.cuda.set_device(0)
            rp.comm_init(1, 0, rp.comm_unique_id())
            A = rp.CSR(rp_, ci, va, (m, n))
            r1 = rp.pca(A, k, raw=False, its=2, l=l, seed=0, m_total=m, row0=0)
            r2 = rp.pca(A, k, raw=False, its=2, l=l, seed=0, m_total=m, row0=0)
            torch.cuda.synchronize()
            out.update(r1=r1, r2=r2)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            out["err"] = e
        finally:
            rp.release_context()

    th = threading.Thread(target=body, daemon=True)
    th.start()
    th.join(300)
    assert not th.is_alive()
    if out.get("err") is not None:
        raise out["err"]
    compare(*[t.cpu().numpy() for t in out["r1"]], o, k)
    assert all(torch.equal(a, b) for a, b in zip(out["r1"], out["r2"]))


@pytest.mark.parametrize("raw", [True, False])
def test_sharded_diffsnorm(raw):
    A = synth.make_c1(device=dev()) + (0.0 if raw else 2.0)
    U1, S1, V1 = rp.pca(A, 10, raw=raw, its=2, l=12, seed=0)
    Un, Sn, Vn = U1.cpu().numpy(), S1.cpu().numpy(), V1.cpu().numpy()
    ref = oracle.diffsnorm(A.cpu().numpy(), Un, Sn, Vn, raw=raw, its=20, seed=1)
    sp = splits_of(A.shape[0], 3)

    def fn(r):
        r0, ml = sp[r]
        return rp.diffsnorm(A[r0:r0 + ml].contiguous(), U1[r0:r0 + ml], S1, V1, raw=raw, its=20, seed=1,
                            m_total=A.shape[0], row0=r0)

    for est in run_ranks(3, fn):
        assert abs(est - ref) <= 1e-9 * ref


@pytest.mark.parametrize("variant,P", [("shift_chol", 2), ("sqrt", 3), ("shift_chol", 4)])
def test_sharded_eigens(variant, P):
    n, k, l = 2048, 40, 42
    A = synth.make_c3(n=n, device=dev())
    Uo, lo = oracle.eigens(A.cpu().numpy(), k, its=2, l=l, seed=0,
                           variant=oracle.SHIFT_CHOL if variant == "shift_chol" else oracle.SQRT)

    def fn(r):
        r0, ml = rp.uniform_shard(n, P, r)
        U, lam = rp.eigens(A[r0:r0 + ml].contiguous(), k, its=2, l=l, seed=0, variant=variant, m_total=n, row0=r0)
        return U.cpu().numpy(), lam.cpu().numpy()

    res = run_ranks(P, fn)
    for r in range(1, P):
        assert np.array_equal(res[r][1], res[0][1])
    U, lam = np.concatenate([x[0] for x in res]), res[0][1]
    assert np.max(np.abs(lam - lo) / lo) < 1e-10
    assert cluster_sin_angle(Uo, U, lo, k) < 1e-8


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_reig(P):
    """reig (§8(f) N1) on virtual ranks: the uniform row partition of a
    symmetric indefinite A, λ replicated bit for bit, U by shards."""
    n, k, l = 1537, 12, 16
    lam_t = (-1.0) ** torch.arange(n, dtype=torch.float64) * torch.arange(1, n + 1, dtype=torch.float64) ** -1.5
    V = synth.haar_columns(n, n, 99, device=dev())
    A = (V * lam_t.to(dev())) @ V.T
    A = (0.5 * (A + A.T)).contiguous()
    Uo, lo = oracle.reig(A.cpu().numpy(), k, its=2, l=l, seed=0)

    def fn(r):
        r0, ml = rp.uniform_shard(n, P, r)
        U, lam = rp.reig(A[r0:r0 + ml].contiguous(), k, its=2, l=l, seed=0, m_total=n, row0=r0)
        return U.cpu().numpy(), lam.cpu().numpy()

    res = run_ranks(P, fn)
    for r in range(1, P):
        assert np.array_equal(res[r][1], res[0][1])
    U, lam = np.concatenate([x[0] for x in res]), res[0][1]
    assert np.max(np.abs(lam - lo) / np.abs(lo)) < 1e-10
    assert cluster_sin_angle(Uo, U, np.abs(lo), k) < 1e-8


def test_sharded_apply_and_colmeans():
    m, n, l, P = 3001, 517, 22, 3
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(m, n, generator=g, device=dev(), dtype=torch.float64) + 3.0
    X = torch.randn(n, l, generator=g, device=dev(), dtype=torch.float64)
    Y = torch.randn(m, l, generator=g, device=dev(), dtype=torch.float64)
    An, Xn, Yn = A.cpu().numpy(), X.cpu().numpy(), Y.cpu().numpy()
    sp = splits_of(m, P)

    def fn(r):
        r0, ml = sp[r]
        Ar = A[r0:r0 + ml].contiguous()
        c = rp.colmeans(Ar, m_total=m, row0=r0)
        return (rp.apply(Ar, X, m_total=m, row0=r0).cpu().numpy(),
                rp.apply(Ar, Y[r0:r0 + ml].contiguous(), adjoint=True, m_total=m, row0=r0).cpu().numpy(),
                c.cpu().numpy())

    res = run_ranks(P, fn)
    K = max(m, n)
    gam = K * 2.0**-53 / (1 - K * 2.0**-53)
    ax = np.concatenate([x[0] for x in res])
    assert np.all(np.abs(ax - oracle.apply(An, Xn)) <= 2 * gam * (np.abs(An) @ np.abs(Xn)))
    for x in res:  # the all-reduced Aᵀ·Y and the column means, identical on every rank
        assert np.array_equal(x[1], res[0][1]) and np.array_equal(x[2], res[0][2])
        assert np.all(np.abs(x[1] - oracle.apply(An, Yn, adjoint=True)) <= 2 * gam * (np.abs(An).T @ np.abs(Yn)))
    assert np.allclose(res[0][2], oracle.colmeans(An), rtol=1e-14, atol=1e-14)


def test_shard_errors():
    A = synth.make_c1(device=dev())
    with pytest.raises(rp.RPCAError) as e:  # a shard without a communicator
        rp.pca(A[:500].contiguous(), 10, m_total=1000, row0=0)
    assert e.value.code == rp.E_SHAPE

    def bad_eigens(r):  # non-uniform partition on every rank → E_SHAPE before any collective
        B = synth.make_c3(n=512, device=dev())
        r0, ml = (0, 100) if r == 0 else (100, 412)
        try:
            rp.eigens(B[r0:r0 + ml].contiguous(), 10, m_total=512, row0=r0)
        except rp.RPCAError as ex:
            return ex.code
        return None

    assert run_ranks(2, bad_eigens) == [rp.E_SHAPE, rp.E_SHAPE]


@pytest.mark.parametrize("graph", ["0", "1"])  # captured by default; "0" opts out
def test_nccl_single_rank_runs_sharded_schedule(graph, monkeypatch):
    """A 1-rank NCCL communicator drives the whole sharded schedule through real
    ncclAllReduce / ncclAllGather calls (with RPCA_NCCL_GRAPH=1 also inside the
    captured CUDA graph, replayed on the second call)."""
    monkeypatch.setenv("RPCA_NCCL_GRAPH", graph)
    A = synth.make_c1(device=dev())
    C3 = synth.make_c3(n=1024, device=dev())
    out = {}

    def body():
        torch.cuda.set_device(0)
        rp.comm_init(1, 0, rp.comm_unique_id())
        try:
            r1 = rp.pca(A, 10, its=2, l=12, seed=0, m_total=1000, row0=0)
            r2 = rp.pca(A, 10, its=2, l=12, seed=0, m_total=1000, row0=0)
            e1 = rp.eigens(C3, 20, its=2, l=22, seed=0, m_total=1024, row0=0)
            e2 = rp.eigens(C3, 20, its=2, l=22, seed=0, m_total=1024, row0=0)
            d = rp.diffsnorm(A, *r1, its=20, seed=1, m_total=1000, row0=0)
            torch.cuda.synchronize()
            out.update(r1=r1, r2=r2, e1=e1, e2=e2, d=d)
        finally:
            rp.release_context()

    def run():
        try:
            body()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            out["err"] = e

    th = threading.Thread(target=run, daemon=True)
    th.start()
    th.join(300)
    assert not th.is_alive()
    if out.get("err") is not None:
        raise out["err"]
    U, S, V = [t.cpu().numpy() for t in out["r1"]]
    compare(U, S, V, oracle.pca(A.cpu().numpy(), 10, its=2, l=12, seed=0), 10)
    assert all(torch.equal(a, b) for a, b in zip(out["r1"], out["r2"]))
    assert all(torch.equal(a, b) for a, b in zip(out["e1"], out["e2"]))
    Uo, lo = oracle.eigens(C3.cpu().numpy(), 20, its=2, l=22, seed=0)
    assert np.max(np.abs(out["e1"][1].cpu().numpy() - lo) / lo) < 1e-10
    ref = oracle.diffsnorm(A.cpu().numpy(), U, S, V, its=20, seed=1)
    assert abs(out["d"] - ref) <= 1e-9 * ref


def test_virtual_single_rank():
    A = synth.make_c1(device=dev())
    U, S, V = sharded_pca(A, 1, 10, its=2, l=12, seed=0)
    compare(U, S, V, oracle.pca(A.cpu().numpy(), 10, its=2, l=12, seed=0), 10)
