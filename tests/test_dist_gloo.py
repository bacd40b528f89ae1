"""world_size-2 CPU tests (gloo) of the multi-GPU host logic: the row-shard plan
bench.py uses, its max-over-ranks timing reduction, and the sharded schedule
(tests/dist_model.py — the same exchanges the CUDA driver makes over NCCL)
against the oracle on the whole matrix."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import paper_1412_3510_b200 as rp
import synth
from tests.helpers import cluster_sin_angle


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, fn_name, args, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        res = globals()[fn_name](rank, ws, *args)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(res, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


def run_gloo(fn_name, args=(), ws=2):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(ws, free_port(), fn_name, args, d), nprocs=ws, join=True)
        return [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True).tolist() for r in range(ws)]


# ------------------------------------------------------------------ shard plan
@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("ws", [1, 2, 3, 8])
def test_plan_shard_partitions_rows(name, ws):
    cfg = synth.CONFIGS[name]
    plans = [bench.plan_shard(cfg, ws, r) for r in range(ws)]
    m_total = plans[0]["m_total"]
    assert all(p["m_total"] == m_total for p in plans)
    cover = sorted((p["row0"], p["row0"] + p["m_local"]) for p in plans)
    assert cover[0][0] == 0 and cover[-1][1] == m_total
    assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))  # disjoint, contiguous
    assert all(p["m_local"] >= 1 for p in plans)
    # strong scaling: one global matrix on the uniform
    # partition (the one rpca_eigens requires) — C4 at 8: 250,000 rows per GPU
    assert m_total == cfg.m and all(p["scaling"] == "strong" for p in plans)
    assert all((p["row0"], p["m_local"]) == rp.uniform_shard(cfg.m, ws, r) for r, p in enumerate(plans))
    if name == "C4" and ws == 8:
        assert all(p["m_local"] == 250000 for p in plans)
    if name == "C5" and ws == 8:
        assert all(p["m_local"] == 1250000 for p in plans)


def _max_rank(rank, ws):
    return bench.max_over_ranks(1.0 + 0.5 * rank, ws, torch.device("cpu"))


def test_max_over_ranks_gloo():
    assert run_gloo("_max_rank") == [1.5, 1.5]


# ------------------------------------------------------------------ sharded schedule
def _sharded_pca(rank, ws, A, splits, k, raw, its, l, seed):
    import tests.dist_model as dm
    r0, r1 = splits[rank], splits[rank + 1]
    U, S, V = dm.pca(A[r0:r1], A.shape[0], r0, k, raw=raw, its=its, l=l, seed=seed)
    return [U, S, V]


@pytest.mark.parametrize("m,n,k,l,its,raw,cut", [(1000, 500, 10, 12, 2, True, 380),
                                                 (600, 1500, 8, 10, 2, True, 250),   # m < n: sharded Z
                                                 (1201, 257, 20, 22, 3, False, 700),
                                                 (900, 300, 8, 10, 0, True, 450)])
def test_sharded_schedule_matches_oracle(m, n, k, l, its, raw, cut):
    sig = torch.exp(-torch.arange(min(m, n), dtype=torch.float64) / 4.0)
    A = synth.synth_dense(m, n, sig, seed=m + n).numpy()
    if not raw:
        A = A + np.linspace(-5, 5, n)[None, :]
    res = run_gloo("_sharded_pca", (A, [0, cut, m], k, raw, its, l, 3))
    U = np.concatenate([res[0][0], res[1][0]])
    S, V = res[0][1], res[0][2]
    assert np.array_equal(res[1][1], S) and np.array_equal(res[1][2], V)  # replicated
    Uo, So, Vo = oracle.pca(A, k, raw=raw, its=its, l=l, seed=3)
    assert np.max(np.abs(S - So) / So) < 1e-10
    assert cluster_sin_angle(Uo, U, So, k) < 1e-8
    assert cluster_sin_angle(Vo, V, So, k) < 1e-8
    # the sign convention is global: U·diag(S)·Vᵀ agrees entrywise
    assert np.allclose((U * S) @ V.T, (Uo * So) @ Vo.T, atol=1e-10 * So[0])


# ------------------------------------------------------------------ bench inputs per rank
class _FakeRp:
    """Stands in for the binding's CSR container on a CPU-only box."""

    class CSR:
        def __init__(self, rowptr, colind, vals, shape):
            self.rowptr, self.colind, self.vals, self.shape = rowptr, colind, vals, tuple(shape)


@pytest.mark.parametrize("ws", [2, 3])
def test_bench_shards_reassemble_the_global_matrix(ws, monkeypatch):
    """bench.make_input at N > 1 (strong scaling): every rank's rows of the
    global seeded matrix, dense and CSR — concatenated they are the 1-rank
    input bit for bit (small versions of C2 and C5 on the CPU)."""
    import synth as sy
    monkeypatch.setitem(sy.CONFIGS, "C2", sy.Config("C2", "dense", torch.float64, 1001, 57, 5, 7, 1, True, "pca",
                                                    "small C2"))
    monkeypatch.setitem(sy.CONFIGS, "C5", sy.Config("C5", "csr", torch.float64, 3001, 700, 5, 7, 1, True, "pca",
                                                    "small C5"))

    def small_make(name, device="cpu", **kw):
        if name == "C2":
            return sy.make_c2(m=1001, n=57, device=device, **kw)
        return sy.make_c5(m=3001, n=700, device=device, planted_rows=30, planted_cols=50, **kw)

    monkeypatch.setattr(sy, "make", small_make)
    dev = torch.device("cpu")
    for name in ("C2", "C5"):
        cfg = sy.CONFIGS[name]
        parts = [bench.make_input(cfg, dev, _FakeRp, bench.plan_shard(cfg, ws, r)) for r in range(ws)]
        whole = small_make(name)
        if name == "C2":
            assert torch.equal(torch.cat(parts), whole)
        else:
            rp_, ci, va = whole
            got_ci = torch.cat([p.colind for p in parts])
            got_va = torch.cat([p.vals for p in parts])
            assert torch.equal(got_ci, ci) and torch.equal(got_va, va)
            offs = [0]
            for p in parts:
                assert int(p.rowptr[0]) == 0
                offs.append(offs[-1] + int(p.rowptr[-1]))
            rebuilt = torch.cat([parts[0].rowptr] + [p.rowptr[1:] + o for p, o in zip(parts[1:], offs[1:-1])])
            assert torch.equal(rebuilt, rp_)
