"""Out-of-core A (RPCA_FLAG_STREAM_A):
a host A streamed through two device chunk buffers per pass, and the N2
schedule's fused round (Aᵀ(A·Z) from one stream of A).
Small chunks (RPCA_STREAM_CHUNK_MB) force several chunks per pass."""
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


def compare(res_g, res_o, k, tol_s=1e-10, tol_a=1e-8):
    Ug, Sg, Vg = [t.cpu().numpy().astype(np.float64) for t in res_g]
    Uo, So, Vo = res_o
    assert np.max(np.abs(Sg - So) / So) < tol_s, (Sg, So)
    assert cluster_sin_angle(Uo, Ug, So, k) < tol_a
    assert cluster_sin_angle(Vo, Vg, So, k) < tol_a


@pytest.fixture
def small_chunks(monkeypatch):
    monkeypatch.setenv("RPCA_STREAM_CHUNK_MB", "2")  # ≈ 1 MB per chunk row-block ⇒ many chunks


def chunks_staged(fn):
    with rp.profile() as p:
        out = fn()
        torch.cuda.synchronize()
    return out, p.total("h2d_chunk")[0]


@pytest.mark.parametrize("dtype,raw", [(torch.float64, True), (torch.float64, False), (torch.float32, False)])
def test_streamed_pca_matches_oracle(small_chunks, dtype, raw):
    m, n, k, l, its = 20000, 300, 10, 12, 2
    A = synth.make_c1(m=m, n=n, seed=3, device=dev())
    if not raw:
        A += torch.linspace(-4, 4, n, device=dev(), dtype=torch.float64)
    A = A.to(dtype).contiguous()
    Ah = A.cpu().pin_memory()
    res, staged = chunks_staged(lambda: rp.pca(Ah, k, raw=raw, its=its, l=l, seed=0, stream_a=True))
    nch = -(-m * n * A.element_size() // (2 << 20))
    assert staged >= (2 * its + 2) * 2  # every pass streamed, several chunks each
    o = oracle.pca(A.cpu().numpy(), k, raw=raw, its=its, l=l, seed=0)
    tol = (1e-10, 1e-8) if dtype == torch.float64 else (1e-4, 1e-3)
    compare(res, o, k, *tol)
    # the resident-A call on the device agrees to rounding
    rd = rp.pca(A, k, raw=raw, its=its, l=l, seed=0)
    assert np.max(np.abs(res[1].numpy() - rd[1].cpu().numpy()) / rd[1].cpu().numpy()) < (1e-12 if dtype == torch.float64 else 1e-4)
    # diffsnorm streamed too
    est = rp.diffsnorm(Ah, *[t.to(dev()) for t in res], raw=raw, stream_a=True)
    ref = rp.diffsnorm(A, *[t.to(dev()) for t in res], raw=raw)
    assert abs(est - ref) <= (1e-9 if dtype == torch.float64 else 1e-6) * ref  # fp32: chunked fp32 partial sums
    _ = nch


@pytest.mark.parametrize("raw", [True, False])
def test_fused_round_streams_a_once_per_round(small_chunks, raw):
    """RENORM_ODD + STREAM_A: its + 3 streams of A instead of 2·its + 2, same
    results as the unfused RENORM_ODD schedule (oracle_pca_ex) within the
    variant's tolerance."""
    m, n, k, l, its = 30000, 256, 12, 14, 4
    sig = 1.0 / torch.arange(1, n + 1, dtype=torch.float64)
    A = synth.synth_dense(m, n, sig, seed=21, device=dev()).contiguous()
    if not raw:
        A += torch.linspace(-3, 3, n, device=dev(), dtype=torch.float64)
    Ah = A.cpu().pin_memory()
    res, staged_f = chunks_staged(lambda: rp.pca(Ah, k, raw=raw, its=its, l=l, seed=2, renorm_odd=True,
                                                 stream_a=True))
    _, staged_u = chunks_staged(lambda: rp.pca(Ah, k, raw=raw, its=its, l=l, seed=2, stream_a=True))
    per_pass = staged_u // (2 * its + 2)
    assert staged_u == per_pass * (2 * its + 2)
    assert staged_f == per_pass * (its + 3)
    o = oracle.pca(A.cpu().numpy(), k, raw=raw, its=its, l=l, seed=2, renorm_odd=True)
    compare(res, o, k, tol_s=1e-9, tol_a=1e-7)


def test_streamed_eigens(small_chunks):
    P = synth.make_c3(n=2048, device=dev())
    Ph = P.cpu().pin_memory()
    (U, lam), staged = chunks_staged(lambda: rp.eigens(Ph, 20, its=2, l=22, seed=0, stream_a=True))
    assert staged >= 4 * 2  # its + 2 passes, several chunks each
    Uo, lo = oracle.eigens(P.cpu().numpy(), 20, its=2, l=22, seed=0)
    assert np.max(np.abs(lam.numpy() - lo) / lo) < 1e-10
    assert cluster_sin_angle(Uo, U.numpy(), lo, 20) < 1e-8
