"""B200-native randomized PCA / SVD (Szlam, Kluger & Tygert, arXiv 1412.3510).

Thin Python binding over the C ABI in ``include/rpca.h`` (``librpca.so``,
sm_100a).  This module only marshals arguments: every step of the path —
Ω generation, the passes over A, LU/QR renormalisation, the small SVD, the
lift U = Q·W and the Nyström and power-method extras — runs in the library's
CUDA kernels.  PyTorch supplies device memory and the current stream.

There is no CPU fallback: importing works anywhere, but every call raises
``RuntimeError`` if the library is missing or no sm_100 GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import torch

__all__ = ["pca", "eigens", "reig", "diffsnorm", "omega", "apply", "apply_int8emu", "colmeans", "lu_renorm", "qr",
           "orthonormalize", "small_svd", "launch_count", "library_path", "RPCAError", "CSR", "profile", "clear_cache",
           "comm_unique_id", "comm_init", "comm_init_torch", "VirtualGroup", "uniform_shard", "workspace_query",
           "set_workspace"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# RPCA_LIB_PATH: an alternative build of the same library (tuning experiments)
_LIB_PATH = os.environ.get("RPCA_LIB_PATH") or os.path.join(_HERE, "librpca.so")

OK, E_ARG, E_SHAPE, E_NONFINITE, E_NOTPSD, E_CUDA, E_NCCL, E_WORKSPACE, E_NOTIMPL, E_NOMEM = range(10)
DENSE, CSR_KIND = 0, 1
F64, F32 = 0, 1
DEVICE, HOST = 0, 1
GAUSSIAN, UNIFORM = 0, 1
SHIFT_CHOL, SQRT = 0, 1
FLAG_UNIFORM_OMEGA, FLAG_OUTPUTS_HOST, FLAG_CHECK_FINITE = 0x1, 0x2, 0x4
OP_PCA, OP_EIGENS, OP_DIFFSNORM, OP_APPLY, OP_REIG = 1, 2, 3, 4, 5
FLAG_RENORM_ODD, FLAG_STREAM_A = 0x10, 0x20


class RPCAError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rpca status {code}: {msg}")
        self.code = code


class rpca_mat(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dtype", C.c_int32), ("m", C.c_int64), ("n", C.c_int64),
                ("row0", C.c_int64), ("m_local", C.c_int64), ("a", C.c_void_p), ("lda", C.c_int64),
                ("rowptr", C.c_void_p), ("colind", C.c_void_p), ("vals", C.c_void_p), ("nnz", C.c_int64),
                ("location", C.c_int32), ("reserved", C.c_int32)]


_lib = None
_lock = threading.Lock()
_ctxs = {}


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first")
        L = C.CDLL(_LIB_PATH)
        vp, i64, i32, u64, u32, dp = C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p
        pm = C.POINTER(rpca_mat)
        sig = {
            "rpca_ctx_create": [C.POINTER(vp), i32, vp, u32],
            "rpca_ctx_destroy": [vp],
            "rpca_ctx_set_stream": [vp, vp],
            "rpca_ctx_set_flags": [vp, u32],
            "rpca_ctx_sync": [vp],
            "rpca_ctx_clear_cache": [vp],
            "rpca_launch_count": [vp, C.POINTER(i64)],
            "rpca_workspace_size": [vp, C.POINTER(C.c_size_t)],
            "rpca_workspace_query": [vp, i32, pm, i64, i64, i32, C.POINTER(C.c_size_t)],
            "rpca_set_workspace": [vp, vp, C.c_size_t],
            "rpca_orthonormalize": [vp, dp, i64, i64, dp, C.POINTER(C.c_int)],
            "rpca_profile_begin": [vp],
            "rpca_profile_begin_mode": [vp, i32],
            "rpca_profile_end": [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "rpca_comm_unique_id": [vp, C.c_size_t],
            "rpca_comm_init": [vp, i32, i32, vp],
            "rpca_virtual_group_create": [i32, C.POINTER(vp)],
            "rpca_virtual_group_destroy": [vp],
            "rpca_comm_init_virtual": [vp, vp, i32],
            "rpca_omega": [vp, u64, u32, i64, i64, i32, i32, dp],
            "rpca_colmeans": [vp, pm, dp],
            "rpca_apply": [vp, pm, dp, i32, dp, i64, dp],
            "rpca_apply_int8emu": [vp, pm, dp, i64, dp],
            "rpca_lu_renorm": [vp, dp, i64, i64, dp, vp],
            "rpca_qr": [vp, dp, i64, i64, dp],
            "rpca_small_svd": [vp, dp, i64, i64, dp, dp, dp],
            "rpca_pca": [vp, pm, i64, i32, i32, i64, u64, vp, i64, vp, vp, i64],
            "rpca_eigens": [vp, pm, i64, i32, i64, u64, i32, vp, i64, vp],
            "rpca_reig": [vp, pm, i64, i32, i64, u64, vp, i64, vp],
            "rpca_diffsnorm": [vp, pm, i32, dp, i64, dp, dp, i64, i64, i32, u64, C.POINTER(C.c_double)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.rpca_last_error.restype = C.c_char_p
        L.rpca_strerror.restype = C.c_char_p
        L.rpca_strerror.argtypes = [C.c_int]
        _lib = L
        return L


def _check(code):
    if code != OK:
        L = _load()
        raise RPCAError(code, f"{L.rpca_strerror(code).decode()}: {L.rpca_last_error().decode()}")


def _ctx(device: torch.device, flags: int = 0):
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the randomized-PCA kernels need an sm_100a GPU (no CPU fallback)")
    L = _load()
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = (threading.get_ident(), idx)
    h = _ctxs.get(key)
    if h is None:
        h = C.c_void_p()
        _check(L.rpca_ctx_create(C.byref(h), idx, None, 0))
        _ctxs[key] = h
    stream = torch.cuda.current_stream(idx).cuda_stream
    _check(L.rpca_ctx_set_stream(h, C.c_void_p(stream)))
    return L, h


def release_context(device=None):
    """Destroy this thread's context on `device` (and its communicator)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    key = (threading.get_ident(), dev.index)
    h = _ctxs.pop(key, None)
    if h is not None:
        _check(_load().rpca_ctx_destroy(h))


def _ctx_flags(h, flags):
    _check(_load().rpca_ctx_set_flags(h, flags))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dtype_code(dt):
    if dt == torch.float64:
        return F64
    if dt == torch.float32:
        return F32
    raise TypeError("A must be float64 or float32")


def _dense(A: torch.Tensor, host=False, m_total=None, row0=0) -> rpca_mat:
    if A.dim() != 2 or A.stride(1) != 1:
        raise ValueError("A must be a 2-D row-major tensor (stride(1) == 1)")
    ml, n = A.shape
    m = ml if m_total is None else int(m_total)
    return rpca_mat(DENSE, _dtype_code(A.dtype), m, n, int(row0), ml, A.data_ptr(), max(A.stride(0), n), None, None,
                    None, 0, HOST if host else DEVICE, 0)


class CSR:
    """A sparse row-major matrix for the library: rowptr (int64, m+1), colind
    (int32, sorted within rows), vals (float64/float32), shape (m, n), on one
    GPU — or in (pinned) host memory: pca / eigens / diffsnorm then copy it to
    the device inside the call (the end-to-end mode)."""

    def __init__(self, rowptr, colind, vals, shape):
        self.rowptr = rowptr.to(torch.int64).contiguous()
        self.colind = colind.to(torch.int32).contiguous()
        self.vals = vals.contiguous()
        self.shape = tuple(int(x) for x in shape)
        self.device = self.vals.device
        self.dtype = self.vals.dtype

    @classmethod
    def from_torch(cls, T):
        return cls(T.crow_indices(), T.col_indices(), T.values(), T.shape)


def _as_mat(A, host=False, m_total=None, row0=0):
    """(rpca_mat, keepalive) for a dense tensor, a CSR, or a torch sparse CSR
    tensor.  With m_total given, A holds rows [row0, row0 + A.shape[0]) of an
    m_total-row matrix sharded over the ranks of the communicator."""
    if isinstance(A, torch.Tensor) and A.layout == torch.sparse_csr:
        A = CSR.from_torch(A)
    if isinstance(A, CSR):
        ml, n = A.shape
        m = ml if m_total is None else int(m_total)
        loc = HOST if A.device.type == "cpu" else DEVICE
        mat = rpca_mat(CSR_KIND, _dtype_code(A.dtype), m, n, int(row0), ml, None, n, A.rowptr.data_ptr(),
                       A.colind.data_ptr(), A.vals.data_ptr(), A.vals.numel(), loc, 0)
        return mat, A
    return _dense(A, host=host, m_total=m_total, row0=row0), A


# ---------------------------------------------------------------- multi-GPU
def uniform_shard(m: int, nranks: int, rank: int):
    """(row0, m_local) of the uniform row partition (required by eigens)."""
    pad = -(-m // nranks)
    row0 = min(m, rank * pad)
    return row0, min(pad, m - row0)


def comm_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for comm_init."""
    L = _load()
    buf = C.create_string_buffer(128)
    _check(L.rpca_comm_unique_id(buf, 128))
    return buf.raw


def comm_init(nranks: int, rank: int, uid: bytes, device=None):
    """Attach an NCCL communicator to this thread's context on `device`; later
    calls treat their A as this rank's row shard (m_total=, row0=)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    L, h = _ctx(dev)
    _check(L.rpca_comm_init(h, nranks, rank, C.create_string_buffer(bytes(uid), 128)))


def comm_init_torch(group=None, device=None):
    """comm_init over the ranks of an initialised torch.distributed group (rank 0
    draws the id, a broadcast_object_list shares it)."""
    import torch.distributed as dist
    obj = [comm_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    comm_init(dist.get_world_size(group), dist.get_rank(group), obj[0], device)


class VirtualGroup:
    """P virtual ranks on ONE GPU for testing the sharded path: each rank is a
    host thread with its own context; collectives are host-barrier-synchronised
    device copies (include/rpca.h)."""

    def __init__(self, nranks: int):
        L = _load()
        self.nranks = nranks
        self.h = C.c_void_p()
        _check(L.rpca_virtual_group_create(nranks, C.byref(self.h)))

    def attach(self, rank: int, device=None):
        """Call from the thread that will act as `rank`."""
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        L, h = _ctx(dev)
        _check(L.rpca_comm_init_virtual(h, self.h, rank))

    def close(self):
        if self.h:
            _check(_load().rpca_virtual_group_destroy(self.h))
            self.h = C.c_void_p()


def workspace_query(op: int, A, k: int = 1, l: int | None = None, its: int = 2, m_total=None, row0=0) -> int:
    """Device bytes one call of `op` (OP_PCA, OP_EIGENS, OP_DIFFSNORM, OP_APPLY) needs for A."""
    dev = A.device if isinstance(A, torch.Tensor) and A.device.type == "cuda" else torch.device(
        "cuda", torch.cuda.current_device())
    L, h = _ctx(dev)
    mat, keep = _as_mat(A, host=isinstance(A, torch.Tensor) and A.device.type == "cpu", m_total=m_total, row0=row0)
    out = C.c_size_t(0)
    _check(L.rpca_workspace_query(h, op, C.byref(mat), k, -1 if l is None else l, its, C.byref(out)))
    return out.value


def set_workspace(buf: torch.Tensor | None, device=None):
    """Use `buf` (a device tensor, 256-byte aligned, kept alive by the caller)
    as this thread's context workspace; None returns to a context-owned one."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    L, h = _ctx(buf.device if buf is not None else dev)
    if buf is None:
        _check(L.rpca_set_workspace(h, None, 0))
    else:
        _check(L.rpca_set_workspace(h, C.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size()))


def clear_cache(device=None):
    """Drop captured graphs and the cached CSR(Aᵀ) (after modifying a sparse A in place)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    L, h = _ctx(dev)
    _check(L.rpca_ctx_clear_cache(h))


def launch_count(device=None) -> int:
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    L, h = _ctx(dev)
    n = C.c_int64(0)
    _check(L.rpca_launch_count(h, C.byref(n)))
    return n.value


class profile:
    """Context manager timing library launches on the current stream:
    ``with profile() as p: ...`` then ``p.records`` = [(kernel, ms), ...].
    ``passes_only=True`` records events only around the pass kernels that
    stream A (everything between them is reported as "gap")."""

    def __init__(self, device=None, passes_only=False):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.records = []
        self.mode = 2 if passes_only else 1

    def __enter__(self):
        L, h = _ctx(self.device)
        _check(L.rpca_profile_begin_mode(h, self.mode))
        return self

    def __exit__(self, *exc):
        L, h = _ctx(self.device)
        need = C.c_size_t(0)
        _check(L.rpca_profile_end(h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value + 1)
        # second call returns the same text (records are kept until the next begin)
        _check(L.rpca_profile_end(h, buf, need.value + 1, C.byref(need)))
        for line in buf.value.decode().splitlines():
            name, ms = line.split("\t")
            self.records.append((name, float(ms)))
        return False

    def total(self, prefix):
        v = [ms for n, ms in self.records if n.startswith(prefix)]
        return len(v), sum(v)


def omega(rows: int, cols: int, seed: int = 0, stream_id: int = 0, dist: int = GAUSSIAN, round_f32: bool = False,
          device=None) -> torch.Tensor:
    """Ω (rows×cols, fp64) — PAPER.md:163-168 / 437-440; counter layout in include/rpca.h."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    L, h = _ctx(dev)
    out = torch.empty(rows, cols, dtype=torch.float64, device=dev)
    _check(L.rpca_omega(h, seed, stream_id, rows, cols, dist, int(round_f32), _ptr(out)))
    return out


def colmeans(A, m_total=None, row0=0) -> torch.Tensor:
    L, h = _ctx(A.device)
    c = torch.empty(A.shape[1], dtype=torch.float64, device=A.device)
    mat, keep = _as_mat(A, m_total=m_total, row0=row0)
    _check(L.rpca_colmeans(h, C.byref(mat), _ptr(c)))
    return c


def apply(A: torch.Tensor, X: torch.Tensor, adjoint: bool = False, cmean: torch.Tensor | None = None,
          m_total=None, row0=0):
    """Y = A·X (adjoint=False) or Aᵀ·X, optionally centred by the column means `cmean`
    (sharded: A·X gives this rank's rows, Aᵀ·X is all-reduced)."""
    L, h = _ctx(A.device)
    X = X.contiguous()
    assert X.dtype == torch.float64
    l = X.shape[1]
    rows = A.shape[1] if adjoint else A.shape[0]
    Y = torch.empty(rows, l, dtype=torch.float64, device=A.device)
    mat, keep = _as_mat(A, m_total=m_total, row0=row0)
    _check(L.rpca_apply(h, C.byref(mat), _ptr(cmean), int(adjoint), _ptr(X), l, _ptr(Y)))
    return Y


def apply_int8emu(A: torch.Tensor, X: torch.Tensor, m_total=None, row0=0):
    """Y = A·X through the int8-digit emulation of the fp64 product (the path
    pca/eigens take for dense fp64 A with 24 < l ≤ 48); for tests and benches."""
    L, h = _ctx(A.device)
    X = X.contiguous()
    assert X.dtype == torch.float64
    l = X.shape[1]
    Y = torch.empty(A.shape[0], l, dtype=torch.float64, device=A.device)
    mat, keep = _as_mat(A, m_total=m_total, row0=row0)
    _check(L.rpca_apply_int8emu(h, C.byref(mat), _ptr(X), l, _ptr(Y)))
    return Y


def lu_renorm(Y: torch.Tensor):
    """(L, U, piv): L = Y·U⁻¹ in original row order (reading Q3)."""
    L_, h = _ctx(Y.device)
    Lm = Y.contiguous().clone()
    m, l = Lm.shape
    U = torch.zeros(l, l, dtype=torch.float64, device=Y.device)
    piv = torch.zeros(l, dtype=torch.int64, device=Y.device)
    _check(L_.rpca_lu_renorm(h, _ptr(Lm), m, l, _ptr(U), _ptr(piv)))
    return Lm, U, piv


def qr(Y: torch.Tensor):
    """(Q, R) Householder TSQR, diag(R) ≥ 0."""
    L_, h = _ctx(Y.device)
    Q = Y.contiguous().clone()
    m, l = Q.shape
    R = torch.zeros(l, l, dtype=torch.float64, device=Y.device)
    _check(L_.rpca_qr(h, _ptr(Q), m, l, _ptr(R)))
    return Q, R


def orthonormalize(Y: torch.Tensor):
    """(Q, R, used_householder): the pipeline's final orthonormalisation
    (LU-Cholesky-QR2, Householder TSQR after a breakdown), diag(R) ≥ 0."""
    L_, h = _ctx(Y.device)
    Q = Y.contiguous().clone()
    m, l = Q.shape
    R = torch.zeros(l, l, dtype=torch.float64, device=Y.device)
    used = C.c_int(0)
    _check(L_.rpca_orthonormalize(h, _ptr(Q), m, l, _ptr(R), C.byref(used)))
    return Q, R, bool(used.value)


def small_svd(G: torch.Tensor):
    """G = Vt·diag(s)·Wᵀ (eq. i3 applied to Bᵀ)."""
    L_, h = _ctx(G.device)
    G = G.contiguous()
    n, l = G.shape
    Vt = torch.empty(n, l, dtype=torch.float64, device=G.device)
    s = torch.empty(l, dtype=torch.float64, device=G.device)
    W = torch.empty(l, l, dtype=torch.float64, device=G.device)
    _check(L_.rpca_small_svd(h, _ptr(G), n, l, _ptr(Vt), _ptr(s), _ptr(W)))
    return Vt, s, W


def pca(A: torch.Tensor, k: int, raw: bool = True, its: int = 2, l: int | None = None, seed: int = 0,
        uniform_omega: bool = False, m_total: int | None = None, row0: int = 0, check_finite: bool = False,
        renorm_odd: bool = False, stream_a: bool = False):
    """Rank-k PCA / SVD of A (§2 eqs. i1-i4, §5): returns (U m×k, S k, V n×k) on A's device.

    renorm_odd=True renormalises only after the odd applications of A / A*
    (PAPER.md:442-449): the interior rounds' long-side LU is skipped.
    stream_a=True (host A only) keeps A out of core: every pass streams it
    through two device chunk buffers (with renorm_odd, one stream per round).

    raw=False centres the columns implicitly.  A may also be
    a pinned host tensor: then the host→device copy and the device→host copy of
    the factors happen inside the call (the end-to-end mode).  With a
    communicator attached (comm_init / VirtualGroup.attach), A is this rank's
    row shard [row0, row0 + A.shape[0]) of an m_total-row matrix and U is
    returned for those rows (V replicated)."""
    host = A.device.type == "cpu"
    dev = torch.device("cuda", torch.cuda.current_device()) if host else A.device
    L_, h = _ctx(dev)
    m, n = A.shape  # m: local rows
    flags = ((FLAG_UNIFORM_OMEGA if uniform_omega else 0) | (FLAG_OUTPUTS_HOST if host else 0) |
             (FLAG_CHECK_FINITE if check_finite else 0) | (FLAG_RENORM_ODD if renorm_odd else 0) |
             (FLAG_STREAM_A if stream_a else 0))
    _ctx_flags(h, flags)
    outdev = torch.device("cpu") if host else dev
    pin = host
    U = torch.empty(m, k, dtype=A.dtype, device=outdev, pin_memory=pin)
    S = torch.empty(k, dtype=A.dtype, device=outdev, pin_memory=pin)
    V = torch.empty(n, k, dtype=A.dtype, device=outdev, pin_memory=pin)
    mat, keep = _as_mat(A, host=host, m_total=m_total, row0=row0)
    try:
        _check(L_.rpca_pca(h, C.byref(mat), k, int(bool(raw)), its, -1 if l is None else l, seed,
                           _ptr(U), k, _ptr(S), _ptr(V), k))
    finally:
        _ctx_flags(h, 0)
    return U, S, V


def eigens(A: torch.Tensor, k: int, its: int = 2, l: int | None = None, seed: int = 0,
           variant: str = "shift_chol", uniform_omega: bool = False, m_total: int | None = None, row0: int = 0,
           check_finite: bool = False, stream_a: bool = False):
    """Stabilised Nyström (§3) of a PSD A: returns (U n×k, lam k).
    Sharded: A holds rows uniform_shard(n, P, rank) and U comes back for them."""
    host = A.device.type == "cpu"
    dev = torch.device("cuda", torch.cuda.current_device()) if host else A.device
    L_, h = _ctx(dev)
    n = A.shape[0]  # local rows
    v = {"shift_chol": SHIFT_CHOL, "sqrt": SQRT}[variant]
    _ctx_flags(h, (FLAG_UNIFORM_OMEGA if uniform_omega else 0) | (FLAG_OUTPUTS_HOST if host else 0) |
               (FLAG_CHECK_FINITE if check_finite else 0) | (FLAG_STREAM_A if stream_a else 0))
    outdev = torch.device("cpu") if host else dev
    U = torch.empty(n, k, dtype=A.dtype, device=outdev, pin_memory=host)
    lam = torch.empty(k, dtype=A.dtype, device=outdev, pin_memory=host)
    mat, keep = _as_mat(A, host=host, m_total=m_total, row0=row0)
    try:
        _check(L_.rpca_eigens(h, C.byref(mat), k, its, -1 if l is None else l, seed, v, _ptr(U), k, _ptr(lam)))
    finally:
        _ctx_flags(h, 0)
    return U, lam


def reig(A: torch.Tensor, k: int, its: int = 2, l: int | None = None, seed: int = 0, uniform_omega: bool = False,
         m_total: int | None = None, row0: int = 0, check_finite: bool = False):
    """Eigendecomposition of a symmetric (possibly indefinite) A (PAPER.md:183-184,
    SPEC.md:229-237): returns (U n×k, lam k) with lam signed, |lam| non-increasing.
    Sharded: A holds rows uniform_shard(n, P, rank) and U comes back for them."""
    host = A.device.type == "cpu"
    dev = torch.device("cuda", torch.cuda.current_device()) if host else A.device
    L_, h = _ctx(dev)
    n = A.shape[0]
    _ctx_flags(h, (FLAG_UNIFORM_OMEGA if uniform_omega else 0) | (FLAG_OUTPUTS_HOST if host else 0) |
               (FLAG_CHECK_FINITE if check_finite else 0))
    outdev = torch.device("cpu") if host else dev
    U = torch.empty(n, k, dtype=A.dtype, device=outdev, pin_memory=host)
    lam = torch.empty(k, dtype=A.dtype, device=outdev, pin_memory=host)
    mat, keep = _as_mat(A, host=host, m_total=m_total, row0=row0)
    try:
        _check(L_.rpca_reig(h, C.byref(mat), k, its, -1 if l is None else l, seed, _ptr(U), k, _ptr(lam)))
    finally:
        _ctx_flags(h, 0)
    return U, lam


def diffsnorm(A: torch.Tensor, U: torch.Tensor, S: torch.Tensor, V: torch.Tensor, raw: bool = True, its: int = 20,
              seed: int = 1, m_total: int | None = None, row0: int = 0, check_finite: bool = False,
              stream_a: bool = False) -> float:
    """Power-method estimate of ‖A − U·diag(S)·Vᵀ‖ (§4 l.362-371).
    Sharded: A and U are this rank's rows, V replicated."""
    host = isinstance(A, torch.Tensor) and A.device.type == "cpu" or isinstance(A, CSR) and A.device.type == "cpu"
    dev = torch.device("cuda", torch.cuda.current_device()) if host else A.device
    L_, h = _ctx(dev)
    U = U.to(torch.float64).contiguous()
    V = V.to(torch.float64).contiguous()
    S = S.to(torch.float64).contiguous()
    k = S.shape[0]
    out = C.c_double(0.0)
    mat, keep = _as_mat(A, host=host, m_total=m_total, row0=row0)
    _ctx_flags(h, (FLAG_CHECK_FINITE if check_finite else 0) | (FLAG_STREAM_A if stream_a else 0))
    try:
        _check(L_.rpca_diffsnorm(h, C.byref(mat), int(bool(raw)), _ptr(U), max(k, 1), _ptr(S), _ptr(V), max(k, 1),
                                 k, its, seed, C.byref(out)))
    finally:
        _ctx_flags(h, 0)
    return out.value
