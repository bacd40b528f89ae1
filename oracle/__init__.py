"""CPU oracle for the randomized PCA hot path (arXiv 1412.3510).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product (``paper_1412_3510_b200``) never imports it and
shares no code with it; see ``oracle/rpca_oracle.c`` for the algorithm, the
PAPER.md citations and the pins.

This module only marshals numpy arrays into the C library (ctypes) and builds
it on first use with gcc (``-O2 -fopenmp -ffp-contract=off``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rpca_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, E_ARG, E_SHAPE, E_NOTPSD, E_NOMEM = 0, 1, 2, 4, 9
GAUSSIAN, UNIFORM = 0, 1
SHIFT_CHOL, SQRT = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so next to its source (idempotent)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-std=gnu99",
               "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            i64, i32, u64, u32, vp, dp = C.c_int64, C.c_int, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p
            L.oracle_philox4x32_10.argtypes = [vp, vp, vp]
            L.oracle_omega.argtypes = [u64, u32, i64, i64, i32, dp]
            L.oracle_lu_renorm.argtypes = [dp, i64, i64, dp, vp]
            L.oracle_house_qr.argtypes = [dp, i64, i64, dp]
            L.oracle_jacobi_svd.argtypes = [dp, i64, i64, dp, dp]
            L.oracle_jacobi_eig.argtypes = [dp, i64, dp, dp]
            mat = [i32, i32, i64, i64, vp, i64, vp, vp, vp]
            L.oracle_pca.argtypes = mat + [i64, i32, i32, i64, u64, i32, dp, dp, dp]
            L.oracle_pca_ex.argtypes = mat + [i64, i32, i32, i64, u64, i32, i32, dp, dp, dp]
            L.oracle_eigens.argtypes = [i32, i32, i64, vp, i64, vp, vp, vp, i64, i32, i64, u64, i32, i32, dp, dp]
            L.oracle_diffsnorm.argtypes = mat + [i32, dp, dp, dp, i64, i32, u64, dp]
            L.oracle_reig.argtypes = [i32, i32, i64, vp, i64, vp, vp, vp, i64, i32, i64, u64, i32, dp, dp]
            L.oracle_apply.argtypes = mat + [i32, i32, dp, i64, dp]
            L.oracle_colmeans.argtypes = mat + [dp]
            L.oracle_num_threads.argtypes = []
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(code, what):
    if code != OK:
        raise OracleError(code, what)


def _dense_args(A):
    A = np.ascontiguousarray(A)
    if A.dtype == np.float64:
        dt = 0
    elif A.dtype == np.float32:
        dt = 1
    else:
        raise TypeError("A must be float32 or float64")
    m, n = A.shape
    return A, [0, dt, m, n, _p(A), n, None, None, None]


def _mat_args(A):
    """Dense ndarray, or a CSR triple (rowptr int64, colind int32, vals, shape)."""
    if isinstance(A, np.ndarray):
        return _dense_args(A)
    rowptr, colind, vals, shape = A
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind, dtype=np.int32)
    vals = np.ascontiguousarray(vals)
    dt = 0 if vals.dtype == np.float64 else 1
    keep = (rowptr, colind, vals)
    return keep, [1, dt, shape[0], shape[1], None, shape[1], _p(rowptr), _p(colind), _p(vals)]


def num_threads() -> int:
    return lib().oracle_num_threads()


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def omega(seed: int, rows: int, cols: int, dist: int = GAUSSIAN, stream: int = 0) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    lib().oracle_omega(seed, stream, rows, cols, dist, _p(out))
    return out


def lu_renorm(Y):
    L = np.array(Y, dtype=np.float64, order="C", copy=True)
    m, l = L.shape
    U = np.zeros((l, l))
    piv = np.zeros(l, dtype=np.int64)
    _check(lib().oracle_lu_renorm(_p(L), m, l, _p(U), _p(piv)), "lu_renorm")
    return L, U, piv


def house_qr(Y):
    Q = np.array(Y, dtype=np.float64, order="C", copy=True)
    m, l = Q.shape
    R = np.zeros((l, l))
    _check(lib().oracle_house_qr(_p(Q), m, l, _p(R)), "house_qr")
    return Q, R


def jacobi_svd(G):
    """G (n×l) = Vt·diag(s)·Wᵀ; returns (Vt, s, W)."""
    V = np.array(G, dtype=np.float64, order="C", copy=True)
    n, l = V.shape
    s = np.zeros(l)
    W = np.zeros((l, l))
    _check(lib().oracle_jacobi_svd(_p(V), n, l, _p(s), _p(W)), "jacobi_svd")
    return V, s, W


def jacobi_eig(S):
    A = np.array(S, dtype=np.float64, order="C", copy=True)
    l = A.shape[0]
    mu = np.zeros(l)
    E = np.zeros((l, l))
    _check(lib().oracle_jacobi_eig(_p(A), l, _p(mu), _p(E)), "jacobi_eig")
    return mu, E


def apply(A, X, adjoint: bool = False, raw: bool = True):
    keep, args = _mat_args(A)
    X = np.ascontiguousarray(X, dtype=np.float64)
    l = X.shape[1]
    rows = args[3] if adjoint else args[2]
    Y = np.empty((rows, l))
    _check(lib().oracle_apply(*args, int(bool(raw)), int(bool(adjoint)), _p(X), l, _p(Y)), "apply")
    return Y


def colmeans(A):
    keep, args = _mat_args(A)
    c = np.empty(args[3])
    _check(lib().oracle_colmeans(*args, _p(c)), "colmeans")
    return c


def pca(A, k: int, raw: bool = True, its: int = 2, l: int | None = None, seed: int = 0, dist: int = GAUSSIAN,
        renorm_odd: bool = False):
    """(U m×k, S k, V n×k) — PAPER.md §2 eqs. (i1)-(i4), §5 (renorm_odd: PAPER.md:442-449)."""
    keep, args = _mat_args(A)
    m, n = args[2], args[3]
    U = np.empty((m, k))
    S = np.empty(k)
    V = np.empty((n, k))
    if renorm_odd:
        _check(lib().oracle_pca_ex(*args, k, int(bool(raw)), its, -1 if l is None else l, seed, dist, 1,
                                   _p(U), _p(S), _p(V)), "pca")
    else:
        _check(lib().oracle_pca(*args, k, int(bool(raw)), its, -1 if l is None else l, seed, dist,
                                _p(U), _p(S), _p(V)), "pca")
    return U, S, V


def eigens(A, k: int, its: int = 2, l: int | None = None, seed: int = 0, dist: int = GAUSSIAN,
           variant: int = SHIFT_CHOL):
    """(U n×k, lam k) — PAPER.md §3 stabilised Nyström."""
    keep, args = _mat_args(A)
    n = args[2]
    if args[2] != args[3]:
        raise ValueError("eigens needs a square matrix")
    U = np.empty((n, k))
    lam = np.empty(k)
    a = [args[0], args[1], n, args[4], args[5], args[6], args[7], args[8]]
    _check(lib().oracle_eigens(*a, k, its, -1 if l is None else l, seed, dist, variant, _p(U), _p(lam)),
           "eigens")
    return U, lam


def reig(A, k: int, its: int = 2, l: int | None = None, seed: int = 0, dist: int = GAUSSIAN):
    """(U n×k, lam k) — self-adjoint eigendecomposition, PAPER.md:183-184 / SPEC.md:229-237
    (|lam| non-increasing, signed)."""
    keep, args = _mat_args(A)
    n = args[2]
    if args[2] != args[3]:
        raise ValueError("reig needs a square matrix")
    U = np.empty((n, k))
    lam = np.empty(k)
    a = [args[0], args[1], n, args[4], args[5], args[6], args[7], args[8]]
    _check(lib().oracle_reig(*a, k, its, -1 if l is None else l, seed, dist, _p(U), _p(lam)), "reig")
    return U, lam


def diffsnorm(A, U, S, V, raw: bool = True, its: int = 20, seed: int = 1) -> float:
    """Power-method estimate of ‖A − U diag(S) Vᵀ‖ — PAPER.md §4 l.362-371."""
    keep, args = _mat_args(A)
    U = np.ascontiguousarray(U, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    S = np.ascontiguousarray(S, dtype=np.float64)
    k = S.shape[0]
    out = C.c_double(0.0)
    _check(lib().oracle_diffsnorm(*args, int(bool(raw)), _p(U), _p(S), _p(V), k, its, seed,
                                  C.cast(C.pointer(out), C.c_void_p)), "diffsnorm")
    return out.value
