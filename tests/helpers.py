"""Test-only helpers: comparisons that several test files share."""
from __future__ import annotations

import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def sin_angle(Ua: np.ndarray, Ub: np.ndarray) -> float:
    """sin of the largest principal angle between span(Ua) and span(Ub) (orthonormal
    columns): ‖Ub − Ua(Uaᵀ Ub)‖₂ (reading Q10; arccos cannot resolve 1e-8)."""
    Ua = np.asarray(Ua, dtype=np.float64)
    Ub = np.asarray(Ub, dtype=np.float64)
    if Ua.shape[1] == 0:
        return 0.0
    R = Ub - Ua @ (Ua.T @ Ub)
    return float(np.linalg.norm(R, 2))


def cluster_sin_angle(Ua, Ub, s, k, rel=1e-12):
    """Largest principal angle over the leading k columns, grouping columns whose
    σ agree within rel·σ1 (equal σ make single vectors non-unique, reading Q10).
    Columns with σ = 0 (within rel·σ1) are skipped."""
    s = np.asarray(s)
    worst = 0.0
    j = 0
    tol = rel * max(s[0], 1e-300)
    while j < k:
        if s[j] <= tol:
            break
        e = j + 1
        while e < k and abs(s[e] - s[j]) <= tol:
            e += 1
        if e == k and e < len(s) and abs(s[e] - s[j]) <= tol:
            # cluster crosses the truncation point: not comparable
            break
        worst = max(worst, sin_angle(Ua[:, j:e], Ub[:, j:e]))
        j = e
    return worst


_KAT = None


def curand_kat_binary() -> str:
    """Compile tests/curand_kat.cpp (cuRAND header, host path) once per session."""
    global _KAT
    if _KAT is None:
        out = os.path.join(tempfile.gettempdir(), f"rpca_curand_kat_{os.getpid()}")
        subprocess.run(["g++", "-O1", "-I/usr/local/cuda/include", "-o", out,
                        os.path.join(HERE, "curand_kat.cpp")], check=True)
        _KAT = out
    return _KAT


def curand_philox(rows):
    """rows: iterable of (c0,c1,c2,c3,k0,k1) → (N, 4) uint32 array from cuRAND's header."""
    txt = "\n".join(" ".join(str(int(v)) for v in r) for r in rows) + "\n"
    res = subprocess.run([curand_kat_binary()], input=txt, capture_output=True, text=True, check=True)
    return np.array([[int(v) for v in line.split()] for line in res.stdout.strip().splitlines()],
                    dtype=np.uint64).astype(np.uint32)
