"""CPU model of the row-sharded schedule (DESIGN.md
"Multi-GPU") over a torch.distributed process group — test infrastructure.

It runs, rank by rank with real collectives (gloo here), exactly the data
movement the CUDA driver performs with NCCL: Ω rows by global offset, A·X local,
Aᵀ·Y and the centring sums all-reduced, the LU's tournament candidates
all-gathered and a final GEPP over the stacked candidates, the Cholesky-QR
Grams all-reduced, U returned for the local rows and V replicated.  The local
arithmetic is the oracle's (oracle/, plain C) so that a wrong exchange — a
missing reduction, a wrong row offset, a dropped candidate — shows up as a
mismatch against oracle.pca on the whole matrix.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import oracle


def allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).clone()
    dist.all_reduce(t)
    return t.numpy()


def allgather(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def lu_sharded(Y, r0):
    """Tournament LU across ranks: local GEPP nominates l rows, the stacked
    winners of all ranks (in rank order) pick the global pivots; L = Y·U⁻¹."""
    l = Y.shape[1]
    _, _, piv = oracle.lu_renorm(Y)
    cand = np.concatenate([Y[piv], (r0 + piv)[:, None].astype(np.float64)], axis=1)
    stacked = np.concatenate(allgather(cand))
    _, U, _ = oracle.lu_renorm(stacked[:, :l])
    d = np.diag(U)
    Ui = np.linalg.inv(U + np.diag(np.where(d == 0.0, 1.0, 0.0)))  # zero-pivot rule (reading Q3)
    return Y @ Ui


def qr_sharded(Y, r0):
    """LU-Cholesky-QR2 with all-reduced Grams: Y = Q·R, diag(R) ≥ 0."""
    Q = lu_sharded(Y, r0)
    for _ in range(2):
        G = allreduce(Q.T @ Q)
        R1 = np.linalg.cholesky(G).T
        Q = np.linalg.solve(R1.T, Q.T).T
    R = allreduce(Q.T @ Y)  # R = QᵀY (upper up to rounding)
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return Q * s, (R.T * s).T


def pca(A_loc, m, r0, k, raw=True, its=2, l=None, seed=0):
    """Sharded randomized PCA of the m-row matrix whose rows [r0, r0+ml) are A_loc."""
    l = k + 2 if l is None else l
    ml, n = A_loc.shape
    trans = m < n
    cm = None if raw else allreduce(A_loc.sum(axis=0)) / m

    def ax(X):
        Y = A_loc @ X
        return Y if cm is None else Y - (cm @ X)[None, :]

    def aty(Y):
        Z = A_loc.T @ Y
        if cm is not None:
            Z = Z - np.outer(cm, Y.sum(axis=0))
        return allreduce(Z)

    fwd, adj = (aty, ax) if trans else (ax, aty)
    # sharded block = the m-long one
    lu_y = (lambda Y: oracle.lu_renorm(Y)[0]) if trans else (lambda Y: lu_sharded(Y, r0))
    lu_z = (lambda Z: lu_sharded(Z, r0)) if trans else (lambda Z: oracle.lu_renorm(Z)[0])
    qr_y = (lambda Y: oracle.house_qr(Y)) if trans else (lambda Y: qr_sharded(Y, r0))
    qr_z = (lambda Z: qr_sharded(Z, r0)) if trans else (lambda Z: oracle.house_qr(Z))
    Om = oracle.omega(seed, m, l)[r0:r0 + ml] if trans else oracle.omega(seed, n, l)
    Y = fwd(Om)
    Y = qr_y(Y)[0] if its == 0 else lu_y(Y)
    for it in range(1, its + 1):
        Z = lu_z(adj(Y))
        Y = fwd(Z)
        Y = lu_y(Y) if it < its else qr_y(Y)[0]
    QB, R = qr_z(adj(Y))
    Vr, s, W = oracle.jacobi_svd(R)
    if not trans:
        V, U = QB @ Vr[:, :k], Y @ W[:, :k]
    else:
        V, U = Y @ W[:, :k], QB @ Vr[:, :k]
    idx = np.argmax(np.abs(V), axis=0)  # largest-|·| entry of each V column positive (lowest index)
    sg = np.where(V[idx, np.arange(k)] < 0, -1.0, 1.0)
    return U * sg, s[:k], V * sg
