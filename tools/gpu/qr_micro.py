"""Householder TSQR (rp.qr) against the pipeline's LU-Cholesky-QR2
(rp.orthonormalize) on the configs' block shapes: µs per call (CUDA events)
and the orthogonality ‖QᵀQ − I‖.

  python tools/gpu/qr_micro.py [m:l,...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1412_3510_b200 as rp  # noqa: E402

shapes = [tuple(int(v) for v in s.split(":")) for s in
          (sys.argv[1] if len(sys.argv) > 1 else
           "4000:22,100000:22,32768:42,1000000:32,2000000:52,10000000:32").split(",")]
for m, l in shapes:
    g = torch.Generator(device="cuda").manual_seed(m + l)
    Y = torch.randn(m, l, generator=g, device="cuda", dtype=torch.float64) * torch.logspace(
        0, -3, l, device="cuda", dtype=torch.float64)
    out = []
    for name, fn in (("tsqr", rp.qr), ("lu_cholqr2", rp.orthonormalize)):
        for _ in range(2):
            fn(Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            r = fn(Y)
        e1.record()
        torch.cuda.synchronize()
        Q = r[0]
        orth = float(torch.linalg.matrix_norm(Q.T @ Q - torch.eye(l, device="cuda", dtype=torch.float64)))
        out.append(f"{name} {1e3 * e0.elapsed_time(e1) / 5:9.1f} us (orth {orth:.1e})")
    print(f"m={m:9d} l={l:2d}  " + "   ".join(out), flush=True)
