"""Run-to-run check of the fp32 tcgen05 Aᵀ·Y pass: repeated calls on the same
inputs must agree bitwise and with the fp64 product (rel. 1e-4); prints the
corrupted rows of any disagreeing call.  python tools/gpu/aty_f32_diag.py [lib] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if len(sys.argv) > 1 and sys.argv[1] != "-":
    os.environ["RPCA_LIB_PATH"] = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import paper_1412_3510_b200 as rp  # noqa: E402

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
A32 = torch.randn(400000, 600, generator=g, device=dev, dtype=torch.float32) + 3.0
bad_total = 0
for l in (22, 32, 40, 44, 64, 52):
    Q = torch.randn(400000, l, generator=g, device=dev, dtype=torch.float64)
    ref = A32.double().T @ Q
    bad = 0
    for i in range(reps):
        out = rp.apply(A32, Q, adjoint=True)
        d = (out - ref).abs()
        err = (d.max() / ref.abs().max()).item()
        if err > 1e-4:
            bad += 1
            rows = torch.nonzero(d.amax(1) > 1e-4 * ref.abs().max()).flatten().tolist()
            print(f"l={l} call {i}: err {err:.3e} rows {rows[:8]}...{rows[-4:]} ({len(rows)})", flush=True)
    print(f"l={l}: {bad}/{reps} corrupted", flush=True)
    bad_total += bad
print("TOTAL corrupted", bad_total)
