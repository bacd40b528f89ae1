"""Time the int8-emulated fp64 A·X (rp.apply_int8emu: row exponents + X planes +
the pass) against the DMMA pass (rp.apply) on a C3-sized A, with a per-kernel
profile of the emulated call.  python tools/gpu/emu_micro.py [n] [l] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1412_3510_b200 as rp
import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
l = int(sys.argv[2]) if len(sys.argv) > 2 else 42
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda", 0)
A = synth.make_c3(n=n, device=dev)
X = torch.randn(n, l, device=dev, dtype=torch.float64)
for name, fn in (("dmma", lambda: rp.apply(A, X)), ("int8emu", lambda: rp.apply_int8emu(A, X))):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:8s} {e0.elapsed_time(e1) / reps:8.3f} ms/call", flush=True)
with rp.profile() as p:
    for _ in range(reps):
        rp.apply_int8emu(A, X)
    torch.cuda.synchronize()
agg = {}
for k, ms in p.records:
    c, s = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, s + ms)
for k, (c, s) in agg.items():
    print(f"  {k:14s} {c // reps}x {s / c:8.3f} ms" + (f"  {A.numel() * 8 / 1e9 / (s / c):6.2f} TB/s" if k in ("ax_f64_emu", "emu_row_exp") else ""))
d = (rp.apply_int8emu(A, X) - rp.apply(A, X)).abs().max().item()
print("max |emu − dmma|", d, "max |A·X|", rp.apply(A, X).abs().max().item())
