"""Per-kernel times of the fp32 passes at the C4 size (tuning aid):
   python tools/gpu/pass_micro.py [m] [n] [l] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1412_3510_b200 as rp
import synth
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2000000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
l = int(sys.argv[3]) if len(sys.argv) > 3 else 52
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
A = synth.make_c4(m=m, n=n, device=dev)
X = torch.randn(n, l, generator=g, device=dev, dtype=torch.float64)
Q = torch.randn(m, l, generator=g, device=dev, dtype=torch.float64)
for _ in range(2):
    rp.apply(A, X)
    rp.apply(A, Q, adjoint=True)
torch.cuda.synchronize()
gb = m * n * 4 / 1e9
for name, fn in (("A·X", lambda: rp.apply(A, X)), ("Aᵀ·Y", lambda: rp.apply(A, Q, adjoint=True))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) / reps
    print(f"{name:6s} {per:8.3f} ms/call (split + pass + reduce)  {gb / per:6.2f} TB/s of A", flush=True)
with rp.profile() as p:
    for _ in range(reps):
        rp.apply(A, X)
        rp.apply(A, Q, adjoint=True)
    torch.cuda.synchronize()
agg = {}
for k, ms in p.records:
    c, s_ = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, s_ + ms)
for k, (c, s_) in agg.items():
    print(f"  {k:16s} {c // reps}x {s_ / c:8.3f} ms/launch" + (f"  {gb / (s_ / c):6.2f} TB/s" if "f32_tc" in k else ""))
