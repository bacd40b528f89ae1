"""Per-call time of rp.small_svd (QR + l×l Jacobi + Q·V; tuning aid — compare
   library variants that differ in the Jacobi kernel only):
   python tools/gpu/svd_micro.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1412_3510_b200 as rp
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = torch.device("cuda", 0)
for n, l in ((1000, 12), (4000, 22), (4000, 32), (32768, 42), (4096, 52)):
    g = torch.Generator(device=dev).manual_seed(l)
    G = torch.randn(n, l, generator=g, device=dev, dtype=torch.float64) * torch.exp(
        -torch.arange(l, device=dev, dtype=torch.float64) / 4.0)
    rp.small_svd(G)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rp.small_svd(G)
    e1.record()
    torch.cuda.synchronize()
    print(f"l={l:3d} small_svd {1000 * e0.elapsed_time(e1) / reps:8.1f} us/call", flush=True)
