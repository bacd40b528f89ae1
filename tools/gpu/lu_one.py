"""One rp.lu_renorm on an m×l Gaussian block (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1412_3510_b200 as rp
m, l = int(sys.argv[1]), int(sys.argv[2])
Y = torch.randn(m, l, device="cuda", dtype=torch.float64)
for _ in range(2):
    rp.lu_renorm(Y)
torch.cuda.synchronize()
