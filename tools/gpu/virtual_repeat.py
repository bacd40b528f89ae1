import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1412_3510_b200 as rp, synth
from tests.test_gpu_sharded import run_ranks, splits_of
dev = torch.device("cuda", 0)
m, n, k, l = 300000, 140000, 30, 32
rp_, ci, va = synth.make_c5(m=m, n=n, seed=11, device=dev, planted_rows=m // 100, planted_cols=200)
P = 2
sp = splits_of(m, P)
def fn(r):
    r0, ml = sp[r]
    a, b = int(rp_[r0]), int(rp_[r0 + ml])
    Ar = rp.CSR(rp_[r0:r0 + ml + 1] - a, ci[a:b], va[a:b], (ml, n))
    U, S, V = rp.pca(Ar, k, raw=False, its=2, l=l, seed=0, m_total=m, row0=r0)
    return U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy()
ref = None
bad = 0
t0 = time.time()
for it in range(int(sys.argv[1])):
    res = run_ranks(P, fn)
    cur = (np.concatenate([x[0] for x in res]), res[0][1], res[0][2], res[1][1], res[1][2])
    if ref is None:
        ref = cur
        continue
    same = all(np.array_equal(a, b) for a, b in zip(ref, cur))
    if not same:
        bad += 1
        ds = np.max(np.abs(cur[1] - ref[1]) / np.abs(ref[1]))
        print(f"iter {it}: MISMATCH  max rel dS {ds:.3e}; rank-1 S vs rank-0 S equal: {np.array_equal(cur[1], cur[3])}", flush=True)
print(f"{int(sys.argv[1])} iterations, {bad} mismatches, {time.time()-t0:.1f}s")
