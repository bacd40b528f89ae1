"""Per-launch times (CUDA events behind every launch) of one driver call on a
config — where the non-pass time of a PCA goes.

  python tools/gpu/launch_list.py C2 [C4 …]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_3510_b200 as rp  # noqa: E402
import synth  # noqa: E402

for name in sys.argv[1:] or ["C2"]:
    cfg = synth.CONFIGS[name]
    A = bench.make_input(cfg, torch.device("cuda", 0), rp)
    for _ in range(3):
        bench.run_step(rp, cfg, A)
    with rp.profile() as p:
        bench.run_step(rp, cfg, A)
        torch.cuda.synchronize()
    print(f"== {name}: {len(p.records)} launches, {sum(ms for _, ms in p.records):.3f} ms")
    for i, (k, ms) in enumerate(p.records):
        print(f"{i:3d} {k:22s} {1e3 * ms:9.1f} us")
    del A
    torch.cuda.empty_cache()
