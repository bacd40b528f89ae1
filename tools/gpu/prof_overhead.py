"""Step time of one config with and without the per-launch profiling events."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synth, bench
import paper_1412_3510_b200 as rp
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg, conf = bench.workload(cfgname)
A = bench.make_input(cfg, torch.device("cuda", 0), rp)
for _ in range(3):
    bench.run_step(rp, cfg, A)
torch.cuda.synchronize()
def timed(n, prof):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if prof:
        with rp.profile() as p:
            e0.record()
            for _ in range(n): bench.run_step(rp, cfg, A)
            e1.record(); torch.cuda.synchronize()
    else:
        e0.record()
        for _ in range(n): bench.run_step(rp, cfg, A)
        e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for prof in (False, True, False, True):
    timed(2, prof)
    print(cfgname, "profiled" if prof else "plain", round(timed(10, prof), 4), "ms/step", flush=True)
