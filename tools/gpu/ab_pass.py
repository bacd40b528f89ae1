"""Interleaved A/B timing of library variants in ONE process (each variant's
librpca.so loaded under its own module name), so box-to-box and
power-cap drift hit every variant alike:
   python tools/gpu/ab_pass.py <op> <rounds> <lib1> <lib2> ...
op: aty | ax (fp32 C4 passes), aty64 | ax64 (fp64 C2 passes), pca:<config>.
Prints per-variant median ms over rounds and the SM clock seen."""
import importlib.util
import os
import statistics
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import synth  # noqa: E402

op, rounds, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
pkg_init = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                        "paper_1412_3510_b200", "__init__.py")
mods = []
for i, lib in enumerate(libs):
    os.environ["RPCA_LIB_PATH"] = os.path.abspath(lib)
    spec = importlib.util.spec_from_file_location(f"rpvar{i}", pkg_init)
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    mods.append(m)

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
if op in ("aty", "ax"):
    A = synth.make_c4(device=dev)
    m_, n_, l = A.shape[0], A.shape[1], 52
    As = None
elif op in ("aty64", "ax64"):
    A = synth.make("C2", device=dev)
    m_, n_, l = A.shape[0], A.shape[1], 22
elif op in ("csr_ax", "csr_aty"):
    rp_, ci, va = synth.make("C5", device=dev)
    m_, n_, l = 10000000, 1000000, 32
    A = None
    As = [mm.CSR(rp_, ci, va, (m_, n_)) for mm in mods]
if op.startswith("pca:"):
    import bench
    cfg = synth.CONFIGS[op[4:]]
    A = bench.make_input(cfg, dev, mods[0])
    if isinstance(A, torch.Tensor):
        Ai = [A] * len(mods)
    else:  # each module's own CSR wrapper around the same device arrays
        Ai = [mm.CSR(A.rowptr, A.colind, A.vals, A.shape) for mm in mods]
    fns = [lambda rp=rp, a=a: bench.run_step(rp, cfg, a) for rp, a in zip(mods, Ai)]
else:
    X = torch.randn(n_, l, generator=g, device=dev, dtype=torch.float64)
    Q = torch.randn(m_, l, generator=g, device=dev, dtype=torch.float64)
    Ai = As if A is None else [A] * len(mods)
    if op.startswith("aty") or op == "csr_aty":
        fns = [lambda rp=rp, a=a: rp.apply(a, Q, adjoint=True) for rp, a in zip(mods, Ai)]
    else:
        fns = [lambda rp=rp, a=a: rp.apply(a, X) for rp, a in zip(mods, Ai)]

clocks, stop = [], threading.Event()


def sampler():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        stop.wait(0.05)


for f in fns:
    for _ in range(3):
        f()
torch.cuda.synchronize()
th = threading.Thread(target=sampler, daemon=True)
th.start()
times = [[] for _ in fns]
for r in range(rounds):
    for i, f in enumerate(fns):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        times[i].append(e0.elapsed_time(e1) / 3)
stop.set()
th.join()
for lib, t in zip(libs, times):
    print(f"{op:8s} {lib:40s} median {statistics.median(t):8.3f} ms  min {min(t):8.3f}  max {max(t):8.3f}")
print("sm clock MHz: median", statistics.median(clocks) if clocks else None, "min", min(clocks) if clocks else None)
