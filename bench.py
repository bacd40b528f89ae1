#!/usr/bin/env python
"""bench.py — rank-k randomized PCA (Szlam, Kluger & Tygert, arXiv 1412.3510) on B200.

Metric (BASELINE.json): rank-k PCA wall time (s) and per-pass HBM GB/s vs the
roofline.  A step = one whole rpca_pca call (Ω, 2·its+2 passes over A, LU/QR
renormalisations, the small SVD and the lift U = Q·W) on the workload of
BASELINE.json configs[1] (C2: dense fp64 A 100000×4000 = 3.2 GB, k = 20,
l = 22, its = 2), A resident in HBM; A is larger than L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]

Prints ONE JSON line (rank 0).  `roofline` is for the dominant kernel (the
A-streaming pass), timed with CUDA events on the library's stream inside the
timed region; `cpu_baseline` is the CPU oracle (oracle/, plain C + OpenMP) on
a bounded row sample of the same workload, extrapolated linearly in m.
--impl reference times that oracle as the reference arm.

Multi-GPU (torchrun, one rank per GPU, NCCL): A is sharded by rows
 and every config scales STRONGLY, as SURVEY §8(d) fixes it:
the same global matrix at every N, rank r holding the uniform row block
[r·⌈m/N⌉, min(m, (r+1)·⌈m/N⌉)) (C4: 250,000 rows per GPU at N = 8; C5:
1.25e6).  `value` stays the whole-job PCA time (max over ranks) and
`roofline.aggregate` the whole-job A-streaming rate against N × the peak.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "traffic.json")  # written by tools/gpu/make_traffic.py from ncu
NCU_NAME = {"ax_f64_dmma": "ax_f64_tma_kernel", "aty_f64_dmma": "aty_f64_tma_kernel", "ax_f32_tc": "ax_f32_tc_kernel",
            "ax_f64_emu": "ax_f64_emu_kernel",
            "aty_f32_tc": "aty_f32_tc_kernel", "csr_spmm": "csr_spmm"}


def ncu_traffic(config, kernel):
    """dram read+write bytes per launch of `kernel` on `config` from the committed
    ncu --set full capture (the A-streaming launches: the largest-traffic records;
    CSR: the mean of its A·X and Aᵀ·Y launches), or None."""
    try:
        with open(TRAFFIC_PATH) as f:
            d = json.load(f)[config]
    except Exception:
        return None
    prefix = NCU_NAME.get(kernel, kernel)
    recs = [r for k, v in d.items() if k.startswith(prefix) for r in v]
    if not recs:
        return None
    if kernel == "csr_spmm":
        return {"bytes": sum(r["traffic_bytes"] for r in recs) / len(recs), "source": recs[0]["source"]}
    r = max(recs, key=lambda r: r["traffic_bytes"])
    return {"bytes": r["traffic_bytes"], "source": r["source"]}
DMMA_PEAK_TF = 37.1  # fp64 tensor (DMMA) throughput measured by tools/microbench/peaks.cu, TF/s
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, GB/s


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0, help="target oracle seconds per sample run")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self._interval = sys.getswitchinterval()
            sys.setswitchinterval(0.0005)  # let the sampler in between the (GIL-releasing) library calls
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 0.5:
                time.sleep(0.0005)
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            sys.setswitchinterval(self._interval)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def plan_shard(cfg, ws, rank):
    """How rank `rank` of `ws` holds the workload: strong scaling — one global
    matrix, rows split uniformly (the partition rpca_eigens requires)."""
    pad = -(-cfg.m // ws)
    row0 = min(cfg.m, rank * pad)
    return {"scaling": "strong", "m_total": cfg.m, "row0": row0, "m_local": min(pad, cfg.m - row0)}


def sum_over_ranks(x, ws, device):
    """sum of a per-rank number over the process group (identity at ws = 1)."""
    if ws == 1:
        return float(x)
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=device, dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


def max_over_ranks(x, ws, device):
    """max of a per-rank float over the process group (identity at ws = 1)."""
    if ws == 1:
        return float(x)
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload(name):
    cfg = synth.CONFIGS[name]
    return cfg, {
        "workload": f"{name}: {cfg.desc}",
        "m": cfg.m, "n": cfg.n, "k": cfg.k, "l": cfg.l, "its": cfg.its, "raw": cfg.raw,
        "passes_over_A": (cfg.its + 2) if cfg.op == "eigens" else (2 * cfg.its + 2),
    }


def make_input(cfg, device, rp=None, plan=None):
    """This rank's rows of the config's (global, seeded) matrix."""
    plan = plan or {"row0": 0, "m_local": cfg.m}
    r0, r1 = plan["row0"], plan["row0"] + plan["m_local"]
    A = synth.make(cfg.name, device=device)
    if cfg.kind == "csr":
        rowptr, colind, vals = A
        if (r0, r1) != (0, cfg.m):
            t0, t1 = int(rowptr[r0]), int(rowptr[r1])
            rowptr = (rowptr[r0:r1 + 1] - t0).contiguous()
            colind, vals = colind[t0:t1].clone(), vals[t0:t1].clone()
        if device.type == "cuda":
            torch.cuda.synchronize()
        return rp.CSR(rowptr, colind, vals, (r1 - r0, cfg.n))
    if (r0, r1) != (0, cfg.m):
        A = A[r0:r1].clone()
    if device.type == "cuda":
        torch.cuda.synchronize()
    return A


def a_bytes(A):
    """bytes of A as stored (dense elements, or CSR row pointers + indices + values)."""
    if isinstance(A, torch.Tensor):
        return A.numel() * A.element_size()
    return (A.rowptr.numel() * 8 + A.colind.numel() * 4 + A.vals.numel() * A.vals.element_size())


def pass_bytes(A, cfg):
    """algorithmic bytes of one pass of the dominant kernel: all of A, plus for CSR
    the gathered operand rows (8·l per nonzero) and the written output rows."""
    if isinstance(A, torch.Tensor):
        return a_bytes(A)
    nnz = A.vals.numel()
    return a_bytes(A) + nnz * 8 * cfg.l + cfg.m * 8 * cfg.l


def run_step(rp, cfg, A, plan=None):
    sh = {} if plan is None or plan["m_total"] == plan["m_local"] else {"m_total": plan["m_total"],
                                                                         "row0": plan["row0"]}
    if cfg.op == "eigens":
        return rp.eigens(A, cfg.k, its=cfg.its, l=cfg.l, seed=0, **sh)
    return rp.pca(A, cfg.k, raw=cfg.raw, its=cfg.its, l=cfg.l, seed=0, **sh)


# ------------------------------------------------------------------ CPU oracle
def host_of(A):
    """A as the oracle takes it: a dense ndarray, or the CSR triple + shape."""
    if isinstance(A, torch.Tensor):
        return A.cpu().numpy()
    if isinstance(A, (tuple, list)):
        rp_, ci, va = A[:3]
        m = rp_.numel() - 1
        return (rp_.cpu().numpy(), ci.cpu().numpy(), va.cpu().numpy(), (m, None))
    return (A.rowptr.cpu().numpy(), A.colind.cpu().numpy(), A.vals.cpu().numpy(), tuple(A.shape))


def leading_rows(A_host, ms, n):
    """The leading ms rows of a dense or CSR host matrix."""
    if isinstance(A_host, np.ndarray):
        return np.ascontiguousarray(A_host[:ms])
    rp_, ci, va, _ = A_host
    nz = int(rp_[ms])
    return (np.ascontiguousarray(rp_[:ms + 1]), ci[:nz], va[:nz], (ms, n))


def oracle_sample(cfg, A_host, target_s):
    """Time the oracle (as it stands) on a leading-row sample of the workload,
    growing the sample until one run takes ≥ target_s / 4; extrapolate to full m.
    CSR samples start at n rows so that the sample keeps the m ≥ n orientation."""
    import oracle

    m = cfg.m
    ms = min(m, max(cfg.l * 4, 2000, 0 if isinstance(A_host, np.ndarray) else cfg.n))
    while True:
        As = leading_rows(A_host, ms, cfg.n)
        t0 = time.perf_counter()
        if cfg.op == "eigens":
            # the Nyström path needs a square matrix: sample its leading ms×ms block
            As = np.ascontiguousarray(A_host[:ms, :ms])
            oracle.eigens(As, cfg.k, its=cfg.its, l=cfg.l, seed=0)
        else:
            oracle.pca(As, cfg.k, raw=cfg.raw, its=cfg.its, l=cfg.l, seed=0)
        dt = time.perf_counter() - t0
        if dt >= target_s / 4 or ms >= m:
            break
        ms = min(m, int(ms * max(2.0, target_s / max(dt, 1e-3) * 0.9)))
    scale = (m / ms) ** (2 if cfg.op == "eigens" else 1)
    return ms, dt, scale


def cpu_model():
    """The host CPU model (lscpu), for cpu_baseline."""
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(cfg, A_host, target_s):
    import oracle

    ms, dt, scale = oracle_sample(cfg, A_host, target_s)
    what = (f"leading {ms}x{ms} block" if cfg.op == "eigens" else f"leading {ms} of {cfg.m} rows")
    if not isinstance(A_host, np.ndarray):
        what += " (CSR; the n-side work does not grow with m, so linear extrapolation overstates it slightly)"
    return {"value": dt * scale, "unit": "s", "cores": oracle.num_threads(), "cpu_model": cpu_model(),
            "kind": "oracle", "sample": f"oracle on the {what} ({dt:.2f} s), extrapolated "
                      f"{'quadratically in n' if cfg.op == 'eigens' else 'linearly in m'} (x{scale:.1f})"}


def reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg, conf = workload(args.config)
    import oracle

    A = synth.make(cfg.name, device="cuda" if torch.cuda.is_available() else "cpu")
    A_host = host_of(A)
    del A
    ms, dt, scale = oracle_sample(cfg, A_host, args.cpu_seconds)
    times = []
    for it in range(args.warmup + args.steps):
        As = np.ascontiguousarray(A_host[:ms, :ms]) if cfg.op == "eigens" else leading_rows(A_host, ms, cfg.n)
        t0 = time.perf_counter()
        if cfg.op == "eigens":
            oracle.eigens(As, cfg.k, its=cfg.its, l=cfg.l, seed=0)
        else:
            oracle.pca(As, cfg.k, raw=cfg.raw, its=cfg.its, l=cfg.l, seed=0)
        if it >= args.warmup:
            times.append((time.perf_counter() - t0) * scale)
    v = float(np.mean(times))
    what = (f"leading {ms}x{ms} block" if cfg.op == "eigens" else f"leading {ms} of {cfg.m} rows")
    line = {"impl": "reference", "metric": "rank-k PCA wall time (s)", "value": v, "unit": "s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if cfg.dtype == torch.float64 else "f32",
            "data": "synthetic", "config": conf,
            "cpu_baseline": {"value": v, "unit": "s", "cores": oracle.num_threads(), "cpu_model": cpu_model(),
                             "kind": "oracle",
                             "sample": f"oracle on the {what} per step, extrapolated x{scale:.1f}"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_1412_3510_b200 as rp
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        rp.comm_init_torch()  # the library's own NCCL communicator over the same ranks

    cfg, conf = workload(args.config)
    plan = plan_shard(cfg, ws, rank)
    A = make_input(cfg, dev, rp, plan)
    abytes = a_bytes(A)  # this rank's shard
    pbytes = pass_bytes(A, cfg)
    passes = conf["passes_over_A"]
    conf.update({"l2": f"A ({abytes / 1e9:.2f} GB per GPU) > L2 (126 MB): no flush needed",
                 "parallelism": f"row-sharded dp{ws} ({plan['scaling']} scaling, m_total={plan['m_total']}, "
                                f"{plan['m_local']} rows on rank 0)" if ws > 1 else "single GPU"})

    for _ in range(args.warmup):
        run_step(rp, cfg, A, plan)
    # one more warm-up step in the timed region's profile mode: the library
    # captures a separate CUDA graph per profile mode, so this keeps the
    # capture and instantiation out of the timed steps
    with rp.profile(passes_only=True):
        run_step(rp, cfg, A, plan)
    torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    stream = torch.cuda.current_stream(dev)
    launches0 = rp.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # timed region: CUDA events on the library's stream bracket only the pass
    # kernels that stream A (profile mode "passes"), so the per-launch event
    # overhead stays out of the step time
    with ClockSampler(local) as clk, rp.profile(passes_only=True) as prof:
        e0.record(stream)
        for _ in range(args.steps):
            run_step(rp, cfg, A, plan)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = e0.elapsed_time(e1)
    launches = rp.launch_count() - launches0
    t_step = max_over_ranks(ms_total / 1e3 / args.steps, ws, dev)
    a_total = sum_over_ranks(abytes, ws, dev)  # all shards' bytes (strong scaling: the global A)

    # per-kernel breakdown: the same K steps again with an event behind every
    # launch (reported as "kernels"; not part of the timed region)
    with rp.profile() as prof_all:
        for _ in range(args.steps):
            run_step(rp, cfg, A, plan)
        torch.cuda.synchronize()

    # dominant kernel: the A-streaming passes
    hbm, peak_src = peaks()
    kern = {}
    for name, msec in prof.records:
        c, s = kern.get(name, (0, 0.0))
        kern[name] = (c + 1, s + msec)
    kern_all = {}
    for name, msec in prof_all.records:
        c, s = kern_all.get(name, (0, 0.0))
        kern_all[name] = (c + 1, s + msec)
    step_ms = ms_total / args.steps
    passes_k = {k: v for k, v in kern.items() if k.startswith(("ax_", "aty_f64", "aty_f32", "aty_generic", "csr_spmm"))}
    dom = max(passes_k.items(), key=lambda kv: kv[1][1]) if passes_k else None
    roof = None
    if dom:
        cnt, tot = dom[1]
        avg_ms = tot / cnt
        achieved = pbytes / (avg_ms / 1e3) / 1e9
        achieved = max_over_ranks(-achieved, ws, dev) * -1.0  # slowest rank
        tr = ncu_traffic(cfg.name, dom[0]) if ws == 1 else None
        roof = {"bound": "hbm", "kernel": dom[0], "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": round(tr["bytes"]) if tr else None,
                "traffic_source": ("ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch: "
                                   + os.path.relpath(tr["source"], ROOT)) if tr else None,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": pbytes, "avg_launch_ms": round(avg_ms, 5),
                "share_of_step": round(tot / args.steps / step_ms, 4)}
        if tr and not isinstance(A, torch.Tensor):
            # CSR: the gather-inclusive algorithmic bytes count every gathered
            # operand row as DRAM traffic while part of X hits L2; the fraction
            # from ncu's measured DRAM bytes per launch is reported beside it
            roof["dram_based"] = {"achieved": round(tr["bytes"] / (avg_ms / 1e3) / 1e9, 1),
                                  "frac": round(tr["bytes"] / (avg_ms / 1e3) / 1e9 / hbm, 4),
                                  "note": "ncu dram bytes per launch / live launch time"}
        if dom[0] in ("ax_f64_dmma", "aty_f64_dmma") and isinstance(A, torch.Tensor):
            # the fp64 passes issue DMMA (m8n8k4) on l padded to a multiple of 8:
            # the fp64 tensor pipe, not HBM, caps them
            lp = -(-cfg.l // 8) * 8
            fl = 2.0 * A.shape[0] * A.shape[1] * lp
            tf = fl / (avg_ms / 1e3) / 1e12
            roof["fp64_tensor"] = {
                "issued_flops_per_launch": fl, "achieved_tflops": round(tf, 2), "peak_tflops": DMMA_PEAK_TF,
                "frac": round(tf / DMMA_PEAK_TF, 4),
                "hbm_frac_ceiling": round(8 * DMMA_PEAK_TF * 1e12 / (2 * lp) / 1e9 / hbm, 4),
                "peak_source": "dmma_peak of tools/microbench/peaks.cu at 1965 MHz (DESIGN.md §6)"}
        all_pass_ms = sum(v[1] for v in passes_k.values()) / args.steps
        roof["all_passes"] = {"launches_per_step": sum(v[0] for v in passes_k.values()) // args.steps,
                              "gbs_per_pass": round(abytes * passes / (all_pass_ms / 1e3) / 1e9, 1)}
        if ws > 1:  # whole-job A-streaming rate: all shards' bytes over the step time
            total = sum_over_ranks(abytes, ws, dev)
            roof["aggregate"] = {"gbs_per_pass_step": round(total * passes / t_step / 1e9, 1),
                                 "peak": hbm * ws, "frac": round(total * passes / t_step / 1e9 / (hbm * ws), 4)}
    breakdown = {k: {"launches_per_step": v[0] / args.steps, "ms_per_step": round(v[1] / args.steps, 5)}
                 for k, v in sorted(kern_all.items(), key=lambda kv: -kv[1][1])}

    e2e = None
    if not args.no_e2e:  # every rank (the call has collectives)
        if isinstance(A, torch.Tensor):
            Ah = A.cpu().pin_memory()
        else:  # host CSR: the three arrays are copied (and CSR(Aᵀ) rebuilt) inside each call
            Ah = rp.CSR(A.rowptr.cpu().pin_memory(), A.colind.cpu().pin_memory(), A.vals.cpu().pin_memory(),
                        A.shape)
        run_step(rp, cfg, Ah, plan)  # warm
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        ne = max(3, min(args.steps, 10))
        for _ in range(ne):
            out = run_step(rp, cfg, Ah, plan)
        te = max_over_ranks((time.perf_counter() - t0) / ne, ws, dev)
        d2h = sum(o.numel() * o.element_size() for o in out)
        e2e = {"value": te, "unit": "s", "h2d_bytes_per_step": int(sum_over_ranks(abytes, ws, dev)),
               "d2h_bytes_per_step": int(sum_over_ranks(d2h, ws, dev)),
               "note": "host-pinned A (shard) copied H2D and the factors copied D2H inside each library call"
                       + ("" if isinstance(A, torch.Tensor) else "; CSR(A^T) rebuilt on the device per call")
                       + "; host wall clock, max over ranks"}
        del Ah

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, host_of(A), args.cpu_seconds)

    if rank == 0:
        line = {"metric": "rank-k PCA wall time (s)", "value": t_step, "unit": "s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
                "higher_is_better": False, "scaling": plan["scaling"], "vs_baseline": None,
                "dtype": "f64" if A.dtype == torch.float64 else "f32",
                "a_bytes": abytes, "data": "synthetic", "config": conf,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "kernels": breakdown,
                "kernels_note": "per-launch CUDA events in a second, untimed run of the same steps",
                "roofline_time_s": abytes * passes / (hbm * 1e9)}
        if ws > 1:
            line["a_bytes_total"] = a_total
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
