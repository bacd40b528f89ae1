"""Key metrics + stall mix of every kernel in an ncu report: python ncu_summary.py REP.ncu-rep"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
keys = ["launch__grid_size", "launch__block_size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread"]
for row in r[2:]:
    d = dict(zip(h, row))
    print("====", d["Kernel Name"][:90])
    for k in keys:
        if k in d:
            print(f"  {k:75s} {d[k]}")
    items = [(k, v) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    items = [(k, float(v.replace(",", ""))) for k, v in items if v.replace(",", "").replace(".", "").isdigit()]
    tot = sum(v for _, v in items) or 1
    print("  stalls:", ", ".join(f"{k[33:]} {100 * v / tot:.1f}%" for k, v in sorted(items, key=lambda x: -x[1])[:7]))
