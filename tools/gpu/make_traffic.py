"""profiles/traffic.json from ncu --set full captures: per kernel of each config,
dram bytes read+write per launch, duration, SM clock and key pipe metrics.
usage: python tools/gpu/make_traffic.py OUT.json CFG=REP.ncu-rep ..."""
import csv, io, json, re, subprocess, sys

out = {}
try:
    out = json.load(open(sys.argv[1]))
except Exception:
    pass
for arg in sys.argv[2:]:
    cfg, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        name = re.sub(r"\(.*", "", d["Kernel Name"]).split("::")[-1].replace("void ", "")

        def val(k, scale_to=None):
            v = float(d[k].replace(",", ""))
            unit = u.get(k, "")
            mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12,
                    "ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9,
                    "GHz": 1e9, "MHz": 1e6, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}.get(unit, 1.0)
            return v * mult
        rec = {"duration_s": val("gpu__time_duration.sum"),
               "dram_read_bytes": val("dram__bytes_read.sum"), "dram_write_bytes": val("dram__bytes_write.sum"),
               "sm_clock_hz": val("smsp__cycles_elapsed.avg.per_second") if "smsp__cycles_elapsed.avg.per_second" in d else None,
               "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
               "regs": d.get("launch__registers_per_thread"), "source": rep}
        for k in ["sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                  "lts__t_sector_hit_rate.pct"]:
            if k in d:
                try:
                    rec[k] = float(d[k].replace(",", ""))
                except ValueError:
                    pass
        rec["traffic_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        out.setdefault(cfg, {}).setdefault(name, []).append(rec)
json.dump(out, open(sys.argv[1], "w"), indent=1)
for cfg, ks in out.items():
    for k, recs in ks.items():
        for rec in recs:
            print(f"{cfg} {k:28s} {rec['duration_s']*1e3:8.3f} ms  R {rec['dram_read_bytes']/1e9:8.3f} GB  W {rec['dram_write_bytes']/1e9:7.3f} GB")
