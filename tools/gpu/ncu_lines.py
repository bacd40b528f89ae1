"""Per-source-line stall-sample shares of one kernel in an ncu report:
   python tools/gpu/ncu_lines.py REPORT [kernel-index] [top-N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
idx = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", idx, "--launch-count", "1"], capture_output=True, text=True).stdout
res, f = [], ""
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            res.append((int(r[4] or 0), f, r[0], int(r[7] or 0), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
print("samples", tot, "instructions", sum(x[3] for x in res))
for s, f, l, ie, src in sorted(res, reverse=True)[:top]:
    print(f"{f}:{l}".ljust(18), f"{100 * s / tot:5.1f}%", str(ie).rjust(11), src)
