"""Per-kernel totals of the last bench step in an ncu --metrics gpu__time_duration.sum launch list."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ks = [(r[h.index("Kernel Name")], float(r[h.index("Metric Value")])) for r in rows[hi + 1:]]
start = [i for i, (k, v) in enumerate(ks) if "omega_kernel" in k][-1]
if start > 0 and "row_exp_kernel" in ks[start - 1][0]:  # the emulated path's exponent read opens the step
    start -= 1
last = ks[start:]
agg = collections.OrderedDict()
for k, v in last:
    n = re.sub(r"\(.*", "", k).split("::")[-1]
    c, s = agg.get(n, (0, 0.0))
    agg[n] = (c + 1, s + v)
tot = sum(v for _, v in last)
print(f"last step: {len(last)} launches, {tot / 1e3:.1f} us (serialised, cold)")
for n, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {n:40s} {c:4d} {s / 1e3:10.1f} us {100 * s / tot:5.1f}%")
