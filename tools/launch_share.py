"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, mean duration and share of the total."""
import csv, sys, re, collections
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("fftpde::", "")
    v = float(r[vi].replace(",", ""))
    if r[ui] in ("ns", "nsecond"): v /= 1000.0
    elif r[ui] in ("ms", "msecond"): v *= 1000.0
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'mean us':>9s} {'total us':>10s} {'share':>6s}")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:70]:70s} {n:8d} {t/n:9.2f} {t:10.1f} {100*t/tot:5.1f}%")
print(f"{'total':70s} {sum(v[0] for v in agg.values()):8d} {'':9s} {tot:10.1f}")
