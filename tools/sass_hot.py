"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"] +
                     (["-k", kfilter] if kfilter else []), capture_output=True, text=True).stdout
lines = out.splitlines()
# the csv may contain several kernels; take the first block
rows = list(csv.reader(lines))
h = rows[1]
data = []
for r in rows[2:]:
    if len(r) != len(h):
        break
    data.append(r)
si = h.index('Warp Stall Sampling (All Samples)'); src = h.index('Source'); ad = h.index('Address')
tot = sum(float(r[si] or 0) for r in data)
cols = [c for c in h if c.startswith('stall_') and '(Not Issued)' not in c]
ix = [h.index(c) for c in cols]
agg = {}
for r in data:
    op = r[src].split()[0] if r[src].split() else ''
    if op.startswith('@'):
        op = r[src].split()[1]
    op = op.split('.')[0]
    agg[op] = agg.get(op, 0) + float(r[si] or 0)
print("total samples", tot, " by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:14]))
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    print(f"{r[ad][-5:]:>5} {100*float(r[si])/tot:5.1f}% {r[src][:58]:58s}", " ".join(f"{c[6:]}={r[i]}" for c, i in zip(cols, ix) if r[i] not in ('0', '')))
