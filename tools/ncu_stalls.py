"""Per-instruction warp-stall attribution from an ncu report (source page, SASS).
usage: python tools/ncu_stalls.py report.ncu-rep [kernel-substring] [top]"""
import csv, subprocess, sys, re, collections
rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for row in csv.reader(lines):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]; blocks.append(cur); continue
    if row and row[0] == "Address":
        cur[1] = row; continue
    if cur and cur[1]:
        cur[2].append(row)
for name, hdr, rows in blocks:
    if ksub not in name:
        continue
    h = {k: i for i, k in enumerate(hdr)}
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(float(r[h["Warp Stall Sampling (All Samples)"]] or 0) for r in rows)
    print("=" * 100); print(name[:150]); print(f"total samples {tot:.0f}")
    byop = collections.Counter(); byst = collections.Counter()
    for r in rows:
        s = float(r[h["Warp Stall Sampling (All Samples)"]] or 0)
        op = r[h["Source"]].split()[0] if r[h["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[h["Source"]].split()[1]
        byop[op.split(".")[0]] += s
        for c in stall_cols:
            byst[c] += float(r[h[c]] or 0)
    print("by opcode:", ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in byop.most_common(10)))
    print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.0f}%" for k, v in byst.most_common(8)))
    rs = sorted(rows, key=lambda r: -float(r[h["Warp Stall Sampling (All Samples)"]] or 0))[:top]
    for r in rs:
        s = float(r[h["Warp Stall Sampling (All Samples)"]] or 0)
        reasons = sorted(((float(r[h[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"  {100*s/tot:5.1f}%  {r[h['Address']][-5:]}  {r[h['Source']].strip()[:60]:60s} " +
              " ".join(f"{n}:{100*v/tot:.1f}" for v, n in reasons if v))
