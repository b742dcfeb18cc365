"""Warp-stall samples of one kernel aggregated per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep object.o kernel-substring [top]
Maps the report's SASS addresses (relative to the function start) to source
lines with nvdisasm --print-line-info on the cubin inside the object file."""
import csv, collections, os, re, subprocess, sys, tempfile
rep, obj, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, hdr, name = [], None, None
for row in csv.reader(out.splitlines()):
    if row and row[0] == "Kernel Name":
        name = row[1]; hdr = None; continue
    if row and row[0] == "Address":
        hdr = row; continue
    if hdr and name and ksub in name:
        rows.append(row)
si = hdr.index("Warp Stall Sampling (All Samples)")
base = int(rows[0][0], 16)
samples = {int(r[0], 16) - base: int(r[si] or 0) for r in rows}
sass = {int(r[0], 16) - base: r[1].strip() for r in rows}
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", "-fun", "", os.path.join(d, cubin)],
                     capture_output=True, text=True).stdout
# find the function whose name contains ksub's mangled pieces: use the first function with matching size
funcs, cur, line = {}, None, None
for l in dis.splitlines():
    m = re.match(r'\s*\.text\.(\S+):', l) or re.match(r'^(\S+):\s*$', l)
    if l.strip().startswith(".text.") and l.strip().endswith(":"):
        cur = l.strip()[6:-1]; funcs[cur] = {}; continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and cur is not None:
        funcs[cur][int(m.group(1), 16)] = line
key = [f for f in funcs if "rowt" in f or ksub in f]
fmap = funcs[key[0]] if key else {}
agg = collections.Counter()
tot = sum(samples.values())
for off, s in samples.items():
    agg[fmap.get(off, ("?", 0))] += s
print(f"{name[:100]}\ntotal samples {tot}")
for (f, ln), s in agg.most_common(top):
    print(f"{100.0*s/tot:6.1f}%  {f}:{ln}")
