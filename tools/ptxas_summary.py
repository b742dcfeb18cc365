"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spill bytes, smem."""
import re
import subprocess
import sys

def demangle(n):
    try:
        return subprocess.run(["c++filt"], input=n, capture_output=True, text=True).stdout.strip()
    except Exception:
        return n

cur = None
rows = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = {"name": demangle(m.group(1))}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
for r in rows:
    name = re.sub(r"fftpde::|\(.*", "", r["name"])
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', 0):>6}  {name}")
