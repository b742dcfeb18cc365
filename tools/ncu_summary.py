"""Print key metrics per kernel from an ncu report (details page)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Registers Per Thread', 'Executed Ipc Active',
        'Issue Slots Busy', 'L1/TEX Cache Throughput', 'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size']
ki, mi, vi, ui, idi = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
cur = None
for row in r[1:]:
    if row[mi] in want:
        if row[idi] != cur:
            cur = row[idi]
            print(f"--- [{cur}] {row[ki][:90]}")
        print(f"    {row[mi]:36s} {row[vi]:>12s} {row[ui]}")
