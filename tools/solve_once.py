"""One solve of a BASELINE workload on cuda:0 (the unit ncu captures for tools/kernel_counts.py).
usage: python tools/solve_once.py c5 [warmup_solves]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I
wl = I.WORKLOADS[sys.argv[1]]
dtype = {"c128": torch.complex128, "c64": torch.complex64}[wl.dtype]
dev_in, host, _ = bench.make_device_inputs(wl, dtype)
out = [torch.empty_like(d) for d in dev_in]
p = F.Plan(wl.nx, wl.ny, batch=wl.batch, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 0):
    bench.reset_wave(wl, dev_in, out); bench.run_solve(p, wl, dev_in, out)
bench.reset_wave(wl, dev_in, out)
bench.run_solve(p, wl, dev_in, out)
torch.cuda.synchronize()
print("launches", p.launches)
