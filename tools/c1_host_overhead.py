"""Host-side cost of one C1 solve: the Python API call, the raw C-ABI call, an event record."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, ctypes
from paper_2412_12308_b200 import fftpde as F, inputs as I
d = I.c1_inputs(64)
p = F.Plan(64, 64)
x = torch.from_numpy(d.rho).cuda(); o = torch.empty_like(x)
for _ in range(100): p.poisson(x, out=o)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N): p.poisson(x, out=o)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("python API per call (host) %.2f us; with drain %.2f us" % ((t1 - t0) / N * 1e6, (t2 - t0) / N * 1e6))
lib = p.lib; h = p._h; xp = x.data_ptr(); op = o.data_ptr()
t0 = time.perf_counter()
for _ in range(N): lib.fftpde_poisson_batched(h, xp, op, 1, 4096)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("raw ctypes C-ABI call (host) %.2f us; with drain %.2f us" % ((t1 - t0) / N * 1e6, (t2 - t0) / N * 1e6))
s = torch.cuda.current_stream(); ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
t0 = time.perf_counter()
for _ in range(N): ev[0].record(s)
t1 = time.perf_counter()
print("event record %.2f us" % ((t1 - t0) / N * 1e6))
