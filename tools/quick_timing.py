"""Quick CUDA-event timing of the five workloads (development aid, not bench.py)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_12308_b200 import fftpde as F, inputs as I

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)

hbm = 6538.3e9
# C1
d = I.c1_inputs(64); p = F.Plan(64, 64); x = torch.from_numpy(d.rho).cuda(); o = torch.empty_like(x)
t = timeit(lambda: p.poisson(x, out=o), 20); print(f"C1 poisson 64^2: {t*1e3:.1f} us")
# C2
g = I.c2_inputs(1024); p = F.Plan(1024, 1024); x = torch.from_numpy(g.u0).cuda(); o = torch.empty_like(x)
t = timeit(lambda: p.diffuse(x, 1e-3, 0.01, 200, out=o)); print(f"C2 diffusion 1024^2 x200: {t:.3f} ms  {1024*1024*200/t/1e-3:.3e} pts/s  {t/200*1e3:.1f} us/step  alg {32*2**20*200/(t*1e-3)/1e9:.0f} GB/s")
# C3
w = I.c3_inputs(4096, noise=1e-3); p = F.Plan(4096, 4096); u = torch.from_numpy(w.u).cuda(); v = torch.from_numpy(w.ut).cuda()
for n in (10,):
    t = timeit(lambda: p.wave_step(u, v, 1.0, 1e-4, n), 2); print(f"C3 wave 4096^2 x{n}: {t:.3f} ms  {t/n:.3f} ms/step  3-pass HBM {3*64*4096*4096/(t/n*1e-3)/1e9:.0f} GB/s  alg {64*4096*4096/(t/n*1e-3)/1e9:.0f} GB/s")
# C4
s = I.c4_inputs(512, 256); p = F.Plan(512, 512, batch=256, dtype=torch.complex64); x = torch.from_numpy(s).cuda(); o = torch.empty_like(x)
t = timeit(lambda: p.poisson(x, out=o), 5); print(f"C4 batched poisson: {t:.3f} ms  {256*512*512/(t*1e-3):.3e} pts/s  3-pass {3*16*256*512*512/(t*1e-3)/1e9:.0f} GB/s")
# individual passes on C3-size field
p = F.Plan(4096, 4096); a = torch.from_numpy(w.u).cuda(); b = torch.empty_like(a)
t = timeit(lambda: p.forward(a, out=b), 5); print(f"fwd 4096^2 c128 (2 passes): {t:.3f} ms  {2*2*16*4096*4096/(t*1e-3)/1e9:.0f} GB/s")
t = timeit(lambda: p.poisson(a, out=b), 5); print(f"poisson 4096^2 c128 (3 passes): {t:.3f} ms  {3*2*16*4096*4096/(t*1e-3)/1e9:.0f} GB/s")
