"""Round-2 check of the four-step passes (fourstep.cuh) on the C5 grid:
separable-input parity against the fp64 oracle, agreement with the round-1
row2d/col2 path, and CUDA-event times of both paths."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I
from oracle import oracle as O

N = 32768
D, dt = 1e-4, 0.01
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = np.random.default_rng(7)
f = rng.standard_normal(N) + 1j * rng.standard_normal(N)
g = rng.standard_normal(N) + 1j * rng.standard_normal(N)
O.set_threads(os.cpu_count() or 1)
t0 = time.time()
Df = O.diffuse(f.reshape(1, N), D, dt, steps).ravel()
Dg = O.diffuse(g.reshape(1, N), D, dt, steps).ravel()
print("oracle 1D", time.time() - t0, flush=True)
fd = torch.from_numpy(f).cuda(); gd = torch.from_numpy(g).cuda()
u0 = torch.outer(gd, fd)                       # u0[y][x] = g[y] f[x]
ref = torch.outer(torch.from_numpy(Dg).cuda(), torch.from_numpy(Df).cuda())
p = F.Plan(N, N, dtype=torch.complex128)
out = p.diffuse(u0, D, dt, steps)
torch.cuda.synchronize()
err = (torch.linalg.vector_norm(out - ref) / torch.linalg.vector_norm(ref)).item()
print(json.dumps({"separable_parity_rel_l2": err, "steps": steps}), flush=True)
del ref, out, u0
# agreement with the round-1 passes on the C5 recipe field
c5, _, _, _ = I.c5_field_torch(N, dtype=torch.complex128)
a = p.diffuse(c5, D, dt, steps)
os.environ["FFTPDE_NO_FOURSTEP"] = "1"
q = F.Plan(N, N, dtype=torch.complex128)
del os.environ["FFTPDE_NO_FOURSTEP"]
b = q.diffuse(c5, D, dt, steps)
torch.cuda.synchronize()
print(json.dumps({"fourstep_vs_r01_rel_l2": (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b)).item()}), flush=True)
del b
def timeit(plan, n=3):
    for _ in range(2):
        plan.diffuse(c5, D, dt, 20, out=a)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); plan.diffuse(c5, D, dt, 20, out=a); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return ts
print(json.dumps({"fourstep_ms_per_20_steps": timeit(p)}), flush=True)
del p
print(json.dumps({"r01_ms_per_20_steps": timeit(q)}), flush=True)
