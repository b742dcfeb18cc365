"""Small invocations of every kernel family for compute-sanitizer (one tool per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F

torch.manual_seed(0)
def rnd(*s, dt=torch.complex128):
    return torch.randn(*s, dtype=dt, device="cuda")
# row2d (16384-point rows: FWD, INV and MID through diffuse) + col pass
p = F.Plan(16384, 16); x = rnd(16, 16384)
y = p.forward(x); z = p.inverse(y); p.diffuse(x, 1e-4, 0.01, 3)
# two-level cluster column pass (ny = 2048), poisson / diffuse / wave
q = F.Plan(16, 2048); a = rnd(2048, 16)
q.poisson(a); q.diffuse(a, 1e-3, 0.01, 2); u, v = a.clone(), a.clone(); q.wave_step(u, v, 1.0, 1e-3, 2)
# pipe passes (1024), small-grid solve, line kernel (c64 512 batch)
r = F.Plan(1024, 64); b = rnd(64, 1024); r.poisson(b); r.diffuse(b, 1e-3, 0.01, 2)
s = F.Plan(64, 64); s.poisson(rnd(64, 64))
t = F.Plan(512, 512, batch=4, dtype=torch.complex64); t.poisson(rnd(4, 512, 512, dt=torch.complex64))
# RK4 source path
w = F.Plan(64, 64, Lx=4.0, Ly=4.0); uu = torch.zeros(64, 64, dtype=torch.complex128, device="cuda")
w.wave_rk4(uu, torch.zeros_like(uu), 1 / 64, 3, xmin=-2.0, ymin=-2.0)
torch.cuda.synchronize()
print("sanitize case ok")
