"""Run one workload a few times for ncu capture (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F, inputs as I
case = sys.argv[1]
if case == "poisson4096":
    p = F.Plan(4096, 4096); x = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda"); o = torch.empty_like(x)
    for _ in range(3): p.poisson(x, out=o)
elif case == "wave4096":
    p = F.Plan(4096, 4096); u = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda"); v = torch.zeros_like(u)
    p.wave_step(u, v, 1.0, 1e-4, 3)
elif case == "c4":
    p = F.Plan(512, 512, batch=256, dtype=torch.complex64); x = torch.randn(256, 512, 512, dtype=torch.complex64, device="cuda"); o = torch.empty_like(x)
    for _ in range(3): p.poisson(x, out=o)
elif case == "c2":
    p = F.Plan(1024, 1024); x = torch.randn(1024, 1024, dtype=torch.complex128, device="cuda"); o = torch.empty_like(x)
    p.diffuse(x, 1e-3, 0.01, 10, out=o)
torch.cuda.synchronize()
print("ok", case)
