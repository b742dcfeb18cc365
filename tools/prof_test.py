import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2412_12308_b200 import fftpde as F
p = F.Plan(1024, 1024)
x = torch.randn(1024, 1024, dtype=torch.complex128, device="cuda"); o = torch.empty_like(x)
p.diffuse(x, 1e-3, 0.01, 20, out=o); torch.cuda.synchronize()
p.read_profile(); p.set_profiling(True)
for _ in range(3): p.diffuse(x, 1e-3, 0.01, 20, out=o)
torch.cuda.synchronize(); print(p.read_profile()); p.set_profiling(False)
