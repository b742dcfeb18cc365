"""CUDA-event time of the C5 20-step diffusion solve (current plan settings)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I
N = 32768
c5, _, _, _ = I.c5_field_torch(N, dtype=torch.complex128)
p = F.Plan(N, N, dtype=torch.complex128)
a = torch.empty_like(c5)
for _ in range(2):
    p.diffuse(c5, 1e-4, 0.01, 20, out=a)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); p.diffuse(c5, 1e-4, 0.01, 20, out=a); e.record(); torch.cuda.synchronize()
    ts.append(round(s.elapsed_time(e), 1))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("FFTPDE")}, "ms_per_20_steps": ts}), flush=True)
