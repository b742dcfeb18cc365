"""Cost of the 1024-point line passes at C5 scale: a batch of 1024 grids of
1024 x 1024 complex128 (2^30 points, 16 GiB) diffused with the round-1 row and
column line kernels (one row pass + one column pass per step)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F
B = 1024
x = torch.randn(B, 1024, 1024, dtype=torch.complex128, device="cuda")
p = F.Plan(1024, 1024, batch=B, dtype=torch.complex128)
out = torch.empty_like(x)
for _ in range(2):
    p.diffuse(x, 1e-3, 0.01, 2, out=out)
torch.cuda.synchronize()
p.read_profile(); p.set_profiling(True)
p.diffuse(x, 1e-3, 0.01, 4, out=out)
torch.cuda.synchronize()
prof = p.read_profile(); p.set_profiling(False)
ts = []
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); p.diffuse(x, 1e-3, 0.01, 4, out=out); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) / 4)
print(json.dumps({"ms_per_step": ts, "profile_ms_per_step": {k: v[0] / 4 for k, v in prof.items()},
                  "field_GiB": 16}))
