"""C5 20-step solve: CUDA-event time and per-kernel-class shares (fftpde profiling)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I
N = 32768
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c5, _, _, _ = I.c5_field_torch(N, dtype=torch.complex128)
p = F.Plan(N, N, dtype=torch.complex128)
a = torch.empty_like(c5)
for _ in range(2):
    p.diffuse(c5, 1e-4, 0.01, steps, out=a)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); p.diffuse(c5, 1e-4, 0.01, steps, out=a); e.record(); torch.cuda.synchronize()
    ts.append(round(s.elapsed_time(e), 2))
p.read_profile(); p.set_profiling(True)
p.diffuse(c5, 1e-4, 0.01, steps, out=a); torch.cuda.synchronize()
prof = p.read_profile(); p.set_profiling(False)
tot = sum(v[0] for v in prof.values())
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("FFTPDE")}, "steps": steps,
                  "ms_per_solve": ts,
                  "share_ms_per_step": {k: round(v[0] / tot * min(ts) / steps, 3) for k, v in prof.items() if v[1]},
                  "launches": {k: v[1] for k, v in prof.items() if v[1]}}), flush=True)
