import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_12308_b200 import fftpde as F
for nx, ny in [(16384, 32), (32768, 16), (16384, 64)]:
    p = F.Plan(nx, ny)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.complex(torch.randn(ny, nx, generator=g, device="cuda", dtype=torch.float64),
                      torch.randn(ny, nx, generator=g, device="cuda", dtype=torch.float64))
    for name, fn in [("fwd", lambda: p.forward(x)), ("inv", lambda: p.inverse(x)),
                     ("dif", lambda: p.diffuse(x, 1e-4, 0.01, 3))]:
        ref = fn(); bad = 0; mx = 0.0
        for _ in range(20):
            o = fn()
            if not torch.equal(o, ref):
                bad += 1; d = (o - ref).abs()
                mx = max(mx, float(d.max()))
                rows = torch.nonzero(d.amax(dim=1) > 0).flatten().tolist()
        print(nx, ny, name, "mismatching runs", bad, "max diff", mx, "rows", rows[:10] if bad else [], flush=True)
