"""Measured parity of every BASELINE config against the fp64 oracle:
prints one JSON line; run once per library build (FFTPDE_TWPOW=0 / 1)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I

O.set_threads(os.cpu_count() or 1)
C128 = torch.complex128


def rel(a, b):
    a = np.asarray(a, np.complex128).ravel(); b = np.asarray(b, np.complex128).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def noise(shape, seed):
    return I.white_noise(shape, seed)


out = {"build": os.environ.get("TAG", "")}
t0 = time.time()
# C1
d = I.c1_inputs(64)
p = F.Plan(64, 64, dtype=C128)
out["c1"] = rel(p.poisson(torch.from_numpy(d.rho).cuda()).cpu().numpy(), O.poisson(d.rho))
# C2 full stepped
g = I.c2_inputs(1024)
p = F.Plan(1024, 1024, dtype=C128)
u = p.diffuse(torch.from_numpy(g.u0).cuda(), 1e-3, 0.01, 200).cpu().numpy()
out["c2_stepped"] = rel(u, O.diffuse(g.u0, 1e-3, 0.01, 200))
# C3: 50-step prefix at 4096^2 with the workload's dt, and the full run vs collapsed
w = I.c3_inputs(4096)
p = F.Plan(4096, 4096, dtype=C128)
uu, vv = torch.from_numpy(w.u).cuda(), torch.from_numpy(w.ut).cuda()
p.wave_step(uu, vv, 1.0, 1e-4, 50)
uo, vo = O.wave(w.u, w.ut, 1.0, 1e-4, 50)
out["c3_prefix50_u"], out["c3_prefix50_ut"] = rel(uu.cpu().numpy(), uo), rel(vv.cpu().numpy(), vo)
uu, vv = torch.from_numpy(w.u).cuda(), torch.from_numpy(w.ut).cuda()
p.wave_step(uu, vv, 1.0, 1e-4, 500)
uo, vo = O.wave(w.u, w.ut, 1.0, 1e-4, 500, collapsed=True)
out["c3_full_vs_collapsed_u"], out["c3_full_vs_collapsed_ut"] = rel(uu.cpu().numpy(), uo), rel(vv.cpu().numpy(), vo)
# oracle's own spread: stepped vs collapsed for the 50-step prefix
uo2, vo2 = O.wave(w.u, w.ut, 1.0, 1e-4, 50, collapsed=True)
uo1, vo1 = O.wave(w.u, w.ut, 1.0, 1e-4, 50)
out["c3_oracle_stepped_vs_collapsed50_u"], out["c3_oracle_stepped_vs_collapsed50_ut"] = rel(uo1, uo2), rel(vo1, vo2)
del w, uu, vv
# C4: all 256 grids
s = I.c4_inputs(512, 256)
p = F.Plan(512, 512, batch=256, dtype=torch.complex64)
uc = p.poisson(torch.from_numpy(s.astype(np.complex64)).cuda()).cpu().numpy()
errs = [rel(uc[k], O.poisson(s[k].astype(np.complex64).astype(np.complex128))) for k in range(256)]
out["c4_max_over_256"], out["c4_mean"] = max(errs), float(np.mean(errs))
# long-axis wave u_t (the round-1 10x tolerance) and the small reversal case (4x / 10x)
for (ny, nx) in [(32768, 16), (16, 32768), (16384, 32), (8, 16384)]:
    x = noise((ny, nx), 77 + nx); y = noise((ny, nx), 78)
    pp = F.Plan(nx, ny, Lx=1.0, Ly=2.0)
    a, b = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    pp.wave_step(a, b, 0.3, 1e-4, 2)
    ua, va = O.wave(x, y, 0.3, 1e-4, 2, 1.0, 2.0)
    out[f"wave_{ny}x{nx}_u"], out[f"wave_{ny}x{nx}_ut"] = rel(a.cpu().numpy(), ua), rel(b.cpu().numpy(), va)
u0, v0 = noise((2, 128, 64), 21), noise((2, 128, 64), 22)
pp = F.Plan(64, 128, batch=2, Lx=1.3, Ly=0.9)
a, b = torch.from_numpy(u0).cuda(), torch.from_numpy(v0).cuda()
pp.wave_step(a, b, 0.7, 3e-3, 9)
uo, vo = O.wave(u0, v0, 0.7, 3e-3, 9, 1.3, 0.9)
uo1, vo1 = O.wave(u0, v0, 0.7, 3e-3, 9, 1.3, 0.9, path=1)
out["rev_u"], out["rev_ut"] = rel(a.cpu().numpy(), uo), rel(b.cpu().numpy(), vo)
out["rev_oracle_path1_vs_path2_u"], out["rev_oracle_path1_vs_path2_ut"] = rel(uo1, uo), rel(vo1, vo)
pp.wave_step(a, b, 0.7, -3e-3, 9)
out["rev_back_u"] = rel(a.cpu().numpy(), u0)
ub, vb = O.wave(uo, vo, 0.7, -3e-3, 9, 1.3, 0.9)
out["rev_back_oracle_u"] = rel(ub, u0)
out["seconds"] = round(time.time() - t0, 1)
print(json.dumps(out), flush=True)
