"""Distributed four-step (R28) in single-process loopback: P virtual ranks on one
B200, every rank's passes in turn, the all-to-all as device copies.  Prints the
solve time and the per-class kernel time (CUDA events inside the library), from
which the per-rank compute of a real P-GPU run is (class time) / P."""
import json
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_12308_b200 import fftpde as F

n, D, dt, steps = 32768, 1e-4, 0.01, 20
u0 = torch.randn(n, n, dtype=torch.complex128, device="cuda")
out = torch.empty_like(u0)
for P in [int(a) for a in sys.argv[1:]] or [2, 8]:
    p = F.ShardedPlan(n, n, dtype=torch.complex128, loopback=P if P > 1 else 0)
    p.diffuse(u0, D, dt, steps, out=out)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.diffuse(u0, D, dt, steps, out=out)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    p.read_profile()
    p.set_profiling(True)
    p.diffuse(u0, D, dt, steps, out=out)
    torch.cuda.synchronize()
    prof = p.read_profile()
    p.set_profiling(False)
    kern = sum(v[0] for v in prof.values())
    print(json.dumps({"P": P, "solve_ms": sorted(times)[1], "kernel_ms_by_class": prof,
                      "kernel_ms": kern, "per_rank_kernel_ms": kern / P}))
    del p
    torch.cuda.empty_cache()

# the fused variant (sharded.FusedFourStepSolver: the exchange in the B-pass epilogues)
from paper_2412_12308_b200 import sharded as S
plan = F.Plan(n, n, dtype=torch.complex128)
for P in [int(a) for a in sys.argv[1:]] or [2, 8]:
    solver = S.FusedFourStepSolver(n, S.LoopbackPeerComm(P), plan)
    R = n // P
    slabs = [u0[r * R:(r + 1) * R] for r in range(P)]
    outs = [out[r * R:(r + 1) * R] for r in range(P)]
    solver.diffuse(slabs, D, dt, steps, outs=outs)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        solver.diffuse(slabs, D, dt, steps, outs=outs)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    plan.read_profile()
    plan.set_profiling(True)
    solver.diffuse(slabs, D, dt, steps, outs=outs)
    torch.cuda.synchronize()
    prof = plan.read_profile()
    plan.set_profiling(False)
    kern = sum(v[0] for v in prof.values())
    print(json.dumps({"fused": True, "P": P, "solve_ms": sorted(times)[1], "kernel_ms_by_class": prof,
                      "kernel_ms": kern, "per_rank_kernel_ms": kern / P}))
    del solver
    torch.cuda.empty_cache()
