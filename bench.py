"""bench.py -- timed run of the 2D FFT-PDE hot path (arXiv 2412.12308) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl reference]

A *step* is one pass of the whole hot path over one batch of synthetic input
(SURVEY.md 8(a) a1-a5): for the default workload c2 (BASELINE.json configs[1])
that is one ``fftpde_diffuse`` call of 200 exact diffusion steps on a
1024 x 1024 complex128 grid (each step a forward 2D FFT, the k-space
multiply and an inverse 2D FFT, 3 kernel launches).  The metric is grid-points
per second (nx*ny*batch*nsteps / time) for the whole job; rank 0 prints one
JSON line.

Timing: W untimed warm-up steps, then exactly K steps, each bracketed by CUDA
events on the plan's stream; L2 (126 MB) is flushed with a 256 MiB write
between timed steps (outside the events).  Barrier + synchronize on both sides
of the timed region; the per-rank device time is reduced with MAX over ranks.
Multi-GPU (torchrun, one process per GPU): c1-c4 fit one GPU, so N > 1 runs N
independent replicas (weak scaling, no collective on the data path).

Extra keys: ``e2e`` (the same metric through the public API with host buffers:
pinned host -> device copy, solve, device -> host copy, every step),
``roofline`` (dominant kernel class, algorithmic bytes / its CUDA-event time vs
MEASURED_PEAKS.json hbm_gbs), ``cpu_baseline`` (the fp64 oracle on this host's
cores, bounded sample; rank 0, N = 1), ``clocks`` (nvidia-smi sampled during
the timed region), ``gpu_launches`` (library kernels in the timed region).

``--impl reference`` times the CPU oracle (the reference arm of this tier) on
the same workload, metric and unit, each step a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2D FFT-PDE solve grid-points/sec and achieved HBM GB/s vs peak (1/2/4/8 GPU)"
UNIT = "grid-points/s"
L2_FLUSH_BYTES = 256 << 20

THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "rk4", "rk4big", "dsrc", "p3d", "d3d",
                             "c2r", "c3r", "c4r"],
                    help="c1-c5: BASELINE.json configs[0..4]; rk4/rk4big: the paper's orbiting-source "
                         "RK4 run (SURVEY.md 8(f) row 1, not a BASELINE config)")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="c5: use the slab-decomposed path even on one GPU (P = 1 process group)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer", "lib", "fused"],
                    help="sharded c5: pack + NCCL all-to-all, or direct peer stores into torch "
                         "symmetric memory (fftpde_peer_transpose, SURVEY.md 8(e) N10)")
    return ap.parse_args()


# ---------------------------------------------------------------------------- inputs

def make_inputs(wl):
    """Seeded synthetic input of the workload (numpy, host) -- paper_2412_12308_b200.inputs."""
    import numpy as np
    from paper_2412_12308_b200 import inputs as I
    if wl.dtype in ("f64", "f32"):          # real storage of the complex recipes (R12)
        base = {"c2r": "c2", "c3r": "c3", "c4r": "c4"}[wl.name[:3]]
        rt = np.float64 if wl.dtype == "f64" else np.float32
        return tuple(np.ascontiguousarray(h.real).astype(rt) for h in make_inputs(I.WORKLOADS[base]))
    if wl.name.startswith("c1"):
        return (I.c1_inputs(wl.nx).rho,)
    if wl.name.startswith("c2"):
        return (I.c2_inputs(wl.nx).u0,)
    if wl.name.startswith("c3"):
        w = I.c3_inputs(wl.nx)
        return (w.u, w.ut)
    if wl.name.startswith("c4"):
        return (I.c4_inputs(wl.nx, wl.batch).astype(np.complex64),)
    if wl.nz > 1:                           # 3D workloads: seeded Gaussians on [0,1)^3
        return (I.gaussians_3d(wl.nx),)
    if wl.op == "dsrc":                     # C2 Gaussians as initial field and as the static source
        g = I.c2_inputs(wl.nx).u0
        return (g, np.ascontiguousarray(0.5 * g))
    if wl.op == "rk4":                      # from rest (R19)
        z = np.zeros((wl.ny, wl.nx), np.complex128)
        return (z, z.copy())
    raise ValueError(wl.name)


def make_device_inputs(wl, dtype):
    """Device tensors of the workload input (C5's 16 GiB field is built on the device)."""
    import numpy as np
    import torch
    from paper_2412_12308_b200 import inputs as I
    if wl.name.startswith("c5"):
        f, _, _, _ = I.c5_field_torch(wl.nx, dtype=dtype)
        return [f], None
    host = make_inputs(wl)
    return [torch.from_numpy(np.ascontiguousarray(h)).to(dtype).cuda() for h in host], host


def alg_bytes_per_launch(wl, kernel_class):
    """Algorithmic HBM bytes of one launch, averaged over the launches of a
    solve: every field the pass touches is read once and written once
    (SURVEY.md 8(d)); in a multi-step solve the row passes between column
    passes are MID passes (inverse rows of step s stored as the physical field
    + forward rows of step s+1: one read, two writes), the first and last are
    plain forward / inverse rows (one read, one write)."""
    esz = {"c128": 16, "c64": 8, "f64": 8, "f32": 4}[wl.dtype]
    field = wl.nx * wl.ny * wl.nz * wl.batch * esz      # real fields: the half spectrum has ~ the same bytes
    if kernel_class == "wave_col_pass":
        return 2 * 2 * field
    if wl.op == "dsrc":
        # per step: forward (rows, columns), u^ <- E u^ + Phi s^ (u^, s^ in, u^ out), inverse
        return 3 * field if kernel_class == "pointwise" else 2 * field
    if wl.op == "rk4":
        # per step: 2 source samplings (1 write each) and the RK4 kernel (u^, v^, 3 source
        # spectra read, u^, v^ written); the transforms are plain forward passes
        return 3 * field if kernel_class == "pointwise" else 2 * field
    # the complex 2D diffusion is separable: each step is one row pass (forward,
    # x factor, inverse) and one column pass, each reading and writing the field
    # once; the wave, the real-field and the 3D diffusion keep the MID row pass
    mid_rows = wl.op == "wave"
    if kernel_class == "row_pass" and mid_rows and wl.nsteps > 1:
        n = wl.nsteps                      # per field: 1 FWD + (n-1) MID + 1 INV launches
        return (2 * field * 2 + 3 * field * (n - 1)) / (n + 1)
    return 2 * field


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # wait for the first sample: nvidia-smi's NVML start-up (which takes driver
        # locks) must be over before the timed region starts
        t0 = time.perf_counter()
        while self.proc is not None and time.perf_counter() - t0 < 5.0:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.05)
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            for b, name in THROTTLE_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- dist

def dist_setup(n_gpus):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------- native arm

def run_solve(plan, wl, dev_in, out):
    """One step of the hot path on device buffers (the timed unit)."""
    if wl.op == "poisson":
        plan.poisson(dev_in[0], out=out[0])
    elif wl.op == "diffuse":
        plan.diffuse(dev_in[0], wl.D, wl.dt, wl.nsteps, out=out[0])
    elif wl.op == "rk4":
        plan.wave_rk4(out[0], out[1], wl.dt, wl.nsteps, c=wl.c, xmin=-0.5 * wl.Lx, ymin=-0.5 * wl.Ly)
    elif wl.op == "dsrc":
        plan.diffuse_source(dev_in[0], dev_in[1], wl.D, wl.dt, wl.nsteps, out=out[0])
    else:  # wave: advance a working copy (reset from the input outside the events)
        plan.wave_step(out[0], out[1], wl.c, wl.dt, wl.nsteps)


def reset_wave(wl, dev_in, out):
    if wl.op in ("wave", "rk4"):
        out[0].copy_(dev_in[0])
        out[1].copy_(dev_in[1])


def native(args, wl, world, rank, local):
    import numpy as np
    import torch
    from paper_2412_12308_b200 import fftpde as F

    dtype = {"c128": torch.complex128, "c64": torch.complex64, "f64": torch.float64,
             "f32": torch.float32}[wl.dtype]
    dev_in, host = make_device_inputs(wl, dtype)
    # C5 (16 GiB field): built on the device; the e2e leg copies it once into pinned
    # host memory (outside the timed region), the CPU baseline takes a bounded sample
    out = [torch.empty_like(d) for d in dev_in]
    if wl.dtype in ("f64", "f32"):
        plan = F.PlanR2C(wl.nx, wl.ny, batch=wl.batch, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
    elif wl.nz > 1:
        plan = F.Plan3D(wl.nx, wl.ny, wl.nz, dtype=dtype)
    else:
        plan = F.Plan(wl.nx, wl.ny, batch=wl.batch, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    # warm-up (also uploads the operator tables for this (D, dt) / (c, dt))
    for _ in range(args.warmup):
        reset_wave(wl, dev_in, out)
        run_solve(plan, wl, dev_in, out)
    torch.cuda.synchronize()

    # ---- timed region: K steps, events per step, L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = plan.launches
    gpu_index = torch.cuda.current_device()
    barrier(world)
    torch.cuda.synchronize()
    vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    smi_index = int(vis[gpu_index]) if len(vis) > gpu_index and vis[gpu_index].isdigit() else gpu_index
    with ClockSampler(smi_index) as clk:
        # one more untimed step right before the timed ones: the GPU idled while the
        # clock sampler started, and the first kernel after an idle period runs slow
        reset_wave(wl, dev_in, out)
        flush.zero_()
        run_solve(plan, wl, dev_in, out)
        launches0 = plan.launches            # count the timed steps' launches only
        for i in range(args.steps):
            reset_wave(wl, dev_in, out)
            flush.zero_()
            starts[i].record(stream)
            run_solve(plan, wl, dev_in, out)
            ends[i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = plan.launches - launches0
    ms_rank = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_total = max_over_ranks(world, ms_rank)
    ms_per_step = ms_total / args.steps
    pts_per_step = wl.points * (wl.nsteps if wl.op != "poisson" else 1)
    value = world * pts_per_step * args.steps / (ms_total * 1e-3)

    # ---- per-kernel timing (same calls, events around every launch)
    plan.read_profile()
    plan.set_profiling(True)
    for i in range(args.steps):
        reset_wave(wl, dev_in, out)
        flush.zero_()
        run_solve(plan, wl, dev_in, out)
    torch.cuda.synchronize()
    prof = plan.read_profile()
    plan.set_profiling(False)
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    total_prof = sum(v[0] for v in prof.values())
    # Event nodes between kernels slow a graph replay down (each costs about a
    # kernel boundary), so the profiled run fixes each kernel class's SHARE of
    # the step and the un-instrumented timed region fixes the step time:
    # dominant launch duration = share x (timed ms/step) / launches per step.
    share = dom_ms / total_prof if total_prof else 1.0
    dom_launches_per_step = dom_n / args.steps
    dom_avg_s = share * ms_per_step * 1e-3 / dom_launches_per_step
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg_bytes_per_launch(wl, dom_name) / dom_avg_s / 1e9
    traffic, pipe_pct = None, None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{wl.name}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(dom_name)
            pipe_pct = (tj.get("_pipe_pct") or {}).get(dom_name)
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": traffic,
        "kernel": dom_name, "launches_per_step": dom_n // args.steps,
        "avg_launch_us": round(dom_avg_s * 1e6, 2),
        "share_of_step": round(dom_ms / total_prof, 3) if total_prof else None,
        "alg_bytes_per_launch": alg_bytes_per_launch(wl, dom_name),
        # DRAM bytes per launch (ncu, caches flushed) / algorithmic bytes: the implied
        # number of field round trips relative to the one the method needs
        "traffic_over_alg": round(traffic / alg_bytes_per_launch(wl, dom_name), 3) if traffic else None,
        # FP64 / FP32-FMA pipe utilisation of the dominant class from the same ncu capture
        "pipe_active_pct": pipe_pct,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks
                       else "fallback 6650 GB/s (B200_PROFILING.md)",
        # every class's share of the profiled replays x the un-instrumented step time
        # (sums to ms_per_step); the raw event-instrumented times over-state short kernels
        "per_kernel_ms_per_step": {k: round(v[0] / total_prof * ms_per_step, 4) if total_prof else None
                                   for k, v in prof.items()},
        "per_kernel_event_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in prof.items()},
        "duration_method": "share of the step from CUDA-event-profiled replays x un-instrumented CUDA-event step time",
    }

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        if host is not None:
            host_in = [torch.from_numpy(np.ascontiguousarray(h)).to(dtype).pin_memory() for h in host]
        else:
            host_in = []
            for d in dev_in:
                h = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
                h.copy_(d)
                host_in.append(h)
        host_out = [torch.empty(h.shape, dtype=dtype, pin_memory=True) for h in host_in]

        def e2e_step():
            if wl.dtype in ("f64", "f32"):   # real plans take device tensors: copies in the timed region
                for d, h in zip(out, host_in):
                    d.copy_(h, non_blocking=True)
                if wl.op == "poisson":
                    r = plan.poisson(out[0])
                    host_out[0].copy_(r, non_blocking=True)
                elif wl.op == "diffuse":
                    r = plan.diffuse(out[0], wl.D, wl.dt, wl.nsteps)
                    host_out[0].copy_(r, non_blocking=True)
                else:
                    plan.wave_step(out[0], out[1], wl.c, wl.dt, wl.nsteps)
                    for h, d in zip(host_out, out):
                        h.copy_(d, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return
            if wl.op == "poisson":
                plan.poisson(host_in[0], out=host_out[0])
            elif wl.op == "diffuse":
                plan.diffuse(host_in[0], wl.D, wl.dt, wl.nsteps, out=host_out[0])
            elif wl.op == "dsrc":
                plan.diffuse_source(host_in[0], host_in[1], wl.D, wl.dt, wl.nsteps, out=host_out[0])
            elif wl.op == "rk4":            # in place on device copies of the host fields
                for d, h in zip(out, host_in):
                    d.copy_(h, non_blocking=True)
                plan.wave_rk4(out[0], out[1], wl.dt, wl.nsteps, c=wl.c, xmin=-0.5 * wl.Lx, ymin=-0.5 * wl.Ly)
                for h, d in zip(host_out, out):
                    h.copy_(d, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            else:
                plan.wave_step(host_in[0], host_in[1], wl.c, wl.dt, wl.nsteps)
        e2e_step()
        torch.cuda.synchronize()
        barrier(world)
        tot = 0.0
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()              # H2D, solve, D2H (synchronises on the result)
            torch.cuda.synchronize()
            tot += time.perf_counter() - t0
        barrier(world)
        tot = max_over_ranks(world, tot)
        nbytes = sum(h.numel() * h.element_size() for h in host_in)
        e2e = {"value": world * pts_per_step * args.steps / tot, "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "timer": "host perf_counter around the public-API call (pinned host buffers)"}

    # ---- CPU oracle baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, host if host is not None else None)

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if wl.dtype in ("c128", "f64") else "f32",
        "data": "synthetic (seeded, BASELINE.json recipe; paper_2412_12308_b200/inputs.py)",
        "config": workload_config(wl, world),
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
        "gpu_launches": launches,
        "hbm_gbs_alg": round(world * alg_step_bytes(wl) * args.steps / (ms_total * 1e-3) / 1e9, 1),
    }
    return line


class _LibSharded:
    """Adapter: a ShardedPlan with the SlabSolver-style call the sharded bench uses."""

    def __init__(self, plan):
        self.plan = plan

    @property
    def launches(self):
        return self.plan.launches

    def diffuse(self, slabs, D, dt, nsteps, outs):
        self.plan.diffuse(slabs[0], D, dt, nsteps, out=outs[0])
        return outs


def sharded_native(args, wl, world, rank, local):
    """C5 at N > 1: the slab decomposition, NCCL all-to-all between
    the libfftpde row and column-slab passes; strong scaling (fixed 32768^2 grid)."""
    import torch
    from paper_2412_12308_b200 import inputs as I
    from paper_2412_12308_b200 import sharded as S
    dtype = torch.complex128
    full, _, _, _ = I.c5_field_torch(wl.nx, dtype=dtype)
    lo, hi = S.slab_rows(wl.ny, world, rank)
    slab = full[lo:hi].contiguous()
    del full
    torch.cuda.empty_cache()
    if args.exchange == "lib":     # the whole slab solve inside the C ABI (fftpde_plan_2d_sharded)
        from paper_2412_12308_b200 import fftpde as F
        ops = _LibSharded(F.ShardedPlan(wl.nx, wl.ny, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly))
        solver = ops
    else:
        ops = S.CudaLocalOps(wl.nx, wl.ny, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
    if args.exchange == "peer":
        solver = S.PeerSlabSolver(wl.nx, wl.ny, S.SymmetricPeerComm(), ops)
    elif args.exchange == "fused":   # row pass stores straight into the peers' column slabs
        solver = S.FusedPeerSlabSolver(wl.nx, wl.ny, S.SymmetricPeerComm(), ops)
    elif args.exchange == "nccl":
        solver = S.SlabSolver(wl.nx, wl.ny, S.DistComm(), ops)
    out = [torch.empty_like(slab)]
    for _ in range(args.warmup):
        solver.diffuse([slab], wl.D, wl.dt, wl.nsteps, outs=out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = ops.launches
    barrier(world)
    torch.cuda.synchronize()
    gpu_index = torch.cuda.current_device()
    vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    smi_index = int(vis[gpu_index]) if len(vis) > gpu_index and vis[gpu_index].isdigit() else gpu_index
    with ClockSampler(smi_index) as clk:
        for i in range(args.steps):
            starts[i].record(stream)
            solver.diffuse([slab], wl.D, wl.dt, wl.nsteps, outs=out)
            ends[i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_total = max_over_ranks(world, sum(a.elapsed_time(b) for a, b in zip(starts, ends)))
    pts = wl.nx * wl.ny * wl.nsteps
    value = pts * args.steps / (ms_total * 1e-3)
    ops.plan.read_profile()
    ops.plan.set_profiling(True)
    solver.diffuse([slab], wl.D, wl.dt, wl.nsteps, outs=out)
    torch.cuda.synchronize()
    prof = ops.plan.read_profile()
    ops.plan.set_profiling(False)
    dom_name, (dom_ms, dom_n) = max(prof.items(), key=lambda kv: kv[1][0])
    slab_bytes = (hi - lo) * wl.nx * 16
    achieved = 2 * slab_bytes / (dom_ms / dom_n * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    a2a_bytes = slab_bytes * (world - 1) // world
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C5 recipe, built on device)",
        "config": {**workload_config(wl, world),
                   "parallelism": f"slab x{world} " + {
                       "peer": "(peer-store exchange, symmetric memory)",
                       "fused": "(row and column passes store into the peers' slabs, symmetric memory; separable diffusion)",
                       "nccl": "(NCCL all-to-all, Python-driven)",
                       "lib": "(NCCL all-to-all inside libfftpde, fftpde_plan_2d_sharded)"}[args.exchange],
                   "l2": "field (16 GiB) larger than L2"},
        "e2e": None, "cpu_baseline": None, "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "kernel": dom_name,
                     "per_kernel_ms_per_solve": {k: round(v[0], 3) for k, v in prof.items()},
                     "alltoall_bytes_per_rank": a2a_bytes, "alltoalls_per_solve": 2 * wl.nsteps},
        "gpu_launches": ops.launches - l0,
    }


def sharded3d_native(args, wl, world, rank, local):
    """3D workloads (p3d / d3d) at N > 1 or with --sharded: the z-slab decomposition
    inside libfftpde (fftpde_plan_3d_sharded, NCCL all-to-all between the xy passes
    and the z-pass); strong scaling (fixed volume)."""
    import torch
    from paper_2412_12308_b200 import fftpde as F
    host = make_inputs(wl)[0]
    nzl = wl.nz // world
    slab = torch.from_numpy(host[rank * nzl:(rank + 1) * nzl].copy()).cuda()
    plan = F.ShardedPlan3D(wl.nx, wl.ny, wl.nz, dtype=torch.complex128, Lx=wl.Lx, Ly=wl.Ly)
    out = torch.empty_like(slab)

    def solve():
        if wl.op == "poisson":
            plan.poisson(slab, out=out)
        else:
            plan.diffuse(slab, wl.D, wl.dt, wl.nsteps, out=out)

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = plan.launches
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            solve()
            ends[i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_total = max_over_ranks(world, sum(a.elapsed_time(b) for a, b in zip(starts, ends)))
    pts = wl.points * (wl.nsteps if wl.op != "poisson" else 1)
    plan.read_profile()
    plan.set_profiling(True)
    solve()
    torch.cuda.synchronize()
    prof = plan.read_profile()
    plan.set_profiling(False)
    dom_name, (dom_ms, dom_n) = max(prof.items(), key=lambda kv: kv[1][0])
    total = sum(v[0] for v in prof.values())
    dom_avg_s = dom_ms / total * (ms_total / args.steps) * 1e-3 / dom_n if total else dom_ms / dom_n * 1e-3
    achieved = 2 * slab.numel() * 16 / dom_avg_s / 1e9
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    return {
        "metric": METRIC, "value": pts * args.steps / (ms_total * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 3D Gaussians)",
        "config": {**workload_config(wl, world),
                   "parallelism": f"z-slab x{world} (NCCL all-to-all inside libfftpde, fftpde_plan_3d_sharded)",
                   "l2": "256 MiB buffer zeroed between timed steps"},
        "e2e": None, "cpu_baseline": None, "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "kernel": dom_name,
                     "per_kernel_ms_per_solve": {k: round(v[0], 3) for k, v in prof.items()},
                     "alltoalls_per_solve": 2 * (wl.nsteps if wl.op != "poisson" else 1)},
        "gpu_launches": plan.launches - l0,
    }


def alg_step_bytes(wl):
    """Algorithmic bytes of one bench step: each state field read + written once per
    solve step."""
    esz = {"c128": 16, "c64": 8, "f64": 8, "f32": 4}[wl.dtype]
    fields = 2 if wl.op in ("wave", "rk4") else 1
    steps = wl.nsteps if wl.op != "poisson" else 1
    return 2 * fields * wl.points * esz * steps


def workload_config(wl, world):
    cfg = {"workload": wl.name, "nx": wl.nx, "ny": wl.ny, **({"nz": wl.nz} if wl.nz > 1 else {}),
           "batch": wl.batch, "dtype": wl.dtype,
           "op": wl.op, "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
           "l2": "flushed between timed steps (256 MiB write)"}
    if wl.op in ("diffuse", "dsrc"):
        cfg.update({"nsteps": wl.nsteps, "D": wl.D, "dt": wl.dt})
    if wl.op == "dsrc":
        cfg.update({"source": "static: 0.5 x the C2 Gaussians", "baseline_config": False})
    if wl.op == "wave":
        cfg.update({"nsteps": wl.nsteps, "c": wl.c, "dt": wl.dt})
    if wl.op == "rk4":
        cfg.update({"nsteps": wl.nsteps, "c": wl.c, "dt": wl.dt, "domain": "[-2,2]^2",
                    "source": "orbiting Gaussian A=1 sigma=0.1 Omega=5 gamma=10 r_s=0.5 (PAPER.md:516-523)",
                    "baseline_config": False})
    return cfg


# ---------------------------------------------------------------------------- CPU oracle

def oracle_sample(wl, host, budget_s=12.0):
    """Time the oracle on a bounded sample of the workload; returns (pts/s, desc)."""
    import numpy as np
    from oracle import oracle as O
    if wl.nz > 1:
        t0 = time.perf_counter()
        if wl.op == "poisson":
            O.poisson3(host[0])
            k, what = 1, "1 3D Poisson solve"
        else:
            O.diffuse3(host[0], wl.D, wl.dt, 1)
            k, what = 1, f"1 of {wl.nsteps} 3D diffusion steps"
        dt = time.perf_counter() - t0
        return wl.points * k / dt, f"{what} ({wl.nz}x{wl.ny}x{wl.nx})"
    if wl.op == "poisson":
        grids = host[0].astype(np.complex128)
        if grids.ndim == 2:
            grids = grids[None]
        n = 0
        t0 = time.perf_counter()
        while n < grids.shape[0]:
            O.poisson(grids[n], wl.Lx, wl.Ly)
            n += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return wl.nx * wl.ny * n / dt, f"{n} of {wl.batch} Poisson solves ({wl.ny}x{wl.nx})"
    if wl.op == "diffuse":
        t0 = time.perf_counter()
        O.diffuse(host[0], wl.D, wl.dt, 1, wl.Lx, wl.Ly)
        one = time.perf_counter() - t0
        k = max(1, min(wl.nsteps, int(budget_s / max(one, 1e-6))))
        t0 = time.perf_counter()
        O.diffuse(host[0], wl.D, wl.dt, k, wl.Lx, wl.Ly)
        dt = time.perf_counter() - t0
        return wl.nx * wl.ny * k / dt, f"{k} of {wl.nsteps} stepped diffusion steps ({wl.ny}x{wl.nx}, full grid)"
    if wl.op == "dsrc":
        t0 = time.perf_counter()
        O.diffuse_source(host[0], host[1], wl.D, wl.dt, 1)
        one = time.perf_counter() - t0
        k = max(1, min(wl.nsteps, int(budget_s / max(one, 1e-6))))
        t0 = time.perf_counter()
        O.diffuse_source(host[0], host[1], wl.D, wl.dt, k)
        dt = time.perf_counter() - t0
        return wl.nx * wl.ny * k / dt, f"{k} of {wl.nsteps} sourced diffusion steps ({wl.ny}x{wl.nx})"
    if wl.op == "rk4":
        src = dict(Lx=wl.Lx, Ly=wl.Ly, xmin=-0.5 * wl.Lx, ymin=-0.5 * wl.Ly)
        t0 = time.perf_counter()
        O.wave_rk4(host[0], host[1], wl.dt, 1, c=wl.c, **src)
        one = time.perf_counter() - t0
        k = max(1, min(wl.nsteps, int(budget_s / max(one, 1e-6))))
        t0 = time.perf_counter()
        O.wave_rk4(host[0], host[1], wl.dt, k, c=wl.c, **src)
        dt = time.perf_counter() - t0
        return wl.nx * wl.ny * k / dt, f"{k} of {wl.nsteps} RK4 steps ({wl.ny}x{wl.nx})"
    t0 = time.perf_counter()
    O.wave(host[0], host[1], wl.c, wl.dt, 1, wl.Lx, wl.Ly)
    one = time.perf_counter() - t0
    k = max(1, min(wl.nsteps, int(budget_s / max(one, 1e-6))))
    if k > 1:
        t0 = time.perf_counter()
        O.wave(host[0], host[1], wl.c, wl.dt, k, wl.Lx, wl.Ly)
        dt = time.perf_counter() - t0
    else:
        dt = one
    return wl.nx * wl.ny * k / dt, f"{k} of {wl.nsteps} stepped wave steps ({wl.ny}x{wl.nx}, both fields)"


def cpu_baseline(wl, host):
    from oracle import oracle as O
    O.set_threads(os.cpu_count() or 1)
    if host is None:   # C5: time the oracle on one 8192^2 diffusion step of the same recipe
        import dataclasses
        from paper_2412_12308_b200 import inputs as I
        sub = dataclasses.replace(wl, nx=8192, ny=8192, nsteps=1)
        g = I.c2_inputs(8192, m=64, sig_lo=0.002, sig_hi=0.01)
        v, desc = oracle_sample(sub, (g.u0,))
        return {"value": v, "unit": UNIT, "cores": O.get_threads(), "kind": "oracle",
                "sample": "1 stepped diffusion step on an 8192^2 sub-problem of the C5 recipe: " + desc}
    v, desc = oracle_sample(wl, host)
    out = {"value": v, "unit": UNIT, "cores": O.get_threads(), "kind": "oracle", "sample": desc}
    if wl.name.split("_")[0] in ("c1", "c2", "c4"):      # also a 1-thread time for C1, C2, C4
        threads = O.get_threads()
        O.set_threads(1)
        try:
            v1, desc1 = oracle_sample(wl, host, budget_s=3.0)
            out["one_thread"] = {"value": v1, "sample": desc1}
        finally:
            O.set_threads(threads)
    return out


def reference(args, wl, world, rank):
    """The reference arm of this tier: the fp64 CPU oracle, as it stands."""
    if rank != 0:
        return None
    from oracle import oracle as O
    O.set_threads(os.cpu_count() or 1)
    if wl.name.startswith("c5"):
        import dataclasses
        from paper_2412_12308_b200 import inputs as I
        wl = dataclasses.replace(wl, nx=8192, ny=8192, nsteps=1)
        host = (I.c2_inputs(8192, m=64, sig_lo=0.002, sig_hi=0.01).u0,)
    else:
        host = make_inputs(wl)
    for _ in range(args.warmup):
        oracle_sample(wl, host, budget_s=2.0)
    vals, descs = [], []
    for _ in range(args.steps):
        v, d = oracle_sample(wl, host, budget_s=8.0)
        vals.append(v)
        descs.append(d)
    value = statistics.median(vals)
    pts_step = wl.points * (wl.nsteps if wl.op != "poisson" else 1)
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pts_step / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json recipe)", "config": workload_config(wl, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.get_threads(), "kind": "oracle",
                         "sample": descs[0] + "; median over steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse_args()
    import torch
    from paper_2412_12308_b200 import inputs as I
    wl = I.WORKLOADS.get(args.workload) or I.EXTRA_WORKLOADS[args.workload]
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        line = reference(args, wl, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    world, rank, local = dist_setup(args.gpus)
    if args.sharded and world == 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    if wl.name.startswith("c5") and (world > 1 or args.sharded):
        line = sharded_native(args, wl, world, rank, local)
    elif wl.nz > 1 and (world > 1 or args.sharded):
        line = sharded3d_native(args, wl, world, rank, local)
    else:
        line = native(args, wl, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
