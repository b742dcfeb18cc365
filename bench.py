"""bench.py -- timed run of the 2D FFT-PDE hot path (arXiv 2412.12308) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl reference]

A *step* is one pass of the whole hot path over one batch of synthetic input
(SURVEY.md 8(a) a1-a5).  The default workload is C5 (BASELINE.json configs[4]),
the largest configuration that fits one GPU: one ``fftpde_diffuse`` call of 20
exact diffusion steps on a 32768 x 32768 complex128 grid (16 GiB; each solve
step a forward 2D FFT, the k-space multiply and an inverse 2D FFT, the field
materialised every step).  The metric is grid-points per second
(nx*ny*batch*nsteps / time) for the whole job; rank 0 prints one JSON line.

Multi-GPU: ``--gpus N`` with N > 1 launches N ranks itself (torch.distributed.run,
127.0.0.1) unless WORLD_SIZE is already set, and checks WORLD_SIZE == N.  C5 at
N > 1 runs the row-slab decomposition of SURVEY.md 8(e) (strong scaling, fixed
32768^2 grid); the default exchange is ``fs``: the distributed four-step (DESIGN.md
R28: each rank runs the single-GPU four-step passes on its Y-part / X-part of the
field) with the part-to-part exchange fused into the B passes (peer stores over
NVLink into torch symmetric memory, one barrier per solve step); ``lib`` runs the
same passes inside libfftpde with one NCCL all-to-all per step.  C1-C4 at N > 1 run independent
replicas (weak scaling, no collective on the data path).

Timing: W untimed warm-up steps, then exactly K steps, each bracketed by CUDA
events on the plan's stream; L2 (126 MB) is flushed with a 256 MiB write
between timed steps (outside the events; C5's field is larger than L2 anyway).
Barrier + synchronize on both sides of the timed region; the per-rank device
time is reduced with MAX over ranks.

Extra keys: ``e2e`` (the same metric through the public API with pinned host
buffers: host -> device copy, solve, device -> host copy, every step),
``roofline`` (every kernel class's share-scaled launch time against the HBM
and the FP64 roofs, the binding one computed per class; the step against the
method's algorithmic bytes), ``parity`` (C5: the periodic heat kernel at
sampled points and the mean drift; C1-C4: relative L2 against the fp64 oracle,
computed in the cpu_baseline leg), ``cpu_baseline`` (the fp64 oracle on this
host's cores, bounded sample; rank 0, N = 1), ``clocks`` (nvidia-smi sampled
during the timed region), ``gpu_launches`` (library kernels in the timed region).

``--impl reference`` times the CPU oracle (the reference arm of this tier) with
the same ``config``, metric and unit, each step a bounded sample named in
``cpu_baseline.sample``.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL's version banner goes to stdout on rank 0; the contract is one JSON line
os.environ.setdefault("NCCL_DEBUG", "WARN")

METRIC = "2D FFT-PDE solve grid-points/sec and achieved HBM GB/s vs peak (1/2/4/8 GPU)"
UNIT = "grid-points/s"
L2_FLUSH_BYTES = 256 << 20
NVLINK_GBS = 770.0            # measured peer copy per direction (B200_PROFILING.md); 900 nominal
FALLBACK_HBM_GBS = 6650.0     # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
L2_BYTES_PER_CLK = 6300.0     # B300_MICROARCH.md full-chip LTS throughput cap (guide value)

THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "rk4", "rk4big", "dsrc", "p3d",
                                                        "d3d", "c2r", "c3r", "c4r"],
                    help="c1-c5: BASELINE.json configs[0..4] (default c5, the largest single-GPU config); "
                         "rk4/rk4big: the paper's orbiting-source RK4 run (SURVEY.md 8(f) row 1, not a BASELINE config)")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="c5: use the slab-decomposed path even on one GPU (P = 1 process group)")
    ap.add_argument("--pencil", default=None, metavar="PZxPY",
                    help="3D workloads: the pencil decomposition on a PZ x PY process grid (PZ*PY = --gpus; "
                         "fftpde_plan_3d_pencil) instead of z-slabs")
    ap.add_argument("--exchange", default="fs", choices=["fs", "lib", "fused", "nccl", "peer"],
                    help="sharded c5: the distributed four-step with its exchange fused into the B passes (peer "
                         "stores into torch symmetric memory; default, falls back to lib), the distributed "
                         "four-step inside libfftpde (fftpde_plan_2d_sharded, one NCCL all-to-all per step), "
                         "or the round-1 slab solvers: exchanges fused into "
                         "the row / column passes (peer stores into torch symmetric memory), pack + NCCL "
                         "all-to-all, a separate peer-store transpose")
    return ap.parse_args()


def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args):
    """--gpus N without a launcher: run this script under torch.distributed.run with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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
        f, centres, sigmas, amps = I.c5_field_torch(wl.nx, dtype=dtype)
        return [f], None, (centres, sigmas, amps)
    host = make_inputs(wl)
    return [torch.from_numpy(np.ascontiguousarray(h)).to(dtype).cuda() for h in host], host, None


def esize(wl):
    return {"c128": 16, "c64": 8, "f64": 8, "f32": 4}[wl.dtype]


def field_bytes(wl):
    return wl.nx * wl.ny * wl.nz * wl.batch * esize(wl)


def pass_bytes_per_launch(wl, kernel_class):
    """Bytes a launch of the class must move by its own function, averaged over the
    launches of a solve: every field it touches read once and written once; a MID
    pass (inverse of step s stored as the physical field + forward of step s+1)
    reads once and writes twice.  Summed over the step these are the design's
    bytes; the method's own minimum is alg_step_bytes."""
    field = field_bytes(wl)
    n = wl.nsteps
    if kernel_class == "wave_col_pass":
        return 2 * 2 * field
    if kernel_class == "aa_pass":          # C5 four-step: 1 AA, n-1 MID, 1 AA^-1 per solve
        return (2 * field * 2 + 3 * field * (n - 1)) / (n + 1) if n > 1 else 2 * field
    if wl.op == "dsrc":
        return 3 * field if kernel_class == "pointwise" else 2 * field
    if wl.op == "rk4":
        return 3 * field if kernel_class == "pointwise" else 2 * field
    if kernel_class == "row_pass" and wl.op == "wave" and n > 1:
        return (2 * field * 2 + 3 * field * (n - 1)) / (n + 1)
    return 2 * field


def alg_step_bytes(wl):
    """The method's algorithmic bytes of one bench step: each state field read and
    written once per solve step (SURVEY.md 8(d) table, 32 B/pt/step for one c128 field)."""
    fields = 2 if wl.op in ("wave", "rk4") else 1
    steps = wl.nsteps if wl.op != "poisson" else 1
    return 2 * fields * wl.points * esize(wl) * steps


def survey_design_passes(wl):
    """the 3-pass design roof (1 pass for the single-CTA C1 grid)."""
    return 1 if wl.name.startswith("c1") else 3


# ---------------------------------------------------------------------------- peaks

def load_peaks():
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs")
    src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if hbm else "fallback 6650 GB/s (B200_PROFILING.md)"
    # FP64 / FP32 instruction roofs measured on this pool (tools/fp64_peak.cu, profiles/r02/fp64_peak.jsonl)
    dp, sp, alu_src = 18.46e12, 36.20e12, "profiles/r02/fp64_peak.jsonl (measured DADD / FADD rate, 1965 MHz)"
    try:
        for line in open(os.path.join(ROOT, "profiles", "r02", "fp64_peak.jsonl")):
            d = json.loads(line)
            if d.get("kind") == "dadd":
                dp = d["ginst_per_s"] * 1e9
            if d.get("kind") == "fadd":
                sp = d["ginst_per_s"] * 1e9
    except Exception:
        alu_src = "vendor lane counts: 64 FP64 / 128 FP32 lanes per SM x 148 SMs x 1965 MHz"
    return {"hbm_gbs": hbm or FALLBACK_HBM_GBS, "hbm_src": src, "dp_inst_s": dp, "sp_inst_s": sp, "alu_src": alu_src}


def load_counts(wl):
    """Per-launch ncu counts of each kernel class (tools/kernel_counts.py): DRAM bytes
    and FP64 / FP32 thread instructions; None where no capture is committed."""
    for name in (f"counts_{wl.name}.json", f"traffic_{wl.name}.json"):
        p = os.path.join(ROOT, "profiles", name)
        if os.path.exists(p):
            try:
                return json.load(open(p)), name
            except Exception:
                pass
    return {}, None


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


def smi_index():
    import torch
    gpu_index = torch.cuda.current_device()
    vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    return int(vis[gpu_index]) if len(vis) > gpu_index and vis[gpu_index].isdigit() else gpu_index


# ---------------------------------------------------------------------------- dist

def dist_setup():
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


def reduce_over_ranks(world, value, op="max"):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
    return float(t.item())


# ---------------------------------------------------------------------------- roofline

def roofline_block(wl, prof, ms_per_step, steps, world=1, slab_fraction=1.0, extra=None):
    """Every kernel class against the HBM and the FP64 (FP32 for complex64) roofs.

    Per class: the launch time is the class's share of the profiled replays x the
    un-instrumented CUDA-event step time / launches per step; T_hbm = the pass's own
    bytes / peak HBM; T_alu = its FP64 (FP32) instructions per launch (ncu counts,
    tools/kernel_counts.py) / the measured instruction rate; the binding roof is the
    larger of the two and frac = T_bound / launch time.  The dominant class (largest
    share) fills the contract keys.  `step` compares the whole step with the method's
    algorithmic bytes (one read + one write of each state field per solve step) and
    with the survey's 3-pass design roof, so no pass is counted against the method twice."""
    peaks = load_peaks()
    counts, counts_src = load_counts(wl)
    fp32 = wl.dtype in ("c64", "f32")
    # a field pair that stays in the 126 MB L2 between passes (C2: 2 x 16 MiB) is not
    # bound by HBM: its memory roof is the L2 slice throughput (B300_MICROARCH.md:
    # ~6300 B/clk full chip, not measured on B200), so the binding roof there is the
    # larger of the L2 and ALU times
    l2_resident = 2 * field_bytes(wl) * slab_fraction <= (64 << 20)
    mem_peak = L2_BYTES_PER_CLK * 1965e6 if l2_resident else peaks["hbm_gbs"] * 1e9
    alu_peak = peaks["sp_inst_s"] if fp32 else peaks["dp_inst_s"]
    classes = {k: v for k, v in prof.items() if v[1] > 0}
    total = sum(v[0] for v in classes.values()) or 1.0
    per = {}
    for k, (ms, n) in classes.items():
        lps = n / steps
        share = ms / total
        t_launch = share * ms_per_step * 1e-3 / lps
        pb = pass_bytes_per_launch(wl, k) * slab_fraction
        t_hbm = pb / mem_peak
        c = counts.get(k) if isinstance(counts.get(k), dict) else None
        inst = None
        if c:
            inst = c.get("sp_inst" if fp32 else "dp_inst")
        t_alu = inst * slab_fraction / alu_peak if inst else None
        bound = "alu" if (t_alu is not None and t_alu > t_hbm) else ("l2" if l2_resident else "hbm")
        traffic = c.get("dram_bytes") if c else (counts.get(k) if isinstance(counts.get(k), (int, float)) else None)
        per[k] = {
            "share_of_step": round(share, 4), "launches_per_step": lps, "ms_per_launch": round(t_launch * 1e3, 4),
            "pass_bytes_per_launch": pb, "gbs": round(pb / t_launch / 1e9, 1),
            "mem_frac": round(t_hbm / t_launch, 4), "mem_roof": "l2" if l2_resident else "hbm",
            "fp_inst_per_launch": inst, "alu_frac": round(t_alu / t_launch, 4) if t_alu else None,
            "bound": bound, "traffic": traffic,
            "traffic_over_pass_bytes": round(traffic / pb, 3) if traffic else None,
        }
    dom = max(per, key=lambda k: per[k]["share_of_step"])
    d = per[dom]
    t_launch = d["ms_per_launch"] * 1e-3
    if d["bound"] == "alu":
        achieved = d["fp_inst_per_launch"] * slab_fraction / t_launch / 1e9
        peak, unit = alu_peak / 1e9, ("GFP32inst/s" if fp32 else "GFP64inst/s")
        peak_src = peaks["alu_src"]
    elif l2_resident:
        achieved = d["pass_bytes_per_launch"] / t_launch / 1e9
        peak, unit = mem_peak / 1e9, "GB/s"
        peak_src = "L2 (field L2-resident): B300_MICROARCH.md LTS cap 6300 B/clk x 1965 MHz (guide value, not measured on B200)"
    else:
        achieved = d["pass_bytes_per_launch"] / t_launch / 1e9
        peak, unit, peak_src = peaks["hbm_gbs"], "GB/s", peaks["hbm_src"]
    step_s = ms_per_step * 1e-3
    alg = alg_step_bytes(wl) * slab_fraction
    design = sum(v["pass_bytes_per_launch"] * v["launches_per_step"] for v in per.values())
    t3 = survey_design_passes(wl) * alg / (peaks["hbm_gbs"] * 1e9)
    out = {
        "bound": d["bound"] if not (l2_resident and d["bound"] == "hbm") else "l2",
        "achieved": round(achieved, 1), "peak": peak, "unit": unit, "l2_resident": l2_resident,
        "frac": round(achieved / peak, 4), "traffic": d["traffic"], "kernel": dom,
        "peak_source": peak_src, "counts_source": counts_src,
        "alg_bytes_per_launch": d["pass_bytes_per_launch"],
        "duration_method": "class share of CUDA-event-profiled replays x un-instrumented CUDA-event step time",
        "per_kernel": per,
        "step": {
            "alg_bytes": alg, "alg_gbs": round(alg / step_s / 1e9, 1),
            "alg_frac": round(alg / step_s / 1e9 / peaks["hbm_gbs"], 4),
            "design_bytes": design, "design_round_trips": round(design / alg, 3),
            "design_gbs": round(design / step_s / 1e9, 1),
            "design_frac": round(design / step_s / 1e9 / peaks["hbm_gbs"], 4),
            "survey_3pass_ms": round(t3 * 1e3, 4), "survey_3pass_frac": round(t3 / step_s, 4),
            "note": "alg_frac: the method's one round trip per solve step (SURVEY.md 8(d)); "
                    "survey_3pass_frac: the survey's 3-pass design roof / step time (north_star's >= 60% bar)",
        },
    }
    if extra:
        out.update(extra)
    return out


# ---------------------------------------------------------------------------- parity

def heat_kernel_points(ks, js, n, centres, sigmas, amps, D, T):
    """The exact solution of u_t = D nabla^2 u from a sum of Gaussians A e^{-d^2/sigma^2}
    (PAPER.md:390-398), summed over the periodic images +-1 (R9):
    u = sum_i A_i sigma_i^2 / (sigma_i^2 + 4 D T) exp(-d^2 / (sigma_i^2 + 4 D T))."""
    import numpy as np
    x, y = js / n, ks / n
    out = np.zeros(len(ks))
    for (cx, cy), s, a in zip(centres, sigmas, amps):
        s2 = s * s + 4 * D * T
        for ix in (-1, 0, 1):
            for iy in (-1, 0, 1):
                dx = x - cx + ix
                dy = y - cy + iy
                out += a * (s * s / s2) * np.exp(-(dx * dx + dy * dy) / s2)
    return out


def c5_parity(u_dev, u0_dev, params, wl, row0=0):
    """Heat kernel at sampled points of this rank's rows [row0, row0 + rows) and the
    sums for the mean drift (Fig. 4)."""
    import numpy as np
    import torch
    centres, sigmas, amps = params
    n = wl.nx
    rows = u_dev.shape[0]
    rng = np.random.default_rng(5 + row0)
    ks = rng.integers(0, rows, 1500)
    js = rng.integers(0, n, 1500)
    near = [(round(cy * n) % n - row0, round(cx * n) % n) for (cx, cy) in centres[:400]
            if 0 <= round(cy * n) % n - row0 < rows]
    if near:
        ks = np.concatenate([ks, np.array([k for k, _ in near])])
        js = np.concatenate([js, np.array([j for _, j in near])])
    got = u_dev[torch.from_numpy(ks).cuda(), torch.from_numpy(js).cuda()].cpu().numpy()
    exact = heat_kernel_points(ks + row0, js, n, centres, sigmas, amps, wl.D, wl.nsteps * wl.dt)
    return {"err2": float(np.sum(np.abs(got - exact) ** 2)), "ref2": float(np.sum(exact ** 2)),
            "max_imag": float(np.max(np.abs(got.imag))), "points": int(len(ks)),
            "sum_u": float(u_dev.real.double().sum().item()), "sum_u0": float(u0_dev.real.double().sum().item())}


def finish_c5_parity(parts, world):
    import math as m
    err2 = reduce_over_ranks(world, parts["err2"], "sum")
    ref2 = reduce_over_ranks(world, parts["ref2"], "sum")
    su = reduce_over_ranks(world, parts["sum_u"], "sum")
    su0 = reduce_over_ranks(world, parts["sum_u0"], "sum")
    mi = reduce_over_ranks(world, parts["max_imag"], "max")
    pts = reduce_over_ranks(world, parts["points"], "sum")
    return {"kind": "closed form: periodic heat kernel at sampled points (PAPER.md:376-398) + mean drift (Fig. 4)",
            "rel_l2": m.sqrt(err2 / ref2), "points": int(pts), "mean_drift": abs(su / su0 - 1.0),
            "max_abs_imag": mi, "tolerance": 1e-12, "pass": m.sqrt(err2 / ref2) <= 1e-12 and abs(su / su0 - 1) <= 1e-12}


def rel_l2(a, b):
    import numpy as np
    a = np.asarray(a, np.complex128).ravel()
    b = np.asarray(b, np.complex128).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_parity(wl, host, outs):
    """C1-C4 parity against the fp64 oracle on the same input bytes (cpu_baseline leg)."""
    import numpy as np
    from oracle import oracle as O
    tol = 1e-5 if wl.dtype == "c64" else 1e-12
    got = [o.cpu().numpy() for o in outs]
    if wl.name.startswith("c1"):
        return {"kind": "oracle, full solve", "rel_l2": rel_l2(got[0], O.poisson(host[0])), "tolerance": tol}
    if wl.name.startswith("c2"):
        ref = O.diffuse(host[0], wl.D, wl.dt, wl.nsteps)
        mean0 = float(np.mean(host[0].real))
        return {"kind": "oracle, full stepped solve", "rel_l2": rel_l2(got[0], ref), "tolerance": tol,
                "mean_drift": abs(float(np.mean(got[0].real)) / mean0 - 1.0)}
    if wl.name.startswith("c3"):
        U, V = O.wave(host[0], host[1], wl.c, wl.dt, wl.nsteps, collapsed=True)
        mean0 = float(np.mean(host[0].real))
        return {"kind": "oracle, collapsed (one propagator at T = nsteps dt)", "rel_l2_u": rel_l2(got[0], U),
                "rel_l2_ut": rel_l2(got[1], V), "tolerance": tol,
                "mean_drift": abs(float(np.mean(got[0].real)) / mean0 - 1.0)}
    if wl.name.startswith("c4"):
        errs = [rel_l2(got[0][g], O.poisson(host[0][g].astype(np.complex128))) for g in (0, 85, 170, 255)]
        return {"kind": "oracle, grids 0/85/170/255 (upcast input)", "rel_l2_max": max(errs), "tolerance": tol}
    return None


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


def timed_steps(args, world, stream, flush, body, pre=None):
    """W warm-up steps, one untimed step after the clock sampler starts, then K
    event-bracketed steps (L2 flushed before each).  Returns (per-step ms, clocks)."""
    import torch
    for _ in range(args.warmup):
        if pre:
            pre()
        body()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(smi_index()) as clk:
        # the GPU idled while the sampler started: one more untimed step
        if pre:
            pre()
        flush.zero_()
        body()
        for i in range(args.steps):
            if pre:
                pre()
            flush.zero_()
            starts[i].record(stream)
            body()
            ends[i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    return [s.elapsed_time(e) for s, e in zip(starts, ends)], clk.summary()


def native(args, wl, world, rank, local):
    import numpy as np
    import torch
    from paper_2412_12308_b200 import fftpde as F

    dtype = {"c128": torch.complex128, "c64": torch.complex64, "f64": torch.float64,
             "f32": torch.float32}[wl.dtype]
    dev_in, host, c5params = make_device_inputs(wl, dtype)
    out = [torch.empty_like(d) for d in dev_in]
    if wl.dtype in ("f64", "f32"):
        plan = F.PlanR2C(wl.nx, wl.ny, batch=wl.batch, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
    elif wl.nz > 1:
        plan = F.Plan3D(wl.nx, wl.ny, wl.nz, dtype=dtype)
    else:
        plan = F.Plan(wl.nx, wl.ny, batch=wl.batch, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    launches = {}

    def body():
        run_solve(plan, wl, dev_in, out)

    l0 = plan.launches
    times, clocks = timed_steps(args, world, stream, flush, body, pre=lambda: reset_wave(wl, dev_in, out))
    launches = (plan.launches - l0) * args.steps // (args.warmup + 1 + args.steps)
    ms_rank = sum(times)
    ms_total = reduce_over_ranks(world, ms_rank)
    ms_per_step = ms_total / args.steps
    pts_per_step = wl.points * (wl.nsteps if wl.op != "poisson" else 1)
    value = world * pts_per_step * args.steps / (ms_total * 1e-3)

    # ---- parity of the last timed step's output (outside the timed region)
    parity = None
    if not args.no_parity and c5params is not None:
        parity = finish_c5_parity(c5_parity(out[0], dev_in[0], c5params, wl), world)

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
    roofline = roofline_block(wl, prof, ms_per_step, args.steps)

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
        tot = reduce_over_ranks(world, tot)
        nbytes = sum(h.numel() * h.element_size() for h in host_in)
        e2e = {"value": world * pts_per_step * args.steps / tot, "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "timer": "host perf_counter around the public-API call (pinned host buffers), one step at a time"}
        if wl.op in ("poisson", "diffuse", "wave") and wl.dtype in ("c128", "c64") and wl.nz == 1:
            host_out.clear()                                  # (pinned host memory of the one-at-a-time leg)
            tp = e2e_pipelined(args, wl, plan, dev_in, out, host_in, dtype, world)
            e2e.update({"value": world * pts_per_step * args.steps / tp, "sync_value": e2e["value"],
                        "timer": "host perf_counter around K steps, each step the H2D copy of its inputs from "
                                 "pinned host memory, the solve, and the D2H copy of its result; the copies of "
                                 "step i+1 / i-1 overlap the solve of step i (copy streams, two buffer slots); "
                                 "sync_value: the same with one step at a time"})
        del host_in, host_out

    # ---- CPU oracle baseline (rank 0, N = 1); C1-C4 parity against the oracle
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, host)
        if not args.no_parity and host is not None and wl.name[:2] in ("c1", "c2", "c3", "c4") and wl.nz == 1 \
                and wl.dtype in ("c128", "c64"):
            reset_wave(wl, dev_in, out)
            run_solve(plan, wl, dev_in, out)
            torch.cuda.synchronize()
            parity = oracle_parity(wl, host, out)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "median_ms_per_step": reduce_over_ranks(world, statistics.median(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if wl.dtype in ("c128", "f64") else "f32",
        "data": "synthetic (seeded, BASELINE.json recipe; paper_2412_12308_b200/inputs.py)",
        "config": workload_config(wl, world),
        "e2e": e2e, "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "clocks": clocks,
        "gpu_launches": launches,
        "hbm_gbs_alg": round(world * alg_step_bytes(wl) * args.steps / (ms_total * 1e-3) / 1e9, 1),
    }
    return line


def e2e_pipelined(args, wl, plan, dev_in, out, host_in, dtype, world):
    """K steps through the public API with host buffers, the copies of neighbouring
    steps overlapping the solve: H2D of step i on one stream, the solve on the plan's
    stream, D2H on a third, two device / host buffer slots ordered by events.
    Returns the max-over-ranks host time of the K steps."""
    import torch
    nslot = 2
    fields = len(dev_in)
    ins = [out] + [[torch.empty_like(d) for d in dev_in] for _ in range(nslot - 1)]
    outs = [[torch.empty_like(d) for d in dev_in] for _ in range(nslot)] if wl.op != "wave" else ins
    houts = [[torch.empty(h.shape, dtype=dtype, pin_memory=True) for h in host_in] for _ in range(nslot)]
    s_c = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(nslot)]
    ev_c = [torch.cuda.Event() for _ in range(nslot)]
    ev_out = [torch.cuda.Event() for _ in range(nslot)]
    used = [False] * nslot

    def one(i):
        j = i % nslot
        with torch.cuda.stream(s_in):
            if used[j]:
                s_in.wait_event(ev_c[j])                  # the slot's previous solve has read it
            for d, h in zip(ins[j], host_in):
                d.copy_(h, non_blocking=True)
            ev_in[j].record(s_in)
        s_c.wait_event(ev_in[j])
        if used[j]:
            s_c.wait_event(ev_out[j])                     # the slot's previous result has been read out
        if wl.op == "poisson":
            plan.poisson(ins[j][0], out=outs[j][0])
        elif wl.op == "diffuse":
            plan.diffuse(ins[j][0], wl.D, wl.dt, wl.nsteps, out=outs[j][0])
        else:
            plan.wave_step(ins[j][0], ins[j][1], wl.c, wl.dt, wl.nsteps)
        ev_c[j].record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_c[j])
            for h, d in zip(houts[j], outs[j][:fields]):
                h.copy_(d, non_blocking=True)
            ev_out[j].record(s_out)
        used[j] = True

    for i in range(nslot):
        one(i)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for i in range(args.steps):
        one(i)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    barrier(world)
    del ins, outs, houts
    torch.cuda.empty_cache()
    return reduce_over_ranks(world, t)


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
    """C5 at N > 1 (or --sharded): the row-slab decomposition; strong
    scaling (fixed 32768^2 grid).  Roofline: max(T_HBM, T_NVL) per rank with the
    variant's own pass count (SURVEY.md 8(e) table and HBM-cost note)."""
    import torch
    from paper_2412_12308_b200 import inputs as I
    from paper_2412_12308_b200 import sharded as S
    dtype = torch.complex128
    full, centres, sigmas, amps = I.c5_field_torch(wl.nx, dtype=dtype)
    lo, hi = S.slab_rows(wl.ny, world, rank)
    slab = full[lo:hi].contiguous()
    del full
    torch.cuda.empty_cache()
    exchange = args.exchange
    fallback = None
    if exchange == "fs":      # R28 with the exchange fused into the B passes (peer stores, symmetric memory)
        try:
            ops = S.CudaLocalOps(wl.nx, wl.ny, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
            solver = S.FusedFourStepSolver(wl.nx, S.SymmetricPeerComm() if world > 1 else S.LoopbackPeerComm(1),
                                           ops.plan)
        except Exception as e:  # no peer-mapped symmetric memory here: the in-library NCCL exchange
            fallback = f"fs unavailable ({type(e).__name__}: {e}); lib"
            exchange = "lib"
            ops = solver = None
            torch.cuda.empty_cache()
    if exchange == "fs":
        pass
    elif exchange == "lib":     # the whole slab solve inside the C ABI (fftpde_plan_2d_sharded)
        from paper_2412_12308_b200 import fftpde as F
        ops = _LibSharded(F.ShardedPlan(wl.nx, wl.ny, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly))
        solver = ops
    else:
        ops = S.CudaLocalOps(wl.nx, wl.ny, dtype=dtype, Lx=wl.Lx, Ly=wl.Ly)
        if exchange == "peer":
            solver = S.PeerSlabSolver(wl.nx, wl.ny, S.SymmetricPeerComm(), ops)
        elif exchange == "fused":   # row and column passes store straight into the peers' slabs
            solver = S.FusedPeerSlabSolver(wl.nx, wl.ny, S.SymmetricPeerComm(), ops)
        else:
            solver = S.SlabSolver(wl.nx, wl.ny, S.DistComm(), ops)
    out = [torch.empty_like(slab)]
    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    l0 = ops.launches

    def body():
        solver.diffuse([slab], wl.D, wl.dt, wl.nsteps, outs=out)

    times, clocks = timed_steps(args, world, stream, flush, body)
    launches = (ops.launches - l0) * args.steps // (args.warmup + 1 + args.steps)
    ms_total = reduce_over_ranks(world, sum(times))
    ms_per_step = ms_total / args.steps
    pts = wl.nx * wl.ny * wl.nsteps
    value = pts * args.steps / (ms_total * 1e-3)
    parity = None
    if not args.no_parity:
        parity = finish_c5_parity(c5_parity(out[0], slab, (centres, sigmas, amps), wl, row0=lo), world)
    ops.plan.read_profile()
    ops.plan.set_profiling(True)
    solver.diffuse([slab], wl.D, wl.dt, wl.nsteps, outs=out)
    torch.cuda.synchronize()
    prof = ops.plan.read_profile()
    ops.plan.set_profiling(False)
    # e2e: every rank's slab from pinned host memory, the solve, the slab back (max over ranks)
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty(slab.shape, dtype=slab.dtype, pin_memory=True)
        host_in.copy_(slab)
        host_out = torch.empty_like(host_in, pin_memory=True)
        dev_in = torch.empty_like(slab)

        def e2e_step():
            dev_in.copy_(host_in, non_blocking=True)
            solver.diffuse([dev_in], wl.D, wl.dt, wl.nsteps, outs=out)
            host_out.copy_(out[0], non_blocking=True)
            torch.cuda.current_stream().synchronize()

        e2e_step()
        barrier(world)
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            e2e_step()
            barrier(world)
            tot += time.perf_counter() - t0
        tot = reduce_over_ranks(world, tot)
        nb = host_in.numel() * host_in.element_size()
        e2e = {"value": pts * args.steps / tot, "unit": UNIT, "h2d_bytes_per_step": nb * world,
               "d2h_bytes_per_step": nb * world,
               "timer": "host perf_counter around H2D slab copy + sharded solve + D2H slab copy, barrier-bracketed, "
                        "max over ranks; bytes summed over ranks"}
        del host_in, host_out, dev_in
    # per rank and step: HBM = passes x (read + write) of the slab, NVLink = the
    # bytes leaving the rank in the two exchanges (per direction).  lib = the
    # distributed four-step (R28): per step Bx + By (2 x slab each) and MID
    # (3 x slab) and ONE all-to-all; per solve the row-slab <-> Y-part conversion (a
    # permutation and a block swap each way, 8 x slab) and two more all-to-alls
    slab_bytes = (hi - lo) * wl.nx * 16
    if exchange in ("lib", "fs"):
        conv = 1 if world > 1 else 0        # P = 1: the parts are the row slab, no conversion
        hbm_step = (7 + conv * 8 / wl.nsteps) * slab_bytes
        nvl_bytes = int(slab_bytes * (world - 1) / world * (1 + 2 / wl.nsteps))
    else:
        hbm_step = {"fused": 2, "peer": 3, "nccl": 5}[exchange] * 2 * slab_bytes
        nvl_bytes = 2 * slab_bytes * (world - 1) // world
    peaks = load_peaks()
    t_hbm = hbm_step / (peaks["hbm_gbs"] * 1e9)
    t_nvl = nvl_bytes / (NVLINK_GBS * 1e9)
    step_s = ms_per_step * 1e-3 / wl.nsteps
    prof_steps = {k: (v[0], v[1]) for k, v in prof.items()}
    extra = {"sharded": {
        "exchange": exchange, "ranks": world, "slab_bytes": slab_bytes,
        "hbm_bytes_per_rank_step": int(hbm_step), "nvlink_bytes_per_rank_step": nvl_bytes,
        "nvlink_gbs_per_rank": round(nvl_bytes / step_s / 1e9, 1) if world > 1 else 0.0,
        "t_hbm_ms": round(t_hbm * 1e3, 4), "t_nvl_ms": round(t_nvl * 1e3, 4),
        "roof": "nvlink" if t_nvl > t_hbm else "hbm",
        "frac_of_max_roof": round(max(t_hbm, t_nvl) / step_s, 4),
        "nvlink_peak_gbs": NVLINK_GBS, "nvlink_peak_source": "B200_PROFILING.md measured peer copy per direction",
    }}
    roofline = roofline_block(wl, prof_steps, ms_per_step, 1, world, slab_fraction=(hi - lo) / wl.ny, extra=extra)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "median_ms_per_step": reduce_over_ranks(world, statistics.median(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C5 recipe, built on device)",
        "config": {**workload_config(wl, world),
                   "parallelism": f"slab x{world} " + {
                       "peer": "(peer-store exchange, symmetric memory)",
                       "fused": "(row and column passes store into the peers' slabs, symmetric memory; separable diffusion)",
                       "nccl": "(NCCL all-to-all, Python-driven)",
                       "lib": "(distributed four-step inside libfftpde, fftpde_plan_2d_sharded: Y-/X-parts, one NCCL "
                              "all-to-all per step)",
                       "fs": "(distributed four-step, the Y-/X-part exchange fused into the B passes: peer stores "
                             "into symmetric memory, one barrier per step)"}[exchange]
                   + (f" [{fallback}]" if fallback else ""),
                   "l2": "field (16 GiB) larger than L2; 256 MiB buffer zeroed between timed steps"},
        "e2e": e2e, "cpu_baseline": None, "clocks": clocks, "parity": parity,
        "roofline": roofline, "gpu_launches": launches,
    }


def sharded3d_native(args, wl, world, rank, local):
    """3D workloads (p3d / d3d) at N > 1 or with --sharded: the z-slab decomposition
    inside libfftpde (fftpde_plan_3d_sharded, NCCL all-to-all between the xy passes
    and the z-pass); strong scaling (fixed volume)."""
    import torch
    from paper_2412_12308_b200 import fftpde as F
    host = make_inputs(wl)[0]
    if args.pencil:
        pz, py = (int(v) for v in args.pencil.lower().split("x"))
        if pz * py != world:
            raise SystemExit(f"--pencil {args.pencil}: {pz * py} ranks, --gpus {world}")
        i, j = rank // py, rank % py
        nzl, nyl = wl.nz // pz, wl.ny // py
        slab = torch.from_numpy(host[i * nzl:(i + 1) * nzl, j * nyl:(j + 1) * nyl].copy()).cuda()
        plan = F.PencilPlan3D(wl.nx, wl.ny, wl.nz, pz, py, dtype=torch.complex128, Lx=wl.Lx, Ly=wl.Ly)
        layout = f"pencils {pz}x{py} (two group all-to-alls per transform inside libfftpde, fftpde_plan_3d_pencil)"
    else:
        nzl = wl.nz // world
        slab = torch.from_numpy(host[rank * nzl:(rank + 1) * nzl].copy()).cuda()
        plan = F.ShardedPlan3D(wl.nx, wl.ny, wl.nz, dtype=torch.complex128, Lx=wl.Lx, Ly=wl.Ly)
        layout = f"z-slab x{world} (NCCL all-to-all inside libfftpde, fftpde_plan_3d_sharded)"
    out = torch.empty_like(slab)

    def body():
        if wl.op == "poisson":
            plan.poisson(slab, out=out)
        else:
            plan.diffuse(slab, wl.D, wl.dt, wl.nsteps, out=out)

    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    l0 = plan.launches
    times, clocks = timed_steps(args, world, stream, flush, body)
    launches = (plan.launches - l0) * args.steps // (args.warmup + 1 + args.steps)
    ms_total = reduce_over_ranks(world, sum(times))
    pts = wl.points * (wl.nsteps if wl.op != "poisson" else 1)
    plan.read_profile()
    plan.set_profiling(True)
    body()
    torch.cuda.synchronize()
    prof = plan.read_profile()
    plan.set_profiling(False)
    roofline = roofline_block(wl, prof, ms_total / args.steps, 1, world, slab_fraction=1.0 / world)
    return {
        "metric": METRIC, "value": pts * args.steps / (ms_total * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 3D Gaussians)",
        "config": {**workload_config(wl, world),
                   "parallelism": layout,
                   "l2": "256 MiB buffer zeroed between timed steps"},
        "e2e": None, "cpu_baseline": None, "clocks": clocks, "parity": None,
        "roofline": roofline, "gpu_launches": launches,
    }


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

def c5_sample_workload(wl):
    """C5's bounded oracle sample: one stepped diffusion step of an 8192^2 grid with the
    C5 recipe (the full 32768^2 step needs ~50 GiB of host memory and about a minute)."""
    import dataclasses
    from paper_2412_12308_b200 import inputs as I
    sub = dataclasses.replace(wl, nx=8192, ny=8192, nsteps=1)
    g = I.c2_inputs(8192, m=64, sig_lo=0.002, sig_hi=0.01)
    return sub, (g.u0,)


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
        if k > 1:
            t0 = time.perf_counter()
            O.diffuse(host[0], wl.D, wl.dt, k, wl.Lx, wl.Ly)
            dt = time.perf_counter() - t0
        else:
            dt = one
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
    if host is None:   # C5: the oracle on a bounded sample of the same recipe
        sub, h = c5_sample_workload(wl)
        v, desc = oracle_sample(sub, h)
        return {"value": v, "unit": UNIT, "cores": O.get_threads(), "kind": "oracle",
                "sample": "bounded sample of c5_diffusion_32768: " + desc + " (C5 recipe, same D and dt)"}
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
    """The reference arm of this tier: the fp64 CPU oracle, as it stands, with the
    native arm's config; each step a bounded sample (named in cpu_baseline.sample)."""
    if rank != 0:
        return None
    from oracle import oracle as O
    O.set_threads(os.cpu_count() or 1)
    if wl.name.startswith("c5"):
        swl, host = c5_sample_workload(wl)
        prefix = "bounded sample of c5_diffusion_32768: "
    else:
        swl, host = wl, make_inputs(wl)
        prefix = ""
    for _ in range(args.warmup):
        oracle_sample(swl, host, budget_s=2.0)
    vals, descs = [], []
    for _ in range(args.steps):
        v, d = oracle_sample(swl, host, budget_s=8.0)
        vals.append(v)
        descs.append(d)
    value = statistics.median(vals)
    pts_step = wl.points * (wl.nsteps if wl.op != "poisson" else 1)
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pts_step / value * 1e3,
        "higher_is_better": True, "scaling": "strong" if (wl.name.startswith("c5") and world > 1) else "weak",
        "vs_baseline": None, "dtype": "f64" if wl.dtype in ("c128", "f64") else "f32",
        "data": "synthetic (seeded, BASELINE.json recipe)", "config": workload_config(wl, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.get_threads(), "kind": "oracle",
                         "sample": prefix + descs[0] + "; median over steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    from paper_2412_12308_b200 import inputs as I
    wl = I.WORKLOADS.get(args.workload) or I.EXTRA_WORKLOADS[args.workload]
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        line = reference(args, wl, world_env, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    import torch
    world, rank, local = dist_setup()
    assert world == args.gpus, (world, args.gpus)
    if (args.sharded or args.pencil) and world == 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    if wl.name.startswith("c5") and (world > 1 or args.sharded):
        line = sharded_native(args, wl, world, rank, local)
    elif wl.nz > 1 and (world > 1 or args.sharded or args.pencil):
        line = sharded3d_native(args, wl, world, rank, local)
    else:
        line = native(args, wl, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or args.sharded or args.pencil:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
