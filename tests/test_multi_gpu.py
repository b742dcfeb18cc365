"""Real multi-GPU runs of the sharded paths: two
processes, one GPU each, NCCL over NVLink.  Skipped when fewer than two CUDA
devices are visible -- the build box and the round-end GPU tier have one, so
the single-process loopback tests (tests/test_gpu_sharded.py) and the gloo
tests (tests/test_sharded_cpu.py) stand in there.  Each rank computes its slab
or pencil; rank 0 gathers and compares with the fp64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2
needs_two = pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < WORLD,
                               reason="needs two CUDA devices")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _worker(rank, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", rank=rank, world_size=WORLD, device_id=torch.device("cuda", rank))
    from paper_2412_12308_b200 import fftpde as F
    from paper_2412_12308_b200 import sharded as S
    out = {}
    if case == "slab2d":               # NCCL inside the library, row slabs
        nx, ny = 256, 128
        x = _rand((ny, nx), 601)
        R = ny // WORLD
        p = F.ShardedPlan(nx, ny, Lx=1.5, Ly=0.75)
        xs = torch.from_numpy(np.ascontiguousarray(x[rank * R:(rank + 1) * R])).cuda()
        out["diffuse"] = p.diffuse(xs, 2e-4, 0.01, 3).cpu().numpy()
        out["poisson"] = p.poisson(xs).cpu().numpy()
    elif case == "fused":              # the row / column epilogues store into the peer's slab
        nx, ny = 256, 128
        x = _rand((ny, nx), 602)
        R = ny // WORLD
        ops = S.CudaLocalOps(nx, ny, Lx=1.5, Ly=0.75)
        solver = S.FusedPeerSlabSolver(nx, ny, S.SymmetricPeerComm(), ops)
        xs = torch.from_numpy(np.ascontiguousarray(x[rank * R:(rank + 1) * R])).cuda()
        out["diffuse"] = solver.diffuse([xs], 2e-4, 0.01, 3)[0].cpu().numpy()
        out["poisson"] = solver.poisson([xs])[0].cpu().numpy()
    elif case.startswith("pencil"):    # pz x py = 1 x 2 or 2 x 1
        pz, py = (1, 2) if case == "pencil12" else (2, 1)
        nz, ny, nx = 16, 64, 32
        x = _rand((nz, ny, nx), 603)
        i, j = rank // py, rank % py
        nzl, nyl = nz // pz, ny // py
        p = F.PencilPlan3D(nx, ny, nz, pz, py, Lx=1.0, Ly=2.0, Lz=0.5)
        xp = torch.from_numpy(np.ascontiguousarray(x[i * nzl:(i + 1) * nzl, j * nyl:(j + 1) * nyl])).cuda()
        out["poisson"] = p.poisson(xp).cpu().numpy()
        out["spectrum"] = p.forward(xp).cpu().numpy()
    elif case in ("c5lib", "c5fs"):    # the distributed four-step (R28) at C5's grid, rank-2 input
        n, D, dt, steps = 32768, 1e-4, 0.01, 3
        f1, g1, f2, g2 = (torch.from_numpy(_rand((n,), 620 + k)).cuda() for k in range(4))
        R = n // WORLD
        slab = (torch.outer(g1[rank * R:(rank + 1) * R], f1) + torch.outer(g2[rank * R:(rank + 1) * R], f2))
        if case == "c5lib":            # NCCL all-to-all inside the library
            u = F.ShardedPlan(n, n).diffuse(slab, D, dt, steps)
        else:                          # the exchange fused into the B passes (symmetric memory)
            plan = F.Plan(n, n)
            u = S.FusedFourStepSolver(n, S.SymmetricPeerComm(), plan).diffuse([slab], D, dt, steps)[0]
        torch.cuda.synchronize()
        out["rows"] = u[::1021].cpu().numpy()          # every 1021st row of the slab
        out["row0"] = rank * R
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _run(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, case, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@needs_two
@pytest.mark.parametrize("case", ["slab2d", "fused"])
def test_two_gpu_slab_vs_oracle(case):
    from oracle import oracle as O
    res = _run(case)
    nx, ny = 256, 128
    x = _rand((ny, nx), 601 if case == "slab2d" else 602)
    u = np.concatenate([res[r]["diffuse"] for r in range(WORLD)])
    p = np.concatenate([res[r]["poisson"] for r in range(WORLD)])
    assert rel(u, O.diffuse(x, 2e-4, 0.01, 3, 1.5, 0.75)) <= 1e-12
    assert rel(p, O.poisson(x, 1.5, 0.75)) <= 1e-12


@needs_two
@pytest.mark.parametrize("case", ["pencil12", "pencil21"])
def test_two_gpu_pencil_vs_oracle(case):
    from oracle import oracle as O
    res = _run(case)
    pz, py = (1, 2) if case == "pencil12" else (2, 1)
    nz, ny, nx = 16, 64, 32
    x = _rand((nz, ny, nx), 603)
    # x-pencils of rank i py + j back into [nz][ny][nx]
    pois = np.zeros((nz, ny, nx), complex)
    spec = np.zeros((nz, ny, nx), complex)
    for r in range(WORLD):
        i, j = r // py, r % py
        nzl, nyl = nz // pz, ny // py
        pois[i * nzl:(i + 1) * nzl, j * nyl:(j + 1) * nyl] = res[r]["poisson"]
        nyl2, nxl = ny // pz, nx // py
        spec[:, i * nyl2:(i + 1) * nyl2, j * nxl:(j + 1) * nxl] = res[r]["spectrum"]
    assert rel(pois, O.poisson3(x, 1.0, 2.0, 0.5)) <= 1e-12
    assert rel(spec, O.fft3(x)) <= 1e-12


@needs_two
@pytest.mark.parametrize("case", ["c5lib", "c5fs"])
def test_two_gpu_c5_distributed_fourstep_vs_oracle(case):
    # R28 on two GPUs: rank-2 separable input, the oracle's stepped 1D solves at
    # sampled rows of both slabs (every point of each sampled row)
    from oracle import oracle as O
    res = _run(case)
    n, D, dt, steps = 32768, 1e-4, 0.01, 3
    f1, g1, f2, g2 = (_rand((n,), 620 + k) for k in range(4))
    Df1, Dg1, Df2, Dg2 = (O.diffuse(v.reshape(1, n), D, dt, steps).ravel() for v in (f1, g1, f2, g2))
    for r in range(WORLD):
        rows = res[r]["row0"] + np.arange(0, n // WORLD, 1021)
        ref = np.outer(Dg1[rows], Df1) + np.outer(Dg2[rows], Df2)
        assert rel(res[r]["rows"], ref) <= 1e-12, r
