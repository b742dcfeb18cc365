"""Multi-process (gloo, world_size 2, CPU) test of the slab decomposition's
host logic: row slabs, per-peer block packing, the two all-to-alls, and the
global-wavenumber column pass.  The per-rank arithmetic runs on host stand-ins
(numpy, paper sign conventions) -- the CUDA kernels need a GPU and are covered
by tests/test_gpu_sharded.py -- and the gathered result is compared with the
fp64 oracle's single-process solve."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class NumpyLocalOps:
    """Host stand-ins with the same contract as sharded.CudaLocalOps."""

    def __init__(self, nx, ny, Lx=1.0, Ly=1.0):
        self.nx, self.ny, self.Lx, self.Ly = nx, ny, Lx, Ly
        f = lambda n, L: 2 * np.pi * np.where(np.arange(n) <= n // 2, np.arange(n), np.arange(n) - n) / L
        self.kx, self.ky = f(nx, Lx), f(ny, Ly)

    def empty(self, shape):
        return torch.empty(shape, dtype=torch.complex128)

    def rows(self, x, out, inverse):
        a = x.numpy()
        r = np.fft.fft(a, axis=1) if inverse else a.shape[1] * np.fft.ifft(a, axis=1)
        out.copy_(torch.from_numpy(r))
        return out

    def cols_slab(self, x, out, col0, op, D, dt):
        a = x.numpy()
        ny, nc = a.shape
        X = ny * np.fft.ifft(a, axis=0)                      # forward along y, + sign
        k2 = self.ky[:, None] ** 2 + self.kx[None, col0:col0 + nc] ** 2
        scale = 1.0 / (self.nx * self.ny)
        if op == 2:
            m = np.where(k2 == 0, 0.0, -1.0 / np.where(k2 == 0, 1.0, k2)) * scale
        else:
            m = np.exp(-D * k2 * dt) * scale
        out.copy_(torch.from_numpy(np.fft.fft(X * m, axis=0)))  # unscaled inverse along y
        return out

    def pack(self, x, out, nrows, nblocks, bw, direction):
        a = x.reshape(-1).numpy()
        if direction == 0:
            r = a.reshape(nrows, nblocks, bw).transpose(1, 0, 2)
        else:
            r = a.reshape(nblocks, nrows, bw).transpose(1, 0, 2)
        out.view(-1).copy_(torch.from_numpy(np.ascontiguousarray(r).reshape(-1)))
        return out


def _worker(rank, world, port, nx, ny, D, dt, nsteps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_12308_b200 import sharded as S
    from paper_2412_12308_b200 import inputs as I
    u0 = I.white_noise((ny, nx), 2412)
    lo, hi = S.slab_rows(ny, world, rank)
    slab = torch.from_numpy(np.ascontiguousarray(u0[lo:hi]))
    solver = S.SlabSolver(nx, ny, S.DistComm(), NumpyLocalOps(nx, ny))
    out = solver.diffuse([slab], D, dt, nsteps)[0]
    pois = solver.poisson([slab])[0]
    gathered = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(gathered, out)
    gp = [torch.empty_like(pois) for _ in range(world)]
    dist.all_gather(gp, pois)
    if rank == 0:
        q.put((torch.cat(gathered).numpy(), torch.cat(gp).numpy()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_slab_diffusion_and_poisson_gloo(world):
    from oracle import oracle as O
    from paper_2412_12308_b200 import inputs as I
    nx, ny, D, dt, nsteps = 64, 32, 1e-3, 0.01, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, ny, D, dt, nsteps, q)) for r in range(world)]
    for p in procs:
        p.start()
    u, pois = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    src = I.white_noise((ny, nx), 2412)
    ref = O.diffuse(src, D, dt, nsteps)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-12
    refp = O.poisson(src)
    assert np.linalg.norm(pois - refp) / np.linalg.norm(refp) <= 1e-12


def _uid_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_12308_b200 import fftpde as F

    def draw():
        if dist.get_rank() != 0:
            raise AssertionError("only rank 0 draws the NCCL unique id")
        return bytes(range(128))

    uid = F.broadcast_unique_id(draw)
    q.put((rank, uid))
    dist.destroy_process_group()


def test_nccl_unique_id_broadcast_gloo():
    # the host half of fftpde_plan_2d_sharded / _3d_sharded set-up: rank 0 draws the
    # 128-byte id, every rank receives the same bytes over the process group
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] == bytes(range(128))
