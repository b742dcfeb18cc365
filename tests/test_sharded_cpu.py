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


# ---------------------------------------------------------------- fused peer-store slab path

class NumpyFusedOps(NumpyLocalOps):
    """Host stand-ins for the fused exchanges (fftpde_rows_to_peers / fftpde_cols_to_peers):
    the pass result is stored straight into the peers' buffers, here shared-memory
    tensors of the other processes (the same element mapping as PeerOut, launch.h)."""

    dtype = torch.complex128
    device = torch.device("cpu")

    def _x_pass(self, a, op, D, dt):
        X = a.shape[1] * np.fft.ifft(a, axis=1)                    # forward along x, + sign
        if op == 0:
            return X
        return np.fft.fft(X * np.exp(-D * self.kx[None, :] ** 2 * dt), axis=1) / self.nx

    def rows_to_peers(self, x, peers, rank, R, op, D=0.0, dt=0.0):
        r = self._x_pass(x.numpy(), op, D, dt)
        bw = self.nx // len(peers)
        for q, buf in enumerate(peers):                            # element a of row k -> rank a / bw, row rank R + k
            buf.numpy()[rank * R:(rank + 1) * R, :] = r[:, q * bw:(q + 1) * bw]

    def cols_to_peers(self, cs, peers, rank, R, op, D=0.0, dt=0.0):
        a = cs.numpy()
        bw = a.shape[1]
        if op == 5:                                                 # y diffusion (R26)
            Y = self.ny * np.fft.ifft(a, axis=0) * np.exp(-D * self.ky[:, None] ** 2 * dt)
            r = np.fft.fft(Y, axis=0) / self.ny
        else:                                                       # Poisson column pass, global kx
            out = torch.empty_like(cs)
            self.cols_slab(cs, out, rank * bw, op, D, dt)
            r = out.numpy()
        for q, buf in enumerate(peers):                             # element y of column c -> rank y / R
            buf.numpy()[:, rank * bw:(rank + 1) * bw] = r[q * R:(q + 1) * R, :]


class SharedPeerComm:
    """Peer 'pointers' are the shared-memory tensors of every rank (alloc order A, Cs);
    the barrier is the process-group barrier."""

    def __init__(self, rank, world, sets):
        self.rank, self.world, self.sets, self.n = rank, world, sets, 0

    def local_ranks(self):
        return [self.rank]

    def alloc(self, shape, dtype, device):
        bufs = self.sets[self.n]
        self.n += 1
        assert tuple(bufs[self.rank].shape) == tuple(shape)
        return [bufs[self.rank]], bufs

    def barrier(self):
        dist.barrier()


def _fused_worker(rank, world, port, nx, ny, D, dt, nsteps, sets, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_12308_b200 import sharded as S
    from paper_2412_12308_b200 import inputs as I
    u0 = I.white_noise((ny, nx), 2413)
    lo, hi = S.slab_rows(ny, world, rank)
    slab = torch.from_numpy(np.ascontiguousarray(u0[lo:hi]))
    solver = S.FusedPeerSlabSolver(nx, ny, SharedPeerComm(rank, world, sets), NumpyFusedOps(nx, ny))
    out = solver.diffuse([slab], D, dt, nsteps)[0]
    gathered = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(gathered, out)
    if rank == 0:
        q.put(torch.cat(gathered).numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_fused_peer_slab_diffusion_two_processes(world):
    # FusedPeerSlabSolver's sequencing (row pass -> peers' column slabs | barrier |
    # column pass -> peers' row slabs | barrier, nsteps times) across two processes
    # whose "peer memory" is shared, against the oracle's single-process solve
    from oracle import oracle as O
    from paper_2412_12308_b200 import inputs as I
    nx, ny, D, dt, nsteps = 64, 32, 1e-3, 0.01, 4
    R, BW = ny // world, nx // world
    sets = [[torch.zeros((R, nx), dtype=torch.complex128).share_memory_() for _ in range(world)],
            [torch.zeros((ny, BW), dtype=torch.complex128).share_memory_() for _ in range(world)]]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, nx, ny, D, dt, nsteps, sets, q))
             for r in range(world)]
    for p in procs:
        p.start()
    u = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    src = I.white_noise((ny, nx), 2413)
    ref = O.diffuse(src, D, dt, nsteps)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-12


def _abi_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes
    from paper_2412_12308_b200 import fftpde as F
    lib = F.load_library()
    uid = F.broadcast_unique_id(lambda: bytes(range(1, 129)))
    buf = ctypes.create_string_buffer(uid, 128)
    h = ctypes.c_void_p()
    st = {}
    # argument checks of the collective plan constructor, per rank, before any CUDA or NCCL call
    st["rank_out_of_range"] = lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, buf, world, world)
    st["negative_rank"] = lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, buf, -1, world)
    st["ranks_not_dividing"] = lib.fftpde_plan_2d_sharded(ctypes.byref(h), 64, 64, 1, 1.0, 1.0, 0, buf, rank, 3)
    st["not_pow2"] = lib.fftpde_plan_2d_sharded(ctypes.byref(h), 48, 64, 1, 1.0, 1.0, 0, buf, rank, world)
    q.put((rank, uid, st, h.value))
    dist.destroy_process_group()


def test_sharded_plan_host_checks_two_processes():
    # the in-library sharded plan's host half on each of two processes: the shared
    # unique id, and the synchronous argument errors that must come back before
    # the constructor touches a device or a communicator
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_abi_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {r: (u, s, h) for r, u, s, h in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0][0] == got[1][0] == bytes(range(1, 129))
    for r in range(world):
        _, s, h = got[r]
        assert s["rank_out_of_range"] == 1 and s["negative_rank"] == 1          # FFTPDE_ERR_INVALID_ARG
        assert s["ranks_not_dividing"] == 5                                      # FFTPDE_ERR_UNSUPPORTED
        assert s["not_pow2"] == 3                                                # FFTPDE_ERR_NOT_POW2_X
        assert h is None                                                         # no plan left behind
