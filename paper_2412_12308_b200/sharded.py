"""Slab-decomposed multi-GPU solves (BASELINE.json configs[4]).

Rank r of P owns the row slab [r ny/P, (r+1) ny/P) of every field.  One exact
diffusion step (ec:solCalorFourier) -- or one Poisson solve
(eq:SolutionPoisson) -- is

    rows forward on the row slab [R][nx]                    (libfftpde kernels)
    pack into per-peer blocks [P][R][nx/P]                  (libfftpde kernel)
    all-to-all  -> column slab [ny][nx/P]                   (NCCL over NVLink)
    column pass: forward along y, multiplier at the global
        wavenumbers, inverse along y                         (libfftpde kernels)
    all-to-all  -> per-peer blocks of the row slab          (NCCL)
    unpack + inverse rows -> the physical row slab           (libfftpde kernels)

two all-to-alls per step, as the row/column split of the 2D DFT
 requires.  The exchange is torch.distributed
(``all_to_all_single``); every arithmetic step is a libfftpde kernel
(``CudaLocalOps``).  ``LoopbackComm`` runs P virtual ranks in one process on
one GPU (the exchange becomes block copies) so the layout logic is testable
without a multi-GPU box; the multi-process path is covered by gloo tests with
host stand-ins for the local kernels (tests/test_sharded_cpu.py).
"""
from __future__ import annotations

import torch

from . import fftpde as F


class CudaLocalOps:
    """The per-rank arithmetic: libfftpde kernels on the rank's GPU (no fallback)."""

    def __init__(self, nx, ny, dtype=torch.complex128, Lx=1.0, Ly=1.0, device=None):
        self.plan = F.Plan(nx, ny, batch=1, dtype=dtype, Lx=Lx, Ly=Ly, device=device)
        self.device = self.plan.device
        self.dtype = dtype

    def empty(self, shape):
        return torch.empty(shape, dtype=self.dtype, device=self.device)

    def rows(self, x, out, inverse):
        return self.plan.rows(x, out, inverse)

    def cols_slab(self, x, out, col0, op, D, dt):
        return self.plan.cols_slab(x, out, col0, op, D, dt)

    def pack(self, x, out, nrows, nblocks, bw, direction):
        return self.plan.pack_blocks(x, out, nrows, nblocks, bw, direction)

    @property
    def launches(self):
        return self.plan.launches


class DistComm:
    """all-to-all over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def local_ranks(self):
        return [self.rank]

    def exchange(self, outs, ins):
        # one local rank: [P][...] blocks, block q goes to rank q
        self.dist.all_to_all_single(outs[0], ins[0], group=self.group)


class LoopbackComm:
    """P virtual ranks in one process (test harness for the layout logic)."""

    def __init__(self, world):
        self.world = world

    def local_ranks(self):
        return list(range(self.world))

    def exchange(self, outs, ins):
        P = self.world
        for r in range(P):
            src_blocks = [ins[q].view(P, -1)[r] for q in range(P)]
            outs[r].view(P, -1).copy_(torch.stack(src_blocks))


class SlabSolver:
    """Sharded Poisson / diffusion on a periodic nx x ny grid, rows split over P ranks."""

    def __init__(self, nx, ny, comm, ops):
        self.comm = comm
        self.P = comm.world
        if ny % self.P or nx % self.P:
            raise ValueError("the rank count must divide nx and ny")
        self.nx, self.ny = nx, ny
        self.R = ny // self.P           # rows per rank
        self.BW = nx // self.P          # columns per rank after the transpose
        self.ops = ops                  # one CudaLocalOps (shared by the local ranks)
        self.ranks = comm.local_ranks()
        n = self.R * nx
        self._A = [ops.empty((self.R, nx)) for _ in self.ranks]
        self._B = [ops.empty((n,)) for _ in self.ranks]
        self._C = [ops.empty((n,)) for _ in self.ranks]

    def _step(self, srcs, dsts, op, D, dt):
        P, R, BW, nx, ny = self.P, self.R, self.BW, self.nx, self.ny
        ops = self.ops
        for i, _ in enumerate(self.ranks):
            ops.rows(srcs[i], self._A[i], False)                         # rows forward
            ops.pack(self._A[i], self._B[i], R, P, BW, 0)                  # [R][P][BW] -> [P][R][BW]
        self.comm.exchange(self._C, self._B)                               # -> column slab [ny][BW]
        for i, r in enumerate(self.ranks):
            c = self._C[i].view(ny, BW)
            ops.cols_slab(c, c, r * BW, op, D, dt)                         # y: fwd, multiplier, inv
        self.comm.exchange(self._B, self._C)                               # -> blocks of the row slab
        for i, _ in enumerate(self.ranks):
            ops.pack(self._B[i], self._A[i], R, P, BW, 1)                  # [P][R][BW] -> [R][nx]
            ops.rows(self._A[i], dsts[i], True)                            # rows inverse

    def diffuse(self, slabs, D, dt, nsteps, outs=None):
        """nsteps exact diffusion steps of the local row slabs (list, one per local rank)."""
        outs = outs if outs is not None else [torch.empty_like(s) for s in slabs]
        if nsteps == 0:
            for o, s in zip(outs, slabs):
                o.copy_(s)
            return outs
        src = slabs
        for _ in range(nsteps):
            self._step(src, outs, F.OP_DIFFUSE, D, dt)
            src = outs
        return outs

    def poisson(self, slabs, outs=None):
        outs = outs if outs is not None else [torch.empty_like(s) for s in slabs]
        self._step(slabs, outs, F.OP_POISSON, 0.0, 0.0)
        return outs


def slab_rows(ny, world, rank):
    """Rows [lo, hi) of rank `rank` (SURVEY.md 8(b) sharded plans)."""
    R = ny // world
    return rank * R, (rank + 1) * R
