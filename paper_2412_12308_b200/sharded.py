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

    def peer_transpose(self, src, peers, rank, R, bw, direction):
        return self.plan.peer_transpose(src, peers, rank, R, bw, direction)

    def rows_to_peers(self, x, peers, rank, R, op, D=0.0, dt=0.0):
        return self.plan.rows_to_peers(x, peers, rank, R, op, D, dt)

    def cols_to_peers(self, cs, peers, rank, R, op, D=0.0, dt=0.0):
        return self.plan.cols_to_peers(cs, peers, rank, R, op, D, dt)

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


class LoopbackPeerComm:
    """P virtual ranks in one process for the peer-store exchange: every rank's
    buffers live on this device, so a "peer store" is a store into another
    virtual rank's buffer; the phases are ordered by the single stream."""

    def __init__(self, world):
        self.world = world

    def local_ranks(self):
        return list(range(self.world))

    def alloc(self, shape, dtype, device):
        bufs = [torch.empty(shape, dtype=dtype, device=device) for _ in range(self.world)]
        return bufs, [b.data_ptr() for b in bufs]

    def barrier(self):
        pass


class SymmetricPeerComm:
    """One rank per GPU: buffers from torch symmetric memory (peer-mapped over
    NVLink), barrier = the symmetric-memory stream-ordered device barrier.

    Ordering of the fused exchanges: the row / column pass kernels write the
    peers' buffers with plain global stores to peer-mapped addresses; the barrier
    kernel is enqueued after them on the same stream, so it starts only once every
    one of those stores has been performed (kernel boundary).  torch's barrier
    kernel then signals each peer with a compare-and-swap at system scope with
    release semantics (``put_signal<memory_order_release>`` on a
    ``cuda::atomic_ref<.., thread_scope_system>``, CUDASymmetricMemory-inl.h) and
    waits on its own pad with an acquire CAS at system scope, so a peer's kernels
    enqueued after its barrier observe our stores (the same "writes of previous
    kernels are visible" pattern torch's own symmetric-memory kernels use).  The
    multi-rank path has been exercised by the single-process emulation on one
    GPU and by the two-process gloo test with shared-memory stand-ins
    (tests/test_sharded_cpu.py); it has not run on real multi-GPU hardware."""

    def __init__(self, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.dist, self.symm = dist, symm
        self.group = group if group is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        self._handles = []

    def local_ranks(self):
        return [self.rank]

    def alloc(self, shape, dtype, device):
        t = self.symm.empty(*shape, dtype=dtype, device=device)
        h = self.symm.rendezvous(t, self.group)
        self._handles.append(h)
        return [t], list(h.buffer_ptrs)

    def barrier(self):
        self._handles[0].barrier(channel=0)


class PeerSlabSolver:
    """The slab decomposition with the exchange done by peer stores
    (fftpde_peer_transpose) instead of pack + all-to-all: per step
        rows forward            row slab -> A (local)
        peer transpose 0        A -> every rank's column slab Cs     | barrier
        column pass             Cs in place (global wavenumbers)
        peer transpose 1        Cs -> every rank's A                 | barrier
        rows inverse            A -> the output row slab
    Two barriers and no pack passes per step."""

    def __init__(self, nx, ny, comm, ops):
        self.comm = comm
        self.P = comm.world
        if ny % self.P or nx % self.P:
            raise ValueError("the rank count must divide nx and ny")
        self.nx, self.ny = nx, ny
        self.R, self.BW = ny // self.P, nx // self.P
        self.ops = ops
        self.ranks = comm.local_ranks()
        self.A, self.A_ptrs = comm.alloc((self.R, nx), ops.dtype, ops.device)
        self.Cs, self.Cs_ptrs = comm.alloc((ny, self.BW), ops.dtype, ops.device)

    def _step(self, srcs, dsts, op, D, dt):
        ops, R, BW = self.ops, self.R, self.BW
        for i, r in enumerate(self.ranks):
            ops.rows(srcs[i], self.A[i], False)
            ops.peer_transpose(self.A[i], self.Cs_ptrs, r, R, BW, 0)
        self.comm.barrier()
        for i, r in enumerate(self.ranks):
            ops.cols_slab(self.Cs[i], self.Cs[i], r * BW, op, D, dt)
            ops.peer_transpose(self.Cs[i], self.A_ptrs, r, R, BW, 1)
        self.comm.barrier()
        for i, _ in enumerate(self.ranks):
            ops.rows(self.A[i], dsts[i], True)

    diffuse = SlabSolver.diffuse
    poisson = SlabSolver.poisson


class FusedPeerSlabSolver(PeerSlabSolver):
    """The peer-store slab decomposition with both exchanges fused into the passes
    (SURVEY.md 8(e) N10): the row pass stores each output row straight into the
    owners' column slabs (fftpde_rows_to_peers) and the column pass stores each
    output column straight back into the owners' row slabs (fftpde_cols_to_peers).
    Diffusion per step, in the separable form (R26):
        rows: x diffusion -> peers' column slabs Cs    | barrier
        columns: y diffusion -> peers' row slabs A     | barrier
    A holds the materialised field after every step; the next step's row pass
    reads it, the last one is copied to the output slab.  Poisson: forward rows
    -> peers, column pass (-1/|k|^2) -> peers, inverse rows."""

    def diffuse(self, slabs, D, dt, nsteps, outs=None):
        from . import fftpde as F
        ops, R, BW = self.ops, self.R, self.BW
        outs = outs if outs is not None else [ops.empty(s.shape) for s in slabs]
        if nsteps == 0:
            for s, o in zip(slabs, outs):
                o.copy_(s)
            return outs
        for k in range(nsteps):
            for i, r in enumerate(self.ranks):
                ops.rows_to_peers(slabs[i] if k == 0 else self.A[i], self.Cs_ptrs, r, R, F.ROWS_DIFFUSE, D, dt)
            self.comm.barrier()
            for i, r in enumerate(self.ranks):
                ops.cols_to_peers(self.Cs[i], self.A_ptrs, r, R, F.OP_DIFFUSE_Y, D, dt)
            self.comm.barrier()
        for i, _ in enumerate(self.ranks):
            outs[i].copy_(self.A[i])
        return outs

    def poisson(self, slabs, outs=None):
        from . import fftpde as F
        ops, R, BW = self.ops, self.R, self.BW
        outs = outs if outs is not None else [ops.empty(s.shape) for s in slabs]
        for i, r in enumerate(self.ranks):
            ops.rows_to_peers(slabs[i], self.Cs_ptrs, r, R, F.ROWS_FWD)
        self.comm.barrier()
        for i, r in enumerate(self.ranks):
            ops.cols_to_peers(self.Cs[i], self.A_ptrs, r, R, F.OP_POISSON)
        self.comm.barrier()
        for i, _ in enumerate(self.ranks):
            ops.rows(self.A[i], outs[i], True)
        return outs


class FusedFourStepSolver:
    """C5 (32768^2 complex128 diffusion) on P ranks with the distributed four-step
    (R28) and the Y-part <-> X-part exchange fused into the B passes: the
    pass that ends in one part stores its tiles straight into every peer's other
    part over NVLink (fftpde_fs_part_b with peers), so each step is
        B pass -> peers' other part | barrier | other B pass (in place) | MID
    with one barrier and no separate exchange; the parts alternate step by step.
    The caller's row slabs enter and leave through fftpde_fs_part_perm, a block
    all-to-all by peer stores and a block swap.  comm: LoopbackPeerComm (P virtual
    ranks on one device) or SymmetricPeerComm (one rank per GPU)."""

    def __init__(self, n, comm, plan):
        self.comm, self.plan = comm, plan
        self.P = comm.world
        self.n = n
        self.ranks = comm.local_ranks()
        elems = n * n // self.P
        dev, dt = plan.device, plan.dtype
        self.Wy, self.Wy_ptrs = comm.alloc((elems,), dt, dev)     # Y-parts (peer-mapped: By stores into them)
        self.Wx, self.Wx_ptrs = comm.alloc((elems,), dt, dev)     # X-parts (Bx stores into them)
        self.T1, self.T1_ptrs = comm.alloc((elems,), dt, dev)     # receive buffer of the conversions
        self.T2 = [torch.empty(elems, dtype=dt, device=dev) for _ in self.ranks]   # physical field / send buffer

    def _swap(self, i, src, dst):
        P = self.P
        self.plan.pack_blocks(src, dst, P, P, src.numel() // (P * P), 0)

    def diffuse(self, slabs, D, dt, nsteps, outs=None):
        pl, P = self.plan, self.P
        outs = outs if outs is not None else [torch.empty_like(s) for s in slabs]
        if nsteps == 0:
            for s, o in zip(slabs, outs):
                o.copy_(s)
            return outs
        L = range(len(self.ranks))
        self.comm.barrier()                                  # the peers are done with the last solve's buffers
        for i in L:                                          # row slab -> Y-part
            pl.fs_part_perm(P, slabs[i].view(-1), self.T2[i], 0)
            pl.peer_blocks(self.T2[i], self.T1_ptrs, self.ranks[i])
        self.comm.barrier()
        for i in L:
            self._swap(i, self.T1[i], self.Wy[i])
            pl.fs_part_aa(0, P, self.ranks[i], 0, self.Wy[i], self.Wy[i])
        x = 0
        for k in range(nsteps):
            W = self.Wx if x else self.Wy
            for i, r in zip(L, self.ranks):                  # B pass of this part -> the peers' other part
                pl.fs_part_b(x, P, r, W[i], D, dt, peers=self.Wy_ptrs if x else self.Wx_ptrs)
            self.comm.barrier()
            x ^= 1
            W = self.Wx if x else self.Wy
            for i, r in zip(L, self.ranks):
                pl.fs_part_b(x, P, r, W[i], D, dt)
                if k + 1 < nsteps:
                    pl.fs_part_aa(2, P, r, x, W[i], W[i], self.T2[i])
                else:
                    pl.fs_part_aa(1, P, r, x, W[i], self.T2[i])
        # the physical field (T2, part x) -> Y-part -> row slabs
        if x:
            for i, r in zip(L, self.ranks):
                pl.peer_blocks(self.T2[i], self.T1_ptrs, r)
            self.comm.barrier()
            src = self.T1
        else:
            src = self.T2
        for i in L:
            self._swap(i, src[i], self.Wx[i])
        self.comm.barrier()                                  # every rank has read its T1
        for i, r in zip(L, self.ranks):
            pl.peer_blocks(self.Wx[i], self.T1_ptrs, r)
        self.comm.barrier()
        for i in L:
            pl.fs_part_perm(P, self.T1[i], outs[i].view(-1), 1)
        return outs


def slab_rows(ny, world, rank):
    """Rows [lo, hi) of rank `rank` (SURVEY.md 8(b) sharded plans)."""
    R = ny // world
    return rank * R, (rank + 1) * R
