"""Host logic of the distributed four-step (R28) on CPU: a numpy model
of every data movement the CUDA path does -- the row-slab -> Y-part permutation
(pack.cu fs_perm_kernel), the block swap (launch_pack), the Y-part <-> X-part
all-to-all (Passes::exchange), the parts' 5D layout [blk][Q][M][Q][M] with the
global m1 / n1 of each tile (fourstep.cuh fs_tile), the Bx line gather over the
blocks q and the By line gather over the blocks r (b3_kernel DIST), the
alternating parts and the exit conversion (Passes::diffuse_fsd) -- at a small
split N = Pf x Qf, with numpy FFTs standing in for the kernels' DFTs.  Two
processes over gloo (world_size 2, real all_to_all_single) and in-process
loopback at P = 1 / 4, against the fp64 oracle's stepped diffusion."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PF, QF = 16, 8                      # the four-step split N = PF QF (the CUDA path: 1024 x 32)
N = PF * QF


def kvec(n, L=1.0):
    a = np.arange(n)
    return 2 * np.pi * np.where(a <= n // 2, a, a - n) / L


class Rank:
    """One rank's passes; `a2a(blocks)` sends blocks[q] to rank q, returns the received [P] blocks."""

    def __init__(self, rank, P, a2a, D, dt):
        self.r, self.P, self.a2a = rank, P, a2a
        self.M, self.T = PF // P, QF // P
        k2 = kvec(N) ** 2
        self.fac = np.exp(-D * k2 * dt)                       # both axes (Lx = Ly = 1)
        self.w = np.exp(-2j * np.pi / N)

    def shape5(self):
        return (self.P, QF, self.M, QF, self.M)

    # row slab [T][P][M][Q][P][M] (m2_l, r, m1_l, n2, q, n1_l) <-> [P][P][T][M][Q][M] (r, q, m2_l, m1_l, n2, n1_l)
    def perm(self, a, direction):
        P, M, T = self.P, self.M, self.T
        if direction == 0:
            return a.reshape(T, P, M, QF, P, M).transpose(1, 4, 0, 2, 3, 5).copy()
        return a.reshape(P, P, T, M, QF, M).transpose(2, 0, 3, 4, 1, 5).copy()

    def swap(self, a):                                        # [P][P][X] -> first two indices swapped
        return a.reshape(self.P, self.P, -1).transpose(1, 0, 2).copy()

    def exchange(self, a):
        return np.stack(self.a2a(list(a.reshape(self.P, -1)))).reshape(self.shape5())

    def globals_(self, xmode):
        b = np.arange(self.P)[:, None, None, None, None]
        l = np.arange(self.M)
        m1 = (b * self.M + l[None, None, :, None, None]) if xmode else (self.r * self.M + l)[None, None, :, None, None]
        n1 = (self.r * self.M + l)[None, None, None, None, :] if xmode else b * self.M + l[None, None, None, None, :]
        return m1, n1

    def aa(self, G, xmode, inverse):
        m1, n1 = self.globals_(xmode)
        kk = np.arange(QF)
        twx = self.w ** (n1 * kk[None, None, None, :, None])   # w_N^{n1 k1}
        twy = self.w ** (m1 * kk[None, :, None, None, None])   # w_N^{m1 l1}
        if not inverse:
            G = np.fft.fft(G, axis=3) * twx
            return np.fft.fft(G, axis=1) * twy
        G = np.fft.ifft(G * np.conj(twy), axis=1)
        return np.fft.ifft(G * np.conj(twx), axis=3)

    def bpass(self, G, xmode):
        P, M = self.P, self.M
        kk = np.arange(QF)[:, None] + QF * np.arange(PF)[None, :]   # wavenumber index k1 + Q k2
        f = self.fac[kk]                                            # [k1][k2]
        if not xmode:     # Bx: lines over n1 = q M + n1_l, class k1 (axis 3)
            L = G.transpose(1, 2, 3, 0, 4).reshape(QF, M, QF, P * M)
            L = np.fft.ifft(np.fft.fft(L, axis=3) * f[None, None, :, :], axis=3)
            return L.reshape(QF, M, QF, P, M).transpose(3, 0, 1, 2, 4).copy()
        # By: lines over m1 = r M + m1_l, class l1 (axis 1)
        L = G.transpose(1, 3, 4, 0, 2).reshape(QF, QF, M, P * M)
        L = np.fft.ifft(np.fft.fft(L, axis=3) * f[:, None, None, :], axis=3)
        return L.reshape(QF, QF, M, P, M).transpose(3, 0, 4, 1, 2).copy()

    def diffuse(self, slab, nsteps):
        """Passes::diffuse_fsd on this rank's row slab [N/P][N]."""
        one = self.P == 1
        if one:
            G = slab.reshape(self.shape5())
        else:
            G = self.swap(self.exchange(self.perm(slab, 0))).reshape(self.shape5())
        G = self.aa(G, 0, False)
        x = 0
        for _ in range(nsteps):
            G = self.bpass(G, x)
            if not one:
                G = self.exchange(G)
            x ^= 1
            G = self.bpass(G, x)
            G = self.aa(G, x, True)          # AA^-1 (the physical field of this step) ...
            phys = G
            G = self.aa(G, x, False)         # ... and the next step's AA (MID)
        if one:
            return phys.reshape(slab.shape)
        if x:
            phys = self.exchange(phys)
        return self.perm(self.exchange(self.swap(phys)), 1).reshape(slab.shape)


def run_loopback(u0, P, D, dt, nsteps):
    # drive the P model ranks step by step with a shared block table
    import threading
    barrier = threading.Barrier(P)
    table = {}
    outs = [None] * P

    def a2a_for(r):
        def a2a(blocks):
            table[r] = blocks
            barrier.wait()
            got = [table[q][r] for q in range(P)]
            barrier.wait()
            return got
        return a2a

    R = N // P

    def work(r):
        outs[r] = Rank(r, P, a2a_for(r), D, dt).diffuse(u0[r * R:(r + 1) * R].copy(), nsteps)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return np.concatenate(outs)


def u0_field():
    rng = np.random.default_rng(2412)
    return rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("nsteps", [1, 2, 3])
def test_fsd_model_loopback_vs_oracle(P, nsteps):
    from oracle import oracle as O
    D, dt = 2e-5, 0.01
    u0 = u0_field()
    u = run_loopback(u0, P, D, dt, nsteps)
    ref = O.diffuse(u0, D, dt, nsteps)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-12


def _worker(rank, world, port, nsteps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def a2a(blocks):
            ins = torch.from_numpy(np.ascontiguousarray(np.stack(blocks)))
            outs = torch.empty_like(ins)
            dist.all_to_all_single(outs, ins)
            return list(outs.numpy())

        u0 = u0_field()
        R = N // world
        u = Rank(rank, world, a2a, 2e-5, 0.01).diffuse(u0[rank * R:(rank + 1) * R].copy(), nsteps)
        parts = [torch.empty(R, N, dtype=torch.complex128) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(u))
        if rank == 0:
            q.put(torch.cat(parts).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nsteps", [2, 3])
def test_fsd_model_gloo_two_processes_vs_oracle(nsteps):
    from oracle import oracle as O
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nsteps, q)) for r in range(2)]
    for p in procs:
        p.start()
    u = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u0 = u0_field()
    ref = O.diffuse(u0, 2e-5, 0.01, nsteps)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-12
