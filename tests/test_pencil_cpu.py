"""Multi-process (gloo, 4 processes on a 2 x 2 grid, CPU) test of the pencil
decomposition's host logic -- the schedule fftpde_plan_3d_pencil runs inside
libfftpde (include/fftpde.h): x-pencils [nz/pz][ny/py][nx],
pack by x-block, all-to-all inside the row group (the py ranks of z-block i),
unpack to the y-pencil [nz/pz][ny][nx/py], pack by y-block of ny/pz, all-to-all
inside the column group (the pz ranks of x-block j), the z-pencil
[nz][ny/pz][nx/py] whose line (yl, xl) is the global line (j nx/py + xl,
i ny/pz + yl), and back.  The block moves are the library's pack semantics
([nrows][P][blk] <-> [P][nrows][blk]) and group routing (block g of rank r to
the group's g-th rank, at r's position in the group), the exchanges are real
torch.distributed all_to_all_single calls on sub-groups; the per-axis
transforms are host stand-ins (numpy, the paper's + sign) -- the CUDA passes
are covered by tests/test_gpu_sharded.py.  The gathered Poisson solve is
compared with the fp64 oracle."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PZ, PY = 2, 2
NZ, NY, NX = 8, 16, 32
L = (1.0, 2.0, 0.5)


def pack(a, nrows, nblocks, blk, direction):
    """The library's pack_blocks: [nrows][P][blk] -> [P][nrows][blk] (0) and back (1)."""
    a = a.reshape(-1)
    if direction == 0:
        return np.ascontiguousarray(a.reshape(nrows, nblocks, blk).transpose(1, 0, 2)).reshape(-1)
    return np.ascontiguousarray(a.reshape(nblocks, nrows, blk).transpose(1, 0, 2)).reshape(-1)


def fwd(a, axis):      # paper forward: X_k = sum_n x_n e^{+2 pi i n k / N}
    return a.shape[axis] * np.fft.ifft(a, axis=axis)


def inv(a, axis):      # unscaled conjugate transform
    return np.fft.fft(a, axis=axis)


def k2(n, Lax):
    m = np.arange(n)
    return (2 * np.pi * np.where(m <= n // 2, m, m - n) / Lax) ** 2


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=PZ * PY)
    i, j = rank // PY, rank % PY
    # every rank creates every group, in the same order
    rows = [dist.new_group([ii * PY + jj for jj in range(PY)]) for ii in range(PZ)]
    cols = [dist.new_group([ii * PY + jj for ii in range(PZ)]) for jj in range(PY)]
    nzl, nyl, nxl, nyl2 = NZ // PZ, NY // PY, NX // PY, NY // PZ
    rng = np.random.default_rng(404)
    x = rng.standard_normal((NZ, NY, NX)) + 1j * rng.standard_normal((NZ, NY, NX))
    xp = x[i * nzl:(i + 1) * nzl, j * nyl:(j + 1) * nyl]           # my x-pencil

    def a2a(buf, group):
        send = torch.from_numpy(np.ascontiguousarray(buf).view(np.float64))
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=group)
        return recv.numpy().view(np.complex128)

    # forward: x-pass, row-group exchange, y-pass, column-group exchange
    A = fwd(xp, 2)
    B = pack(A, nzl * nyl, PY, nxl, 0)
    C = a2a(B, rows[i])
    Yp = pack(C, nzl, PY, nyl * nxl, 1).reshape(nzl, NY, nxl)      # y-pencil of x-block j
    Yp = fwd(Yp, 1)
    D = pack(Yp, nzl, PZ, nyl2 * nxl, 0)
    Zp = a2a(D, cols[j]).reshape(NZ, nyl2, nxl)                    # z-pencil: rows of y-block i
    Zp = fwd(Zp, 0)
    # the multiplier at the global wavenumbers of my lines, -1/|k|^2 / (nx ny nz), k = 0 zeroed
    kk = (k2(NZ, L[2])[:, None, None] + k2(NY, L[1])[None, i * nyl2:(i + 1) * nyl2, None]
          + k2(NX, L[0])[None, None, j * nxl:(j + 1) * nxl])
    m = np.where(kk == 0, 0.0, -1.0 / np.where(kk == 0, 1.0, kk)) / (NX * NY * NZ)
    Zp = inv(Zp * m, 0)
    # back: column-group exchange, y-pass, row-group exchange, x-pass
    E = a2a(Zp, cols[j])
    Yb = pack(E, nzl, PZ, nyl2 * nxl, 1).reshape(nzl, NY, nxl)
    Yb = inv(Yb, 1)
    F_ = pack(Yb, nzl, PY, nyl * nxl, 0)
    G = a2a(F_, rows[i])
    Xb = pack(G, nzl * nyl, PY, nxl, 1).reshape(nzl, nyl, NX)
    u = inv(Xb, 2)
    q.put((rank, u))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_pencil_schedule_poisson_gloo():
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(PZ * PY)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(PZ * PY))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nzl, nyl = NZ // PZ, NY // PY
    u = np.zeros((NZ, NY, NX), complex)
    for r, part in got.items():
        i, j = r // PY, r % PY
        u[i * nzl:(i + 1) * nzl, j * nyl:(j + 1) * nyl] = part
    rng = np.random.default_rng(404)
    x = rng.standard_normal((NZ, NY, NX)) + 1j * rng.standard_normal((NZ, NY, NX))
    ref = O.poisson3(x, *L)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-12
