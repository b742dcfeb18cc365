"""Slab decomposition on one GPU with P virtual ranks: the libfftpde row /
column-slab / pack kernels with the sharded layouts (LoopbackComm: the exchange
is a block copy), and the peer-store exchange kernel (LoopbackPeerComm: every
virtual rank's buffers on this device), against the fp64 oracle.  The
multi-process NCCL path uses the same SlabSolver with DistComm (gloo-tested on
CPU); the multi-GPU peer path uses SymmetricPeerComm (torch symmetric memory)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_12308_b200 import inputs as I
from paper_2412_12308_b200 import sharded as S

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def run(nx, ny, P, dtype, x, D, dt, nsteps, Lx=1.0, Ly=1.0, peer=False, fused=False):
    ops = S.CudaLocalOps(nx, ny, dtype=dtype, Lx=Lx, Ly=Ly)
    if fused:    # first exchange fused into the row pass (fftpde_rows_to_peers)
        solver = S.FusedPeerSlabSolver(nx, ny, S.LoopbackPeerComm(P), ops)
    elif peer:   # exchange by peer stores (fftpde_peer_transpose), P virtual ranks on one device
        solver = S.PeerSlabSolver(nx, ny, S.LoopbackPeerComm(P), ops)
    else:
        solver = S.SlabSolver(nx, ny, S.LoopbackComm(P), ops)
    xt = torch.from_numpy(x).to(dtype).cuda()
    R = ny // P
    slabs = [xt[r * R:(r + 1) * R].contiguous() for r in range(P)]
    u = torch.cat(solver.diffuse(slabs, D, dt, nsteps))
    p = torch.cat(solver.poisson(slabs))
    torch.cuda.synchronize()
    return u.cpu().numpy(), p.cpu().numpy()


@pytest.mark.parametrize("dtype,tol", [(torch.complex128, 1e-12), (torch.complex64, 1e-5)])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_slab_diffusion_poisson_vs_oracle(dtype, tol, P):
    nx, ny, D, dt, n = 256, 128, 2e-4, 0.01, 4
    x = I.white_noise((ny, nx), 99)
    u, p = run(nx, ny, P, dtype, x, D, dt, n, Lx=1.5, Ly=0.75)
    assert rel(u, O.diffuse(x, D, dt, n, 1.5, 0.75)) <= tol
    assert rel(p, O.poisson(x, 1.5, 0.75)) <= tol


def test_slab_results_independent_of_rank_count():
    # the per-element arithmetic does not depend on the slab layout: bitwise equal
    nx, ny = 512, 256
    x = I.white_noise((ny, nx), 7)
    outs = [run(nx, ny, P, torch.complex128, x, 1e-4, 0.01, 3) for P in (1, 2, 4, 8)]
    for u, p in outs[1:]:
        assert np.array_equal(u, outs[0][0]) and np.array_equal(p, outs[0][1])


def test_slab_long_axes_c5_shape_sampled():
    # C5 geometry at reduced size on P = 4 virtual ranks: 32768 x 32 rows (two-level rows)
    nx, ny, P = 32768, 64, 4
    x = I.white_noise((ny, nx), 5)
    u, p = run(nx, ny, P, torch.complex128, x, 1e-9, 0.01, 2)
    assert rel(u, O.diffuse(x, 1e-9, 0.01, 2)) <= 1e-12
    # and long columns: 64 x 32768 on P = 8 (column slabs of 8 columns, two-level columns)
    nx, ny, P = 64, 32768, 8
    x = I.white_noise((ny, nx), 6)
    u, p = run(nx, ny, P, torch.complex128, x, 1e-9, 0.01, 2)
    assert rel(u, O.diffuse(x, 1e-9, 0.01, 2)) <= 1e-12


@pytest.mark.parametrize("dtype,tol", [(torch.complex128, 1e-12), (torch.complex64, 1e-5)])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_peer_store_exchange_vs_oracle_and_pack_path(dtype, tol, P):
    # the fused exchange gives bit-for-bit the pack + all-to-all result
    nx, ny, D, dt, n = 256, 128, 2e-4, 0.01, 3
    x = I.white_noise((ny, nx), 101)
    u, p = run(nx, ny, P, dtype, x, D, dt, n, Lx=1.5, Ly=0.75, peer=True)
    assert rel(u, O.diffuse(x, D, dt, n, 1.5, 0.75)) <= tol
    assert rel(p, O.poisson(x, 1.5, 0.75)) <= tol
    u2, p2 = run(nx, ny, P, dtype, x, D, dt, n, Lx=1.5, Ly=0.75, peer=False)
    assert np.array_equal(u, u2) and np.array_equal(p, p2)


def test_peer_store_exchange_long_axes():
    nx, ny, P = 32768, 64, 4
    x = I.white_noise((ny, nx), 8)
    u, p = run(nx, ny, P, torch.complex128, x, 1e-9, 0.01, 2, peer=True)
    assert rel(u, O.diffuse(x, 1e-9, 0.01, 2)) <= 1e-12


# ---- fftpde_plan_2d_sharded / _3d_sharded: the whole slab solve inside the C ABI ------
from paper_2412_12308_b200 import fftpde as F  # noqa: E402


def spec2_from_slabs(X, P):
    # [P][ny][BW] column slabs -> the natural [ny][nx] spectrum
    return np.concatenate(list(X), axis=1) if P > 1 else X


@pytest.mark.parametrize("dtype,tol", [(torch.complex128, 1e-12), (torch.complex64, 1e-5)])
@pytest.mark.parametrize("nx,ny", [(256, 128), (64, 1024), (2048, 16)])
def test_sharded_plan_p1_vs_oracle(dtype, tol, nx, ny):
    # one process: P = 1, the all-to-all is an NCCL send/recv to self
    x = I.white_noise((ny, nx), 303)
    p = F.ShardedPlan(nx, ny, dtype=dtype, Lx=1.5, Ly=0.75)
    assert (p.P, p.R, p.BW) == (1, ny, nx)
    xd = torch.from_numpy(x).to(dtype).cuda()
    X = p.forward(xd)
    assert rel(X.cpu().numpy(), O.fft2(x)) <= tol
    assert rel(p.inverse(X).cpu().numpy(), x) <= tol
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson(x, 1.5, 0.75)) <= tol
    assert rel(p.diffuse(xd, 2e-4, 0.01, 3).cpu().numpy(), O.diffuse(x, 2e-4, 0.01, 3, 1.5, 0.75)) <= tol
    u = xd.clone()                                       # in place (u0 == u)
    p.diffuse(u, 2e-4, 0.01, 3, out=u)
    assert rel(u.cpu().numpy(), O.diffuse(x, 2e-4, 0.01, 3, 1.5, 0.75)) <= tol


@pytest.mark.parametrize("dtype,tol", [(torch.complex128, 1e-12), (torch.complex64, 1e-5)])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_plan_loopback_vs_oracle(dtype, tol, P):
    # P ranks emulated in one plan: the per-rank kernels, wavenumber offsets and
    # block exchange of the NCCL path, on one device
    nx, ny = 256, 128
    x = I.white_noise((ny, nx), 306)
    p = F.ShardedPlan(nx, ny, dtype=dtype, Lx=1.5, Ly=0.75, loopback=P)
    xd = torch.from_numpy(x).to(dtype).cuda()
    X = p.forward(xd)
    assert tuple(X.shape) == (P, ny, nx // P)
    assert rel(spec2_from_slabs(X.cpu().numpy(), P), O.fft2(x)) <= tol
    assert rel(p.inverse(X).cpu().numpy(), x) <= tol
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson(x, 1.5, 0.75)) <= tol
    assert rel(p.diffuse(xd, 2e-4, 0.01, 3).cpu().numpy(), O.diffuse(x, 2e-4, 0.01, 3, 1.5, 0.75)) <= tol


def test_sharded_plan_rank_count_independence_and_python_slab_solver():
    # the in-library diffusion step is the separable one (R26: x diffusion of the row
    # slab, exchange, y diffusion of the column slab): bit-for-bit independent of the
    # rank count, and within rounding of the Python SlabSolver's 2D multiply; Poisson
    # takes the same kernels in the same order as the SlabSolver: bit for bit
    nx, ny = 512, 256
    x = I.white_noise((ny, nx), 305)
    outs = []
    for P in (1, 4):
        pl = F.ShardedPlan(nx, ny, loopback=P)
        u_lib = pl.diffuse(torch.from_numpy(x).cuda(), 1e-4, 0.01, 3).cpu().numpy()
        p_lib = pl.poisson(torch.from_numpy(x).cuda()).cpu().numpy()
        u_py, p_py = run(nx, ny, P, torch.complex128, x, 1e-4, 0.01, 3)
        assert rel(u_lib, u_py) <= 1e-14
        assert np.array_equal(p_lib, p_py)
        outs.append(u_lib)
    assert np.array_equal(outs[0], outs[1])
    u1 = F.ShardedPlan(nx, ny).diffuse(torch.from_numpy(x).cuda(), 1e-4, 0.01, 3).cpu().numpy()
    assert np.array_equal(u1, outs[1])                   # NCCL P = 1 == loopback P = 4


def test_sharded_plan_long_axes():
    for nx, ny, P in ((32768, 16, 1), (32768, 64, 4), (64, 16384, 1), (64, 16384, 2)):
        x = I.white_noise((ny, nx), 304)
        p = F.ShardedPlan(nx, ny, loopback=P if P > 1 else 0)
        u = p.diffuse(torch.from_numpy(x).cuda(), 1e-9, 0.01, 2).cpu().numpy()
        assert rel(u, O.diffuse(x, 1e-9, 0.01, 2)) <= 1e-12


def rand3(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("P", [0, 2, 4])
@pytest.mark.parametrize("shape,L", [((16, 32, 64), (1.0, 2.0, 0.5)), ((8, 2048, 16), (1.0, 1.0, 1.0))])
def test_sharded_3d_vs_oracle(P, shape, L):
    # P = 0: the NCCL plan at P = 1; P > 1: loopback emulation of P ranks
    nz, ny, nx = shape
    x = rand3(shape, 277)
    p = F.ShardedPlan3D(nx, ny, nz, Lx=L[0], Ly=L[1], Lz=L[2], loopback=P)
    Pn = max(P, 1)
    xd = torch.from_numpy(x).cuda()
    X = p.forward(xd).cpu().numpy()
    full = np.concatenate(list(X), axis=1) if P else X       # y-slabs -> [nz][ny][nx]
    assert rel(full, O.fft3(x)) <= 1e-12
    assert rel(p.inverse(torch.from_numpy(X).cuda()).cpu().numpy(), x) <= 1e-12
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson3(x, *L)) <= 1e-12
    assert rel(p.diffuse(xd, 1e-3, 0.01, 3).cpu().numpy(), O.diffuse3(x, 1e-3, 0.01, 3, *L)) <= 1e-12
    assert p.R == ny // Pn and p.nzl == nz // Pn


def test_sharded_3d_c64_and_closeness_to_plan3d():
    nz, ny, nx = 32, 64, 64
    x = rand3((nz, ny, nx), 278)
    p = F.ShardedPlan3D(nx, ny, nz, dtype=torch.complex64, loopback=4)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda()
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson3(x.astype(np.complex64).astype(np.complex128))) <= 1e-5
    q = F.ShardedPlan3D(nx, ny, nz, loopback=8)
    ref = F.Plan3D(nx, ny, nz)
    x128 = torch.from_numpy(x).cuda()
    assert rel(q.diffuse(x128, 1e-3, 0.01, 2).cpu().numpy(), ref.diffuse(x128, 1e-3, 0.01, 2).cpu().numpy()) <= 1e-14


def test_sharded_plan_errors():
    with pytest.raises(F.FFTPDEError):
        F.ShardedPlan(100, 64)                           # not a power of two
    with pytest.raises(F.FFTPDEError) as e:
        F.ShardedPlan(64, 64, loopback=128)              # P does not divide the axes
    assert e.value.status == F.ERR_UNSUPPORTED
    with pytest.raises(F.FFTPDEError) as e:
        F.ShardedPlan3D(64, 64, 4, loopback=8)           # P does not divide nz
    assert e.value.status == F.ERR_UNSUPPORTED
    p = F.ShardedPlan(64, 64)
    x = torch.zeros(64, 64, dtype=torch.complex128, device="cuda")
    assert p.lib.fftpde_wave_step(p._h, x.data_ptr(), x.data_ptr(), 1.0, 0.1, 1) == F.ERR_UNSUPPORTED
    assert p.lib.fftpde_rows(p._h, x.data_ptr(), x.data_ptr(), 64, 0) == F.ERR_UNSUPPORTED
    with pytest.raises(F.FFTPDEError):
        p.forward(x, out=x)                              # forward is out of place


@pytest.mark.parametrize("dtype,tol", [(torch.complex128, 1e-12), (torch.complex64, 1e-5)])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_fused_row_exchange_vs_oracle_and_library_plan(dtype, tol, P):
    # the row pass stores its output straight into the owners' column slabs
    # (SURVEY.md 8(e) N10); the separable diffusion step is the in-library one,
    # so the result equals ShardedPlan's (pack + exchange) bit for bit
    nx, ny, D, dt, n = 256, 128, 2e-4, 0.01, 3
    x = I.white_noise((ny, nx), 111)
    u, p = run(nx, ny, P, dtype, x, D, dt, n, Lx=1.5, Ly=0.75, fused=True)
    assert rel(u, O.diffuse(x, D, dt, n, 1.5, 0.75)) <= tol
    assert rel(p, O.poisson(x, 1.5, 0.75)) <= tol
    lib = F.ShardedPlan(nx, ny, dtype=dtype, Lx=1.5, Ly=0.75, loopback=P)
    u_lib = lib.diffuse(torch.from_numpy(x).to(dtype).cuda(), D, dt, n).cpu().numpy()
    assert np.array_equal(u, u_lib)
    _, p_peer = run(nx, ny, P, dtype, x, D, dt, n, Lx=1.5, Ly=0.75, peer=True)
    assert np.array_equal(p, p_peer)                   # same kernels as the unfused peer path


@pytest.mark.parametrize("nx,ny,P", [(64, 256, 4), (32, 1024, 2), (16, 16384, 2)])
def test_fused_exchanges_column_kernels(nx, ny, P):
    # the column pass's peer-store epilogue through the pipelined (256-point: the
    # TMA pass is bypassed for peer output), radix-32 line (1024) and col2 (16384)
    # column passes
    x = I.white_noise((ny, nx), 113)
    u, p = run(nx, ny, P, torch.complex128, x, 3e-5, 0.01, 2, fused=True)
    assert rel(u, O.diffuse(x, 3e-5, 0.01, 2)) <= 1e-12
    assert rel(p, O.poisson(x)) <= 1e-12


def test_fused_row_exchange_long_rows():
    # 32768-point rows: the row2d cluster pass with its peer-store epilogue
    nx, ny, P = 32768, 64, 4
    x = I.white_noise((ny, nx), 112)
    u, p = run(nx, ny, P, torch.complex128, x, 1e-9, 0.01, 2, fused=True)
    assert rel(u, O.diffuse(x, 1e-9, 0.01, 2)) <= 1e-12
    assert rel(p, O.poisson(x)) <= 1e-12


def test_rows_to_peers_errors():
    pl = F.Plan(64, 64)
    x = torch.zeros(16, 64, dtype=torch.complex128, device="cuda")
    cs = [torch.zeros(64, 16, dtype=torch.complex128, device="cuda") for _ in range(4)]
    ptrs = [c.data_ptr() for c in cs]
    pl.rows_to_peers(x, ptrs, 0, 16, F.ROWS_FWD)        # valid
    with pytest.raises(F.FFTPDEError):
        pl.rows_to_peers(x, ptrs[:3], 0, 16, F.ROWS_FWD)  # 3 ranks do not divide nx = 64 into a power of two
    with pytest.raises(F.FFTPDEError):
        pl.rows_to_peers(x, ptrs, 4, 16, F.ROWS_FWD)      # rank out of range
    with pytest.raises(F.FFTPDEError):
        pl.rows_to_peers(x, ptrs, 0, 16, 7)               # unknown op


# ---- 3D pencil decomposition (fftpde_plan_3d_pencil) ----------
def to_xpencils(x, pz, py):
    # [nz][ny][nx] -> [P][nz/pz][ny/py][nx], rank r = i py + j: z-block i, y-block j
    nz, ny, nx = x.shape
    return np.ascontiguousarray(x.reshape(pz, nz // pz, py, ny // py, nx).transpose(0, 2, 1, 3, 4)
                                .reshape(pz * py, nz // pz, ny // py, nx))


def from_xpencils(xp, pz, py):
    P, nzl, nyl, nx = xp.shape
    return xp.reshape(pz, py, nzl, nyl, nx).transpose(0, 2, 1, 3, 4).reshape(pz * nzl, py * nyl, nx)


def from_zpencils(zp, pz, py):
    # [P][nz][ny/pz][nx/py] (rank i py + j: y-block i of ny/pz, x-block j) -> [nz][ny][nx]
    P, nz, nyl2, nxl = zp.shape
    return zp.reshape(pz, py, nz, nyl2, nxl).transpose(2, 0, 3, 1, 4).reshape(nz, pz * nyl2, py * nxl)


@pytest.mark.parametrize("pz,py", [(2, 2), (2, 4), (4, 2), (1, 4), (4, 1), (8, 2)])
@pytest.mark.parametrize("shape,L", [((8, 32, 64), (1.0, 2.0, 0.5)), ((16, 64, 32), (1.0, 1.0, 1.0))])
def test_pencil_3d_vs_oracle(pz, py, shape, L):
    nz, ny, nx = shape
    x = rand3(shape, 331)
    p = F.PencilPlan3D(nx, ny, nz, pz, py, Lx=L[0], Ly=L[1], Lz=L[2], loopback=True)
    xp = torch.from_numpy(to_xpencils(x, pz, py)).cuda()
    X = p.forward(xp)
    assert tuple(X.shape) == (pz * py, nz, ny // pz, nx // py)
    assert rel(from_zpencils(X.cpu().numpy(), pz, py), O.fft3(x)) <= 1e-12
    assert rel(from_xpencils(p.inverse(X).cpu().numpy(), pz, py), x) <= 1e-12
    assert rel(from_xpencils(p.poisson(xp).cpu().numpy(), pz, py), O.poisson3(x, *L)) <= 1e-12
    u = p.diffuse(xp, 1e-3, 0.01, 3).cpu().numpy()
    assert rel(from_xpencils(u, pz, py), O.diffuse3(x, 1e-3, 0.01, 3, *L)) <= 1e-12


def test_pencil_more_ranks_than_planes_c64():
    # P = 16 > nz = 8: beyond the z-slab plan (P <= nz); complex64 at 1e-5
    nz, ny, nx = 8, 64, 128
    x = rand3((nz, ny, nx), 332)
    with pytest.raises(F.FFTPDEError):
        F.ShardedPlan3D(nx, ny, nz, dtype=torch.complex64, loopback=16)
    p = F.PencilPlan3D(nx, ny, nz, 2, 8, dtype=torch.complex64, loopback=True)
    x64 = x.astype(np.complex64)
    xp = torch.from_numpy(to_xpencils(x64, 2, 8)).cuda()
    ref = O.poisson3(x64.astype(np.complex128))
    assert rel(from_xpencils(p.poisson(xp).cpu().numpy(), 2, 8), ref) <= 1e-5


def test_pencil_matches_plan3d_and_errors():
    nz, ny, nx = 16, 32, 32
    x = rand3((nz, ny, nx), 333)
    p = F.PencilPlan3D(nx, ny, nz, 4, 2, loopback=True)
    ref = F.Plan3D(nx, ny, nz).diffuse(torch.from_numpy(x).cuda(), 1e-3, 0.01, 2).cpu().numpy()
    u = p.diffuse(torch.from_numpy(to_xpencils(x, 4, 2)).cuda(), 1e-3, 0.01, 2).cpu().numpy()
    assert rel(from_xpencils(u, 4, 2), ref) <= 1e-14
    with pytest.raises(F.FFTPDEError) as e:
        F.PencilPlan3D(32, 32, 16, 32, 1, loopback=True)        # pz does not divide nz
    assert e.value.status == F.ERR_UNSUPPORTED
    with pytest.raises(F.FFTPDEError) as e:
        F.PencilPlan3D(16, 64, 16, 2, 16, dtype=torch.complex64, loopback=True)   # nx / py = one 8-byte element
    assert e.value.status == F.ERR_UNSUPPORTED
    with pytest.raises(ValueError):
        F.PencilPlan3D(32, 32, 16, 2, 2)                        # no process group: P = 1 != 4


def test_pencil_nccl_p1_vs_oracle():
    # the NCCL branch of the group exchanges (grouped send/recv to itself) at pz = py = 1
    nz, ny, nx = 16, 32, 64
    x = rand3((nz, ny, nx), 334)
    p = F.PencilPlan3D(nx, ny, nz, 1, 1, Lx=1.0, Ly=2.0, Lz=0.5)
    xd = torch.from_numpy(x).cuda()
    X = p.forward(xd)
    assert rel(X.cpu().numpy(), O.fft3(x)) <= 1e-12
    assert rel(p.inverse(X).cpu().numpy(), x) <= 1e-12
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson3(x, 1.0, 2.0, 0.5)) <= 1e-12


# ------------------------------------------- C5: the distributed four-step (R28)

@pytest.mark.parametrize("steps", [1, 2])
def test_c5_distributed_fourstep_vs_oracle_and_rank_counts(steps):
    # the sharded plan at C5's grid runs the four-step passes on each rank's Y-part /
    # X-part with one all-to-all per step (R28): P = 1 through NCCL (no exchange), P =
    # 2 / 4 / 8 emulated (loopback: the same per-rank kernels and block exchange).
    # Rank-2 separable input as in test_gpu_parity (every wavenumber populated) against
    # the oracle's own stepped 1D solves at all 2^30 points; every rank count gives the
    # same bits (the passes do the same arithmetic on relocated tiles), and one step
    # (Bx then By, as the single-GPU plan) equals the single-GPU plan bit for bit.
    n, D, dt = 32768, 1e-4, 0.01
    f1, g1, f2, g2 = (I.white_noise((n,), 710 + i) for i in range(4))
    Df1, Dg1, Df2, Dg2 = (O.diffuse(v.reshape(1, n), D, dt, steps).ravel() for v in (f1, g1, f2, g2))
    t = lambda v: torch.from_numpy(v).cuda()
    u0 = torch.outer(t(g1), t(f1)) + torch.outer(t(g2), t(f2))
    single = F.Plan(n, n, dtype=torch.complex128)
    us = single.diffuse(u0, D, dt, steps)
    del single
    torch.cuda.empty_cache()
    first = None
    for P in (1, 2, 4, 8):
        p = F.ShardedPlan(n, n, dtype=torch.complex128, loopback=P if P > 1 else 0)
        u = p.diffuse(u0, D, dt, steps)
        torch.cuda.synchronize()
        del p
        if first is None:
            first = u
            if steps == 1:
                assert torch.equal(u, us), P
            else:
                err = (torch.linalg.vector_norm(u - us) / torch.linalg.vector_norm(us)).item()
                assert err <= 1e-14, err
        else:
            assert torch.equal(u, first), P
            del u
        torch.cuda.empty_cache()
    del us, u0
    torch.cuda.empty_cache()
    ref = torch.outer(t(Dg1), t(Df1)) + torch.outer(t(Dg2), t(Df2))
    err = (torch.linalg.vector_norm(first - ref) / torch.linalg.vector_norm(ref)).item()
    assert err <= 1e-12, err


@pytest.mark.parametrize("steps", [1, 2])
def test_c5_fused_fourstep_peer_solver_vs_oracle(steps):
    # FusedFourStepSolver: R28 with the exchange fused into the B passes (each rank's
    # Bx / By epilogue stores its tiles straight into the peers' other part), P
    # virtual ranks on one device (LoopbackPeerComm).  Every point against the
    # oracle's stepped 1D solves of a rank-2 input (built row block by row block to
    # keep the footprint at u0 + plan + 4 part buffers + u), and the same bits on
    # every P (a strided sample of 2^20 points).
    n, D, dt = 32768, 1e-4, 0.01
    f1, g1, f2, g2 = (I.white_noise((n,), 730 + i) for i in range(4))
    Df1, Dg1, Df2, Dg2 = (torch.from_numpy(O.diffuse(v.reshape(1, n), D, dt, steps).ravel()).cuda()
                          for v in (f1, g1, f2, g2))
    t = lambda v: torch.from_numpy(v).cuda()
    plan = F.Plan(n, n, dtype=torch.complex128)
    sample = None
    for P in (1, 2, 8):
        u0 = torch.outer(t(g1), t(f1)) + torch.outer(t(g2), t(f2))
        solver = S.FusedFourStepSolver(n, S.LoopbackPeerComm(P), plan)
        R = n // P
        slabs = [u0[r * R:(r + 1) * R] for r in range(P)]
        outs = solver.diffuse(slabs, D, dt, steps)
        torch.cuda.synchronize()
        del solver, slabs, u0
        torch.cuda.empty_cache()
        u = torch.cat(outs)
        del outs
        s = u.view(-1)[::1021].clone()
        if sample is None:
            sample = s
        else:
            assert torch.equal(s, sample), P
        num = den = 0.0
        for b in range(0, n, 4096):                          # the reference row block by row block
            ref = torch.outer(Dg1[b:b + 4096], Df1) + torch.outer(Dg2[b:b + 4096], Df2)
            num += torch.linalg.vector_norm(u[b:b + 4096] - ref).item() ** 2
            den += torch.linalg.vector_norm(ref).item() ** 2
        del u
        torch.cuda.empty_cache()
        assert (num / den) ** 0.5 <= 1e-12, (P, (num / den) ** 0.5)


def test_fs_part_errors():
    n = 32768
    p = F.Plan(n, n, dtype=torch.complex128)
    x = torch.zeros(n * n // 2, dtype=torch.complex128, device="cuda")
    with pytest.raises(F.FFTPDEError):
        p.fs_part_aa(0, 3, 0, 0, x, x)                       # P not a power of two
    with pytest.raises(F.FFTPDEError):
        p.fs_part_aa(2, 2, 0, 0, x, x)                       # MID without phys
    with pytest.raises(F.FFTPDEError):
        p.fs_part_b(0, 2, 2, x, 1e-4, 0.01)                  # rank out of range
    with pytest.raises(F.FFTPDEError):
        p.fs_part_b(0, 2, 0, x, 1e-4, 0.01, peers=[x.data_ptr()])   # one peer for two ranks
    small = F.Plan(1024, 1024, dtype=torch.complex128)
    y = torch.zeros(1024 * 1024, dtype=torch.complex128, device="cuda")
    with pytest.raises(F.FFTPDEError):
        small.fs_part_aa(0, 1, 0, 0, y, y)                   # not the 32768^2 grid


def test_3d_long_z_sharded_and_pencil():
    # a 2048-plane volume: the z-pass of the z-slab and pencil plans is the two-level
    # column pass (fftpde_plan_3d's z tables), loopback ranks, against the oracle
    nz, ny, nx = 2048, 8, 16
    x = rand3((nz, ny, nx), 278)
    ref = O.poisson3(x)
    xd = torch.from_numpy(x).cuda()
    for P in (2, 4):
        p = F.ShardedPlan3D(nx, ny, nz, loopback=P)
        assert rel(p.poisson(xd).cpu().numpy(), ref) <= 1e-12, P
        assert rel(p.diffuse(xd, 1e-7, 0.01, 2).cpu().numpy(), O.diffuse3(x, 1e-7, 0.01, 2)) <= 1e-12, P
    p = F.PencilPlan3D(nx, ny, nz, 2, 2, loopback=True)
    xp = torch.from_numpy(to_xpencils(x, 2, 2)).cuda()
    assert rel(from_xpencils(p.poisson(xp).cpu().numpy(), 2, 2), ref) <= 1e-12
