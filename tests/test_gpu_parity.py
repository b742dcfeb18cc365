"""Parity of the CUDA path (through the C-ABI binding) with the fp64 CPU oracle.

Element-by-element relative L2 on the same seeded inputs.  Tolerances are
BASELINE.json north_star's: 1e-12 for complex128, 1e-5 for complex64 (the
complex64 input is upcast exactly for the oracle).  Needs a CUDA device.
"""
import math
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I

pytestmark = pytest.mark.gpu

C128, C64 = torch.complex128, torch.complex64
TOL = {C128: 1e-12, C64: 1e-5}
NP = {C128: np.complex128, C64: np.complex64}


def rel(a, b):
    a = np.asarray(a, np.complex128).ravel()
    b = np.asarray(b, np.complex128).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(x, dtype=C128):
    return torch.from_numpy(np.ascontiguousarray(x).astype(NP[dtype])).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.complex128)


def noise(shape, seed, dtype=C128):
    return I.white_noise(shape, seed, dtype=NP[dtype])


@pytest.fixture(scope="module", autouse=True)
def _lib():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    F.load_library()            # fails loudly if libfftpde.so is missing
    torch.cuda.init()


# ---------------------------------------------------------------- transforms

def test_spec_examples_through_abi():
    # SPEC.md:62-64 (eq:DFT, + sign) on a 1 x 4 grid, and the inverses SPEC.md:72-73
    p = F.Plan(4, 1, dtype=C128)
    cases = [([1, 1, 1, 1], [4, 0, 0, 0]), ([1, 0, 0, 0], [1, 1, 1, 1]), ([0, 1, 0, 0], [1, 1j, -1, -1j])]
    for x, X in cases:
        out = host(p.forward(dev(np.array([x], complex))))
        assert np.max(np.abs(out - np.array([X]))) <= 1e-15
        back = host(p.inverse(dev(np.array([X], complex))))
        assert np.max(np.abs(back - np.array([x]))) <= 1e-15


def _lengths():
    return [2 ** k for k in range(0, 16)]


def _shapes(n):
    if n <= 8192:
        return {(n, min(8192, max(1, 2 ** 18 // n))), (min(8192, max(1, 2 ** 18 // n)), n), (n, 2), (2, n)}
    # two-level cluster passes: long columns need whole 128-byte column blocks
    return {(n, 16), (16, n), (2, n), (n, 32)}


@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("n", _lengths())
def test_forward_inverse_every_length_both_axes(dtype, n):
    # length n along y with a few x lengths, and along x with a few y lengths;
    # batch 3 so CTAs span grid boundaries
    for (ny, nx) in _shapes(n):
        B = 3 if nx * ny <= 2 ** 16 else 1
        x = noise((B, ny, nx), 1000 + n + nx, dtype)
        p = F.Plan(nx, ny, batch=B, dtype=dtype)
        X = host(p.forward(dev(x, dtype)))
        Xo = O.fft2(x.astype(np.complex128))
        assert rel(X, Xo) <= TOL[dtype], (ny, nx)
        xb = host(p.inverse(dev(Xo, dtype)))
        assert rel(xb, O.fft2(Xo, inverse=True)) <= TOL[dtype], (ny, nx)


@pytest.mark.parametrize("dtype,ny,nx", [(C128, 128, 256), (C64, 128, 256),
                                         (C128, 256, 64), (C128, 512, 32), (C128, 1024, 16), (C64, 512, 64)])
def test_in_place_and_strided_batch(dtype, ny, nx):
    # ny = 256 / 512 (c128) and 512 (c64): the TMA column pass (3D tensor maps with
    # the batch stride); ny = 1024 (c128): the radix-32 column pass
    B = 4
    p = F.Plan(nx, ny, batch=B, dtype=dtype)
    x = noise((B, ny, nx), 7, dtype)
    t = dev(x, dtype)
    p.forward(t, out=t)                                          # in place
    assert rel(host(t), O.fft2(x.astype(np.complex128))) <= TOL[dtype]
    # grids 'stride' elements apart inside a larger buffer
    stride = nx * ny + 64
    buf = torch.zeros(B * stride, dtype=dtype, device="cuda")
    for b in range(B):
        buf[b * stride: b * stride + nx * ny] = dev(x[b].ravel(), dtype)
    st = p.lib.fftpde_poisson_batched(p._h, buf.data_ptr(), buf.data_ptr(), B, stride)
    assert st == F.OK
    got = host(buf)
    ref = O.poisson(x.astype(np.complex128))
    for b in range(B):
        assert rel(got[b * stride: b * stride + nx * ny].reshape(ny, nx), ref[b]) <= TOL[dtype]
        assert np.all(got[b * stride + nx * ny: (b + 1) * stride] == 0)   # gaps untouched


# ---------------------------------------------------------------- C1 Poisson

def test_c1_poisson_full():
    d = I.c1_inputs(64)
    p = F.Plan(64, 64, dtype=C128)
    for part in (d.rho, d.rho_sin, d.rho_blobs):
        u = host(p.poisson(dev(part)))
        assert rel(u, O.poisson(part)) <= 1e-12
        assert abs(u.mean()) <= 1e-14 * np.abs(u).max()
    x = I.axis(64)
    u = host(p.poisson(dev(d.rho_sin)))
    assert rel(u, np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x))) <= 1e-13


@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("shape", [(1, 64), (64, 1), (2, 2), (16, 16), (32, 32), (64, 32), (32, 128),
                                   (8, 1024), (512, 16)])
def test_poisson_shapes(dtype, shape):
    ny, nx = shape
    Lx, Ly = 1.7, 0.6
    x = noise((2, ny, nx), 11 + nx, dtype)
    p = F.Plan(nx, ny, batch=2, dtype=dtype, Lx=Lx, Ly=Ly)
    u = host(p.poisson(dev(x, dtype)))
    assert rel(u, O.poisson(x.astype(np.complex128), Lx, Ly)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("shape", [(32768, 16), (16, 32768), (16384, 32), (8, 16384)])
def test_long_axes_solvers(dtype, shape):
    # two-level (cluster) row and column passes inside the solvers
    ny, nx = shape
    x = noise((ny, nx), 77 + nx, dtype)
    p = F.Plan(nx, ny, dtype=dtype, Lx=1.0, Ly=2.0)
    u = host(p.poisson(dev(x, dtype)))
    assert rel(u, O.poisson(x.astype(np.complex128), 1.0, 2.0)) <= TOL[dtype]
    d = host(p.diffuse(dev(x, dtype), 1e-6, 0.01, 3))
    assert rel(d, O.diffuse(x.astype(np.complex128), 1e-6, 0.01, 3, 1.0, 2.0)) <= TOL[dtype]
    uu, vv = dev(x, dtype), dev(noise((ny, nx), 78, dtype), dtype)
    v0 = host(vv)
    p.wave_step(uu, vv, 0.3, 1e-4, 2)
    uo, vo = O.wave(x.astype(np.complex128), v0, 0.3, 1e-4, 2, 1.0, 2.0)
    assert rel(host(uu), uo) <= TOL[dtype] and rel(host(vv), vo) <= TOL[dtype]


@pytest.mark.parametrize("dtype,B,ny,nx", [(C128, 5, 32, 32768), (C64, 3, 16, 32768), (C128, 9, 32, 16384)])
def test_long_row_diffusion_many_rows_per_cluster(dtype, B, ny, nx):
    # rows >> clusters: the row2d diffusion pass runs its steady state (the next
    # row's input staged by cp.async while this one is transformed, the mbarrier
    # cycling through its phases) with ragged per-cluster row counts, batched
    x = noise((B, ny, nx), 91 + ny, dtype)
    p = F.Plan(nx, ny, batch=B, dtype=dtype, Lx=1.0, Ly=0.5)
    u = host(p.diffuse(dev(x, dtype), 3e-7, 0.01, 2))
    assert rel(u, O.diffuse(x.astype(np.complex128), 3e-7, 0.01, 2, 1.0, 0.5)) <= TOL[dtype]


# ---------------------------------------------------------------- C2 diffusion

def test_c2_diffusion_prefix_vs_stepped_oracle():
    g = I.c2_inputs(1024)
    p = F.Plan(1024, 1024, dtype=C128)
    u = host(p.diffuse(dev(g.u0), 1e-3, 0.01, 20))
    assert rel(u, O.diffuse(g.u0, 1e-3, 0.01, 20)) <= 1e-12


def test_c2_diffusion_full_vs_collapsed_and_heat_kernel():
    g = I.c2_inputs(1024)
    p = F.Plan(1024, 1024, dtype=C128)
    u = host(p.diffuse(dev(g.u0), 1e-3, 0.01, 200))
    assert rel(u, O.diffuse(g.u0, 1e-3, 0.01, 200, collapsed=True)) <= 1e-12
    # exact periodic heat kernel (closed form), T = 2
    x = I.axis(1024)
    exact = np.zeros((1024, 1024))
    for (cx, cy), s, a in zip(g.centres, g.sigmas, g.amps):
        s2 = s * s + 4e-3 * 2.0
        gx = sum(np.exp(-(x - cx - m) ** 2 / s2) for m in range(-2, 3))
        gy = sum(np.exp(-(x - cy - m) ** 2 / s2) for m in range(-2, 3))
        exact += a * (s * s / s2) * np.outer(gy, gx)
    assert rel(u, exact) <= 1e-12
    assert abs(u.mean() / g.u0.mean() - 1) <= 1e-12               # Fig. 4


@pytest.mark.parametrize("dtype", [C128, C64])
def test_diffusion_shapes_and_zero_steps(dtype):
    ny, nx = 64, 256
    x = noise((3, ny, nx), 5, dtype)
    p = F.Plan(nx, ny, batch=3, dtype=dtype, Lx=2.0, Ly=0.5)
    u = host(p.diffuse(dev(x, dtype), 0.003, 0.02, 7))
    assert rel(u, O.diffuse(x.astype(np.complex128), 0.003, 0.02, 7, 2.0, 0.5)) <= TOL[dtype]
    t = dev(x, dtype)
    u0 = host(p.diffuse(t, 0.003, 0.02, 0))
    assert np.array_equal(u0, x.astype(np.complex128))           # nsteps = 0 copies


@pytest.mark.parametrize("dtype,ny,nx,B", [(C128, 1024, 1024, 2), (C128, 512, 128, 3), (C128, 256, 2048, 2),
                                           (C64, 512, 512, 3), (C128, 2048, 64, 2), (C64, 1024, 32, 2)])
def test_separable_diffusion_batched_across_kernel_families(dtype, ny, nx, B):
    # the separable step (R26) through every row / column pass family, batched:
    # radix-32 lines (1024 c128), TMA columns (256 / 512), pipelined rows
    # (bulk-copied at 2048), c64 TMA radix-32 columns (512), col2 (2048 columns)
    x = noise((B, ny, nx), 17, dtype)
    p = F.Plan(nx, ny, batch=B, dtype=dtype, Lx=1.3, Ly=0.7)
    u = host(p.diffuse(dev(x, dtype), 2e-3, 0.01, 3))
    assert rel(u, O.diffuse(x.astype(np.complex128), 2e-3, 0.01, 3, 1.3, 0.7)) <= TOL[dtype]


# ---------------------------------------------------------------- C3 wave

def test_c3_wave_prefix_vs_stepped_oracle():
    w = I.c3_inputs(512)
    p = F.Plan(512, 512, dtype=C128)
    u, v = dev(w.u), dev(w.ut)
    p.wave_step(u, v, 1.0, 1e-4 * 8, 50)
    uo, vo = O.wave(w.u, w.ut, 1.0, 1e-4 * 8, 50)
    assert rel(host(u), uo) <= 1e-12
    assert rel(host(v), vo) <= 1e-12


def test_c3_wave_prefix_full_size_vs_stepped_oracle():
    # the C3 workload itself (4096^2, dt = 1e-4) for its first 50 steps against the
    # stepped oracle (SURVEY.md 8(c) coverage plan); measured 5.7e-15 (u), 9.2e-14 (u_t)
    w = I.c3_inputs(4096)
    p = F.Plan(4096, 4096, dtype=C128)
    u, v = dev(w.u), dev(w.ut)
    p.wave_step(u, v, 1.0, 1e-4, 50)
    uo, vo = O.wave(w.u, w.ut, 1.0, 1e-4, 50)
    assert rel(host(u), uo) <= 1e-12
    assert rel(host(v), vo) <= 1e-12


def test_c3_wave_full_vs_collapsed():
    w = I.c3_inputs(4096)
    p = F.Plan(4096, 4096, dtype=C128)
    u, v = dev(w.u), dev(w.ut)
    p.wave_step(u, v, 1.0, 1e-4, 500)
    uo, vo = O.wave(w.u, w.ut, 1.0, 1e-4, 500, collapsed=True)
    uh, vh = host(u), host(v)
    assert rel(uh, uo) <= 1e-12
    assert rel(vh, vo) <= 1e-12
    # mean law of eq:OmegaZero with u_t(0) = 0 (Fig. 6)
    assert abs(uh.mean() / w.u.mean() - 1) <= 1e-12


@pytest.mark.parametrize("dtype", [C128, C64])
def test_wave_shapes_reversal(dtype):
    ny, nx = 128, 64
    u0 = noise((2, ny, nx), 21, dtype)
    v0 = noise((2, ny, nx), 22, dtype)
    p = F.Plan(nx, ny, batch=2, dtype=dtype, Lx=1.3, Ly=0.9)
    u, v = dev(u0, dtype), dev(v0, dtype)
    p.wave_step(u, v, 0.7, 3e-3, 9)
    uo, vo = O.wave(u0.astype(np.complex128), v0.astype(np.complex128), 0.7, 3e-3, 9, 1.3, 0.9)
    assert rel(host(u), uo) <= TOL[dtype] and rel(host(v), vo) <= TOL[dtype]
    p.wave_step(u, v, 0.7, -3e-3, 9)                              # time reversal: two solves, errors add
    assert rel(host(u), u0) <= 2 * TOL[dtype]


@pytest.mark.parametrize("nx,ny,batch", [(8, 2048, 2), (16, 4096, 1), (2, 4096, 3)])
def test_wave_long_columns_batched_vs_stepped_oracle(nx, ny, batch):
    # 2048 / 4096-point columns: the cluster-pair TMA wave pass (one column of
    # U and V per CTA pair, 16-byte boxes), batched and narrow grids
    u0 = noise((batch, ny, nx), 41)
    v0 = noise((batch, ny, nx), 42)
    p = F.Plan(nx, ny, batch=batch, Lx=0.8, Ly=2.0)
    u, v = dev(u0), dev(v0)
    p.wave_step(u, v, 1.3, 2e-3, 4)
    uo, vo = O.wave(u0, v0, 1.3, 2e-3, 4, 0.8, 2.0)
    assert rel(host(u), uo) <= 1e-12 and rel(host(v), vo) <= 1e-12


@pytest.mark.parametrize("nx,ny,nsteps", [(2048, 2048, 3), (4096, 2048, 3), (2048, 4096, 1), (4096, 4096, 2)])
def test_wave_transposed_spectrum_vs_stepped_oracle(nx, ny, nsteps):
    # single grids of 2048 / 4096-point rows and columns (the cluster-pair wave column
    # pass; with FFTPDE_WAVET=1 the transposed-spectrum path of wavet.cuh, run on the
    # B200 in round 2: 13 wave tests passed); nsteps = 1 has no MID row pass
    u0, v0 = noise((ny, nx), 51), noise((ny, nx), 52)
    p = F.Plan(nx, ny, Lx=0.8, Ly=2.0)
    u, v = dev(u0), dev(v0)
    p.wave_step(u, v, 1.3, 2e-3, nsteps)
    uo, vo = O.wave(u0, v0, 1.3, 2e-3, nsteps, 0.8, 2.0)
    assert rel(host(u), uo) <= 1e-12 and rel(host(v), vo) <= 1e-12


def test_wave_zero_speed_and_zero_steps():
    ny, nx = 32, 32
    u0, v0 = noise((ny, nx), 31), noise((ny, nx), 32)
    p = F.Plan(nx, ny)
    u, v = dev(u0), dev(v0)
    p.wave_step(u, v, 0.0, 0.5, 3)                                # c = 0: u <- u + T v
    assert rel(host(u), u0 + 1.5 * v0) <= 1e-13 and rel(host(v), v0) <= 1e-14
    p.wave_step(u, v, 1.0, 0.5, 0)


# ---------------------------------------------------------------- C5 diffusion 32768^2

def heat_kernel_points(ks, js, n, centres, sigmas, amps, D, T):
    """Exact periodic heat-kernel solution at grid points (k, j): each Gaussian
    A exp(-r^2/s^2) becomes A s^2/(s^2+4DT) exp(-r^2/(s^2+4DT)) (minimum image
    suffices: s^2 + 4DT < 2e-4, so images at distance >= 0.5 are below e^-1000)."""
    x = js / n
    y = ks / n
    out = np.zeros(len(ks))
    for (cx, cy), s, a in zip(centres, sigmas, amps):
        s2 = s * s + 4 * D * T
        dx = np.mod(x - cx + 0.5, 1.0) - 0.5
        dy = np.mod(y - cy + 0.5, 1.0) - 0.5
        out += a * (s * s / s2) * np.exp(-(dx * dx + dy * dy) / s2)
    return out


def test_c5_diffusion_full_size_sampled_closed_form():
    # BASELINE configs[4] on one GPU: 32768^2 complex128, D = 1e-4, dt = 0.01, 20 steps
    n, D, dt, steps = 32768, 1e-4, 0.01, 20
    u0, centres, sigmas, amps = I.c5_field_torch(n)
    p = F.Plan(n, n, dtype=C128)
    u = p.diffuse(u0, D, dt, steps)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    ks = rng.integers(0, n, 3000)
    js = rng.integers(0, n, 3000)
    # points near the Gaussian centres too (where the field is large)
    ks = np.concatenate([ks, np.round(centres[:500, 1] * n).astype(int) % n])
    js = np.concatenate([js, np.round(centres[:500, 0] * n).astype(int) % n])
    got = u[torch.from_numpy(ks).cuda(), torch.from_numpy(js).cuda()].cpu().numpy()
    exact = heat_kernel_points(ks, js, n, centres, sigmas, amps, D, steps * dt)
    assert np.linalg.norm(got - exact) / np.linalg.norm(exact) <= 1e-12
    assert np.max(np.abs(got.imag)) <= 1e-14
    m0 = u0.real.double().mean().item()
    assert abs(u.real.double().mean().item() / m0 - 1) <= 1e-12      # mean conservation (Fig. 4)


# ---------------------------------------------------------------- C4 batched Poisson

def test_c4_batched_poisson_every_grid():
    # all 256 grids of the batch against the oracle on the upcast complex64 input;
    # the bar is the maximum over the grids (measured 2.1e-7)
    s = I.c4_inputs(512, 256)
    p = F.Plan(512, 512, batch=256, dtype=C64)
    u = p.poisson(dev(s, C64)).cpu().numpy()
    errs = [rel(u[g], O.poisson(s[g].astype(np.complex64).astype(np.complex128))) for g in range(256)]
    assert max(errs) <= 1e-5, (int(np.argmax(errs)), max(errs))


# ---------------------------------------------------------------- errors

def test_errors_are_reported():
    with pytest.raises(F.FFTPDEError) as e:
        F.Plan(48, 64)
    assert e.value.status == F.ERR_NOT_POW2_X
    with pytest.raises(F.FFTPDEError) as e:
        F.Plan(64, 96)
    assert e.value.status == F.ERR_NOT_POW2_Y
    with pytest.raises(F.FFTPDEError) as e:
        F.Plan(64, 0)
    assert e.value.status == F.ERR_EMPTY
    p = F.Plan(64, 64)
    with pytest.raises(F.FFTPDEError) as e:
        p.diffuse(dev(noise((64, 64), 1)), -1.0, 0.1, 1)
    assert e.value.status == F.ERR_INVALID_ARG
    with pytest.raises(TypeError):
        p.poisson(dev(noise((64, 64), 1), C64))


_NO_TMA_SCRIPT = r"""
import numpy as np, torch
from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F
rng = np.random.default_rng(5)
def noise(shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
worst = 0.0
for ny, nx, B in ((256, 32, 2), (512, 16, 1)):           # column passes without TMA (pipe_kernel)
    x = noise((B, ny, nx))
    p = F.Plan(nx, ny, batch=B)
    worst = max(worst, rel(p.poisson(torch.from_numpy(x).cuda()).cpu().numpy(), O.poisson(x)))
    worst = max(worst, rel(p.diffuse(torch.from_numpy(x).cuda(), 1e-3, 0.01, 3).cpu().numpy(),
                           O.diffuse(x, 1e-3, 0.01, 3)))
for ny, nx, B in ((32, 32768, 3), (16, 16384, 5)):       # row2d passes launched without PDL
    x = noise((B, ny, nx))
    p = F.Plan(nx, ny, batch=B)
    worst = max(worst, rel(p.diffuse(torch.from_numpy(x).cuda(), 1e-6, 0.01, 2).cpu().numpy(),
                           O.diffuse(x, 1e-6, 0.01, 2)))
u0, v0 = noise((4096, 8)), noise((4096, 8))                # wave columns without TMA (col2 four-step)
p = F.Plan(8, 4096)
u, v = torch.from_numpy(u0).cuda(), torch.from_numpy(v0).cuda()
p.wave_step(u, v, 1.1, 2e-3, 3)
uo, vo = O.wave(u0, v0, 1.1, 2e-3, 3)
worst = max(worst, rel(u.cpu().numpy(), uo), rel(v.cpu().numpy(), vo))
print("WORST", worst)
"""


def test_fallback_passes_without_tma(tmp_path):
    # FFTPDE_TMA=0, FFTPDE_PDL=0: the library takes its non-TMA column passes (the path a
    # driver without the tensor-map encoder would get); same parity bar
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FFTPDE_TMA="0", FFTPDE_PDL="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _NO_TMA_SCRIPT], env=env, cwd=root, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    worst = float(r.stdout.strip().split()[-1])
    assert worst <= 1e-12


# ---------------------------------------------------------------- C5 at full size against the oracle

@pytest.mark.parametrize("steps", [1, 20])
def test_c5_full_size_separable_rank2_vs_oracle_every_point(steps):
    # C5's grid (and step count; 1 step: AA, Bx, By, AA^-1 only) through the four-step passes (AA / MID, Bx, By) on a
    # rank-2 input u0 = g1 f1^T + g2 f2^T of seeded complex white noise (every
    # wavenumber populated): the separable diffusion (R26) maps it to
    # (D_y g1)(D_x f1)^T + (D_y g2)(D_x f2)^T, the oracle's own stepped 1D solves
    # (ny = 1 grids), compared at all 2^30 points
    n, D, dt = 32768, 1e-4, 0.01
    f1, g1, f2, g2 = (I.white_noise((n,), 700 + i) for i in range(4))
    Df1, Dg1, Df2, Dg2 = (O.diffuse(v.reshape(1, n), D, dt, steps).ravel() for v in (f1, g1, f2, g2))
    t = lambda v: torch.from_numpy(v).cuda()
    u0 = torch.outer(t(g1), t(f1)) + torch.outer(t(g2), t(f2))
    p = F.Plan(n, n, dtype=C128)
    u = p.diffuse(u0, D, dt, steps)
    del u0
    ref = torch.outer(t(Dg1), t(Df1)) + torch.outer(t(Dg2), t(Df2))
    err = (torch.linalg.vector_norm(u - ref) / torch.linalg.vector_norm(ref)).item()
    assert err <= 1e-12, err


def test_wave_transposed_spectrum_path_subprocess():
    # the opt-in transposed-spectrum wave path (wavet.cuh, FFTPDE_WAVET=1 is read once
    # per process): a fresh interpreter runs 2048^2 for 3 steps (first-step FWD, one MID,
    # last-step INV row passes) against the stepped oracle
    import subprocess
    import sys
    code = (
        "import numpy as np, torch\n"
        "from oracle import oracle as O\n"
        "from paper_2412_12308_b200 import fftpde as F\n"
        "rng = np.random.default_rng(61)\n"
        "u0 = rng.standard_normal((2048, 2048)) + 1j * rng.standard_normal((2048, 2048))\n"
        "v0 = rng.standard_normal((2048, 2048)) + 1j * rng.standard_normal((2048, 2048))\n"
        "p = F.Plan(2048, 2048, Lx=0.8, Ly=2.0)\n"
        "u, v = torch.from_numpy(u0).cuda(), torch.from_numpy(v0).cuda()\n"
        "p.wave_step(u, v, 1.3, 2e-3, 3)\n"
        "uo, vo = O.wave(u0, v0, 1.3, 2e-3, 3, 0.8, 2.0)\n"
        "r = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))\n"
        "eu, ev = r(u.cpu().numpy(), uo), r(v.cpu().numpy(), vo)\n"
        "assert eu <= 1e-12 and ev <= 1e-12, (eu, ev)\n"
        "print('ok', eu, ev)\n")
    env = dict(os.environ, FFTPDE_WAVET="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stdout + res.stderr
