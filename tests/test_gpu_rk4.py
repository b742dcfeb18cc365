"""GPU parity of the time-dependent-source path through
the C-ABI (fftpde_wave_rk4): RK4 on the Fourier-space wave system with the
paper's orbiting Gaussian source, against the fp64
CPU oracle on the same seeded inputs, plus the paper's self-convergence factor
and the forced-oscillator closed form computed on the GPU results."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I

pytestmark = pytest.mark.gpu

L, XMIN = 4.0, -2.0                  # D = [-2, 2]^2
SRC = dict(A=1.0, sigma=0.1, Omega=5.0, gamma=10.0, rs=0.5)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b)))


def gpu_rk4(u0, v0, dt, steps, dtype=torch.complex128, c=1.0, t0=0.0, **src):
    ny, nx = u0.shape
    p = F.Plan(nx, ny, dtype=dtype, Lx=L, Ly=L * ny / nx)
    u = torch.from_numpy(np.ascontiguousarray(u0)).to(dtype).cuda()
    v = torch.from_numpy(np.ascontiguousarray(v0)).to(dtype).cuda()
    kw = dict(SRC)
    kw.update(src)
    m = p.wave_rk4(u, v, dt, steps, c=c, t0=t0, xmin=XMIN, ymin=XMIN * ny / nx, **kw)
    return u.cpu().numpy(), v.cpu().numpy(), m.cpu().numpy()


@pytest.mark.parametrize("shape", [(64, 64), (64, 128), (128, 32)])
def test_rk4_parity_vs_oracle(shape):
    ny, nx = shape
    rng = np.random.default_rng(448)
    u0 = 0.01 * rng.standard_normal((ny, nx)) + 0j
    v0 = 0.01 * rng.standard_normal((ny, nx)) + 0j
    dt, steps = 0.25 * L / max(nx, ny), 24
    ug, vg, mg = gpu_rk4(u0, v0, dt, steps, c=1.3, t0=0.1)
    uo, vo, mo = O.wave_rk4(u0, v0, dt, steps, c=1.3, t0=0.1, Lx=L, Ly=L * ny / nx, xmin=XMIN,
                            ymin=XMIN * ny / nx, **SRC)
    assert rel(ug, uo) <= 1e-12 and rel(vg, vo) <= 1e-12
    assert np.max(np.abs(mg - mo)) <= 1e-12 * np.max(np.abs(mo))


def test_rk4_parity_long_columns_and_c64():
    # ny = 2048 takes the two-level column pass inside every source transform
    ny, nx = 2048, 16
    rng = np.random.default_rng(449)
    u0 = 0.01 * rng.standard_normal((ny, nx)) + 0j
    dt, steps = 0.25 * L / ny, 4
    ug, vg, mg = gpu_rk4(u0, np.zeros_like(u0), dt, steps)
    uo, vo, mo = O.wave_rk4(u0, np.zeros_like(u0), dt, steps, Lx=L, Ly=L * ny / nx, xmin=XMIN,
                            ymin=XMIN * ny / nx, **SRC)
    assert rel(ug, uo) <= 1e-12 and rel(vg, vo) <= 1e-12
    # complex64: oracle on the exactly upcast input
    n = 128
    u0 = (0.01 * rng.standard_normal((n, n))).astype(np.complex64)
    ug, vg, mg = gpu_rk4(u0, np.zeros_like(u0), 0.25 * L / n, 16, dtype=torch.complex64)
    uo, vo, mo = O.wave_rk4(u0.astype(np.complex128), np.zeros((n, n)), 0.25 * L / n, 16, xmin=XMIN,
                            ymin=XMIN, **SRC)
    assert rel(ug, uo) <= 1e-5 and rel(vg, vo) <= 1e-5


def test_rk4_self_convergence_factor_16_on_gpu():
    # eq:SCF, Fig. 8: N = 64, 128, 256 with dt = 0.25 h
    T1 = 2.5
    means = {}
    for n in (64, 128, 256):
        dt = 0.25 * L / n
        z = np.zeros((n, n))
        _, _, m = gpu_rk4(z, z, dt, int(round(T1 / dt)))
        means[n] = m[:: n // 64].real
    t = np.arange(means[64].size) * (0.25 * L / 64)
    win = (t >= 0.5) & (t <= T1)
    d1 = means[128][win] - means[64][win]
    d2 = means[256][win] - means[128][win]
    q = np.linalg.norm(d1) / np.linalg.norm(d2)
    assert 10.0 <= q <= 24.0, q
    assert abs(q - 16.0) <= 0.5                  # the oracle's value is 16.015


def test_rk4_static_source_forced_oscillator_on_gpu():
    n = 64
    h = L / n
    dt = 0.25 * h
    steps = int(round(2.0 / dt))
    T = steps * dt
    z = np.zeros((n, n))
    u, v, m = gpu_rk4(z, z, dt, steps, gamma=0.0, Omega=0.0)
    s = O.orbit_source(n, n, 0.0, gamma=0.0, Omega=0.0, rs=0.5)
    k = 2 * np.pi * np.fft.fftfreq(n, d=h)
    kap2 = k[None, :] ** 2 + k[:, None] ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        fac = np.where(kap2 > 0, (1 - np.cos(np.sqrt(kap2) * T)) / kap2, 0.5 * T * T)
    u_ex = np.fft.ifft2(fac * np.fft.fft2(s))
    assert np.max(np.abs(u - u_ex)) <= 1e-6        # SPEC acceptance 9
    tt = np.arange(steps + 1) * dt
    assert np.max(np.abs(m - 0.5 * tt ** 2 * s.mean())) <= 1e-13 * np.max(np.abs(m))


def test_rk4_errors():
    lib = F.load_library()
    p = F.Plan(32, 32, batch=2)
    u = torch.zeros(32, 32, dtype=torch.complex128, device="cuda")
    v = torch.zeros_like(u)
    with pytest.raises(F.FFTPDEError) as e:
        p.wave_rk4(u, v, 0.01, 2)
    assert e.value.status == F.ERR_UNSUPPORTED
    q = F.Plan(32, 32)
    for bad in (dict(dt=0.0), dict(dt=-1.0), dict(dt=float("nan"))):
        with pytest.raises(F.FFTPDEError) as e:
            q.wave_rk4(u, v, bad["dt"], 2)
        assert e.value.status == F.ERR_INVALID_ARG
    with pytest.raises(F.FFTPDEError) as e:
        q.wave_rk4(u, v, 0.01, 2, sigma=0.0)
    assert e.value.status == F.ERR_INVALID_ARG
    need = lib.fftpde_wave_rk4_scratch_size(q._h)
    small = torch.empty(need // 2, dtype=torch.uint8, device="cuda")
    st = lib.fftpde_wave_rk4(q._h, u.data_ptr(), v.data_ptr(), 1.0, 0.0, 0.0, 1.0, 0.1, 5.0, 10.0, 0.5, 0.0,
                             0.01, 2, None, small.data_ptr(), small.numel())
    assert st == F.ERR_WORKSPACE
    # nsteps = 0 leaves the fields unchanged (forward + inverse round trip)
    x = torch.randn(32, 32, dtype=torch.complex128, device="cuda")
    y = x.clone()
    m = q.wave_rk4(x, torch.zeros_like(x), 0.01, 0)
    assert torch.allclose(x, y, rtol=0, atol=1e-14) and m.numel() == 1
