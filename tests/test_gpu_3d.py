"""GPU parity of the 3D extension through
the C-ABI (fftpde_plan_3d + the whole-plan calls), against the fp64 oracle on
the same seeded inputs, including ragged shapes, the two-level y-pass, the
complex64 line-kernel z-pass, and the error paths."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b)))


def rand(shape, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype)


@pytest.mark.parametrize("shape,L", [((8, 16, 32), (1.0, 2.0, 0.5)), ((32, 64, 64), (1.0, 1.0, 1.0)),
                                     ((64, 8, 16), (3.0, 1.0, 2.0)), ((2, 32, 1024), (1.0, 1.0, 1.0)),
                                     ((4, 2048, 16), (1.0, 1.0, 1.0)), ((1, 16, 16), (1.0, 1.0, 1.0))])
def test_3d_parity_c128(shape, L):
    nz, ny, nx = shape
    x = rand(shape, 275)
    p = F.Plan3D(nx, ny, nz, Lx=L[0], Ly=L[1], Lz=L[2])
    xd = torch.from_numpy(x).cuda()
    assert rel(p.forward(xd).cpu().numpy(), O.fft3(x)) <= 1e-12
    assert rel(p.inverse(xd).cpu().numpy(), O.fft3(x, inverse=True)) <= 1e-12
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson3(x, *L)) <= 1e-12
    assert rel(p.diffuse(xd, 1e-3, 0.01, 5).cpu().numpy(), O.diffuse3(x, 1e-3, 0.01, 5, *L)) <= 1e-12


def test_3d_parity_c64_line_kernel_z_pass():
    nz, ny, nx = 512, 8, 16                       # the z-pass takes the c64 512-point line kernel
    x = rand((nz, ny, nx), 276, np.complex64)
    p = F.Plan3D(nx, ny, nz, dtype=torch.complex64)
    xd = torch.from_numpy(x).cuda()
    x64 = x.astype(np.complex128)
    assert rel(p.forward(xd).cpu().numpy(), O.fft3(x64)) <= 1e-5
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson3(x64)) <= 1e-5
    assert rel(p.diffuse(xd, 1e-3, 0.01, 3).cpu().numpy(), O.diffuse3(x64, 1e-3, 0.01, 3)) <= 1e-5


def test_3d_closed_forms_on_gpu():
    nz, ny, nx = 16, 32, 64
    l, k, j = np.arange(nz), np.arange(ny), np.arange(nx)
    m = (np.exp(2j * np.pi * ((2 * l) % nz) / nz)[:, None, None] *
         np.exp(2j * np.pi * ((-3 * k) % ny) / ny)[None, :, None] *
         np.exp(2j * np.pi * ((5 * j) % nx) / nx)[None, None, :])
    k2 = (2 * math.pi) ** 2 * (2 ** 2 + 3 ** 2 + 5 ** 2)
    p = F.Plan3D(nx, ny, nz)
    u = p.poisson(torch.from_numpy(m).cuda()).cpu().numpy()
    assert np.max(np.abs(u + m / k2)) <= 1e-14
    d = p.diffuse(torch.from_numpy(m).cuda(), 1e-3, 0.01, 50).cpu().numpy()
    assert np.max(np.abs(d - math.exp(-1e-3 * k2 * 0.5) * m)) <= 1e-13


def test_3d_errors():
    with pytest.raises(F.FFTPDEError) as e:
        F.Plan3D(16, 16, 12)
    assert e.value.status == F.ERR_NOT_POW2_Z
    with pytest.raises(F.FFTPDEError) as e:
        F.Plan3D(16, 16, 65536)                   # beyond the two-level z-pass
    assert e.value.status == F.ERR_UNSUPPORTED
    with pytest.raises(F.FFTPDEError) as e:
        F.Plan3D(2, 2, 2048)                      # 4 lines: less than one 128-byte block for the col2 z-pass
    assert e.value.status == F.ERR_UNSUPPORTED
    p = F.Plan3D(16, 16, 8)
    x = torch.zeros(8, 16, 16, dtype=torch.complex128, device="cuda")
    st = p.lib.fftpde_wave_step(p._h, x.data_ptr(), torch.zeros_like(x).data_ptr(), 1.0, 0.1, 1)
    assert st == F.ERR_UNSUPPORTED
    st = p.lib.fftpde_poisson_batched(p._h, x.data_ptr(), x.data_ptr(), 1, 256)
    assert st == F.ERR_UNSUPPORTED


@pytest.mark.parametrize("shape,dtype,tol", [((2048, 4, 16), torch.complex128, 1e-12),
                                             ((4096, 8, 8), torch.complex128, 1e-12),
                                             ((32768, 2, 8), torch.complex128, 1e-12),
                                             ((2048, 8, 16), torch.complex64, 1e-5)])
def test_3d_long_z_two_level_pass(shape, dtype, tol):
    # nz > 1024: the z-pass is the two-level column pass (col2, nz = P Q) with the
    # plan's z tables, against the oracle (fft3 / poisson3 / diffuse3)
    nz, ny, nx = shape
    x = rand(shape, 277, np.complex64 if dtype == torch.complex64 else np.complex128)
    L = (1.0, 2.0, 0.5)
    p = F.Plan3D(nx, ny, nz, dtype=dtype, Lx=L[0], Ly=L[1], Lz=L[2])
    xd = torch.from_numpy(x).cuda()
    x64 = x.astype(np.complex128)
    assert rel(p.forward(xd).cpu().numpy(), O.fft3(x64)) <= tol
    assert rel(p.inverse(xd).cpu().numpy(), O.fft3(x64, inverse=True)) <= tol
    assert rel(p.poisson(xd).cpu().numpy(), O.poisson3(x64, *L)) <= tol
    assert rel(p.diffuse(xd, 1e-7, 0.01, 3).cpu().numpy(), O.diffuse3(x64, 1e-7, 0.01, 3, *L)) <= tol

