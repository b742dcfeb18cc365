"""GPU parity of the diagonal k-space operators and the sourced diffusion
integrator through the C-ABI, against the fp64 oracle
on the same seeded inputs; plus closed forms evaluated on the GPU results."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F

pytestmark = pytest.mark.gpu
C128, C64 = torch.complex128, torch.complex64


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b)))


def rand(shape, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype)


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
@pytest.mark.parametrize("shape,L", [((64, 64), (1.0, 1.0)), ((32, 128), (2.0, 0.5)), ((3, 16, 256), (1.0, 3.0)),
                                     ((2048, 16), (1.0, 1.0)), ((8, 16384), (4.0, 1.0))])
def test_kspace_apply_parity(dtype, tol, shape, L):
    B = shape[0] if len(shape) == 3 else 1
    ny, nx = shape[-2:]
    x = rand(shape, 296, np.complex64 if dtype == C64 else np.complex128)
    p = F.Plan(nx, ny, batch=B, dtype=dtype, Lx=L[0], Ly=L[1])
    xd = torch.from_numpy(x).cuda()
    for op in ("laplacian", "dx", "dy"):
        g = p.apply(xd, op).cpu().numpy()
        o = O.kspace_apply(x.astype(np.complex128), op, L[0], L[1])
        assert rel(g, o) <= tol, (op, rel(g, o))


def test_kspace_apply_modes_and_nyquist_on_gpu():
    n, L = 64, 2.0
    j = np.arange(n)
    m = np.outer(np.exp(2j * np.pi * ((-7 * j) % n) / n), np.exp(2j * np.pi * ((5 * j) % n) / n))
    p = F.Plan(n, n, Lx=L, Ly=L)
    d = p.apply(torch.from_numpy(m).cuda(), "dx").cpu().numpy()
    assert np.max(np.abs(d - 1j * (2 * math.pi * 5 / L) * m)) <= 1e-12 * 2 * math.pi * 5 / L
    d = p.apply(torch.from_numpy(m).cuda(), "dy").cpu().numpy()
    assert np.max(np.abs(d - 1j * (2 * math.pi * -7 / L) * m)) <= 1e-12 * 2 * math.pi * 7 / L
    ny = np.tile((-1.0) ** j, (n, 1)) + 0j               # Nyquist reading R24
    d = p.apply(torch.from_numpy(ny).cuda(), "dx").cpu().numpy()
    assert np.max(np.abs(d - (-1j * math.pi * n / L) * ny)) <= 1e-10


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
@pytest.mark.parametrize("shape", [(64, 64), (128, 32), (2, 64, 128), (2048, 16)])
def test_diffuse_source_parity(dtype, tol, shape):
    B = shape[0] if len(shape) == 3 else 1
    ny, nx = shape[-2:]
    npdt = np.complex64 if dtype == C64 else np.complex128
    u0 = rand(shape, 355, npdt)
    s = rand(shape, 356, npdt)
    D, dt, steps = 2e-3, 0.05, 12
    p = F.Plan(nx, ny, batch=B, dtype=dtype)
    g = p.diffuse_source(torch.from_numpy(u0).cuda(), torch.from_numpy(s).cuda(), D, dt, steps).cpu().numpy()
    o = O.diffuse_source(u0.astype(np.complex128), s.astype(np.complex128), D, dt, steps)
    assert rel(g, o) <= tol


def test_diffuse_source_closed_form_on_gpu():
    nx, ny, D, dt, steps = 64, 32, 0.01, 0.1, 30
    T = dt * steps
    j, k = np.arange(nx), np.arange(ny)
    s = np.outer(np.exp(2j * np.pi * ((3 * k) % ny) / ny), np.exp(2j * np.pi * ((-2 * j) % nx) / nx))
    k2 = (2 * math.pi * 2) ** 2 + (2 * math.pi * 3) ** 2
    p = F.Plan(nx, ny)
    u = p.diffuse_source(torch.zeros(ny, nx, dtype=C128, device="cuda"), torch.from_numpy(s).cuda(), D, dt,
                         steps).cpu().numpy()
    assert np.max(np.abs(u + math.expm1(-D * k2 * T) / (D * k2) * s)) <= 1e-13
    # nsteps = 0 copies u0; bad arguments are reported
    x = torch.randn(ny, nx, dtype=C128, device="cuda")
    assert torch.equal(p.diffuse_source(x, x, D, dt, 0), x)
    with pytest.raises(F.FFTPDEError) as e:
        p.diffuse_source(x, x, -1.0, dt, 2)
    assert e.value.status == F.ERR_INVALID_ARG
    with pytest.raises(F.FFTPDEError) as e:
        F._check(p.lib.fftpde_apply(p._h, x.data_ptr(), x.data_ptr(), 7), "fftpde_apply")   # unknown op
    assert e.value.status == F.ERR_INVALID_ARG
