"""GPU parity of the real-field path through the C-ABI
(fftpde_plan_2d_r2c): the half spectrum against the oracle's complex DFT of the
same real data (bins a <= nx/2), and the real solves against the oracle's
complex solves of the real data (whose imaginary parts vanish)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2412_12308_b200 import fftpde as F
from paper_2412_12308_b200 import inputs as I

pytestmark = pytest.mark.gpu
F64, F32 = torch.float64, torch.float32


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b)))


SHAPES = [(16, 16), (32, 64), (64, 1024), (2, 128, 256), (2048, 16), (8, 16384), (4096, 32)]


@pytest.mark.parametrize("dtype,tol", [(F64, 1e-12), (F32, 1e-5)])
@pytest.mark.parametrize("shape", SHAPES)
def test_r2c_transforms_and_poisson(dtype, tol, shape):
    B = shape[0] if len(shape) == 3 else 1
    ny, nx = shape[-2:]
    if dtype == F32 and nx < 32:
        pytest.skip("complex64 real plans need nx >= 32")
    rng = np.random.default_rng(199)
    f = rng.standard_normal(shape).astype(np.float32 if dtype == F32 else np.float64)
    p = F.PlanR2C(nx, ny, batch=B, dtype=dtype, Lx=1.0, Ly=2.0)
    fd = torch.from_numpy(f).cuda()
    X = p.forward(fd).cpu().numpy()
    Xo = O.fft2(f.astype(np.complex128))[..., : nx // 2 + 1]
    assert rel(X, Xo) <= tol
    g = p.inverse(torch.from_numpy(Xo.astype(X.dtype)).cuda()).cpu().numpy()
    assert rel(g, f) <= tol
    u = p.poisson(fd).cpu().numpy()
    uo = O.poisson(f.astype(np.complex128), 1.0, 2.0)
    assert np.max(np.abs(uo.imag)) <= 1e-12 * np.max(np.abs(uo))
    assert rel(u, uo.real) <= tol


@pytest.mark.parametrize("dtype,tol", [(F64, 1e-12), (F32, 1e-5)])
@pytest.mark.parametrize("shape", [(64, 64), (128, 256), (2048, 32), (2, 64, 128)])
def test_r2c_diffuse_and_wave(dtype, tol, shape):
    B = shape[0] if len(shape) == 3 else 1
    ny, nx = shape[-2:]
    rng = np.random.default_rng(200)
    npdt = np.float32 if dtype == F32 else np.float64
    f = rng.standard_normal(shape).astype(npdt)
    g = rng.standard_normal(shape).astype(npdt)
    p = F.PlanR2C(nx, ny, batch=B, dtype=dtype)
    d = p.diffuse(torch.from_numpy(f).cuda(), 1e-3, 0.01, 7).cpu().numpy()
    assert rel(d, O.diffuse(f.astype(np.complex128), 1e-3, 0.01, 7).real) <= tol
    u, v = torch.from_numpy(f).cuda().clone(), torch.from_numpy(g).cuda().clone()
    p.wave_step(u, v, 1.2, 1e-3, 6)
    uo, vo = O.wave(f.astype(np.complex128), g.astype(np.complex128), 1.2, 1e-3, 6)
    assert rel(u.cpu().numpy(), uo.real) <= tol and rel(v.cpu().numpy(), vo.real) <= tol


def test_r2c_c2_workload_matches_complex_plan():
    # the C2 recipe on real storage agrees with the complex plan (imag = 0, R12)
    u0 = I.c2_inputs(1024).u0
    pr = F.PlanR2C(1024, 1024)
    pc = F.Plan(1024, 1024)
    ur = pr.diffuse(torch.from_numpy(u0.real.copy()).cuda(), 1e-3, 0.01, 20).cpu().numpy()
    uc = pc.diffuse(torch.from_numpy(u0).cuda(), 1e-3, 0.01, 20).cpu().numpy()
    assert rel(ur, uc.real) <= 1e-12 and np.max(np.abs(uc.imag)) <= 1e-13


def test_r2c_errors():
    with pytest.raises(F.FFTPDEError) as e:
        F.PlanR2C(8, 16)                            # nx < 2 x 128-byte column block
    assert e.value.status == F.ERR_UNSUPPORTED
    with pytest.raises(F.FFTPDEError) as e:
        F.PlanR2C(32768, 16)                        # rows beyond the single-CTA pass
    assert e.value.status == F.ERR_UNSUPPORTED
    p = F.PlanR2C(64, 64)
    x = torch.zeros(64, 64, dtype=F64, device="cuda")
    assert p.lib.fftpde_poisson_batched(p._h, x.data_ptr(), x.data_ptr(), 1, 4096) == F.ERR_UNSUPPORTED
