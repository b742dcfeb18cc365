"""ctypes wrapper of the fp64 CPU oracle (oracle/fftpde_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_2412_12308_b200``.  Shares no code with the CUDA path.

Every function takes and returns numpy complex128 arrays (interleaved re/im,
exactly the C ``double[2]`` layout).  Grids are ``[ny, nx]`` or ``[B, ny, nx]``
with x fastest.  See fftpde_oracle.c for the paper
citations of each operation.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fftpde_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (no -ffast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, dbl, p = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        sig = {
            "oracle_root": [i64, i64, p],
            "oracle_dft1": [i64, p, p, ctypes.c_int],
            "oracle_dft1_at": [i64, p, i64, p],
            "oracle_fft1": [i64, p, p, ctypes.c_int],
            "oracle_dft2_direct": [i64, i64, p, p, ctypes.c_int],
            "oracle_fft2": [i64, i64, i64, p, p, ctypes.c_int, ctypes.c_int],
            "oracle_wavenumbers": [i64, dbl, p],
            "oracle_poisson": [i64, i64, i64, dbl, dbl, p, p, ctypes.c_int],
            "oracle_diffuse": [i64, i64, i64, dbl, dbl, dbl, dbl, i64, p, p,
                               ctypes.c_int, ctypes.c_int],
            "oracle_wave": [i64, i64, i64, dbl, dbl, dbl, dbl, i64, p, p,
                            ctypes.c_int, ctypes.c_int],
            "oracle_fft3": [i64, i64, i64, p, p, ctypes.c_int],
            "oracle_solve3": [i64, i64, i64, dbl, dbl, dbl, ctypes.c_int, dbl, dbl, i64, p],
            "oracle_kspace_apply": [i64, i64, i64, dbl, dbl, ctypes.c_int, p, p],
            "oracle_diffuse_source": [i64, i64, i64, dbl, dbl, dbl, dbl, i64, p, p],
            "oracle_orbit_source": [i64, i64, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, p],
            "oracle_wave_rk4": [i64, i64, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, dbl, i64,
                                p, p, p],
            "oracle_set_threads": [ctypes.c_int],
            "oracle_get_threads": [],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(ValueError):
    pass


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _check(rc: int, what: str):
    if rc == -2:
        raise OracleError(f"{what}: axis length is not a power of two (radix-2 restriction)")
    if rc != 0:
        raise OracleError(f"{what}: invalid argument (rc={rc})")


def _grid(a):
    a = _c128(a)
    if a.ndim == 2:
        return a, 1, a.shape[0], a.shape[1]
    if a.ndim == 3:
        return a, a.shape[0], a.shape[1], a.shape[2]
    raise OracleError("expected [ny, nx] or [B, ny, nx]")


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return lib().oracle_get_threads()


def root(n: int, m: int) -> complex:
    """w_n^m = exp(+2 pi i m/n)."""
    out = np.zeros(2)
    _check(lib().oracle_root(n, m, out.ctypes.data), "root")
    return complex(out[0], out[1])


def dft(x, inverse: bool = False) -> np.ndarray:
    """Path 1, direct O(N^2) sum: eq:DFT / iDFT."""
    x = _c128(x)
    X = np.empty_like(x)
    _check(lib().oracle_dft1(x.size, x.ctypes.data, X.ctypes.data, int(inverse)), "dft")
    return X


def dft_at(x, k: int) -> complex:
    """The eq:DFT sum evaluated at any integer k (periodicity)."""
    x = _c128(x)
    out = np.zeros(2)
    _check(lib().oracle_dft1_at(x.size, x.ctypes.data, int(k), out.ctypes.data), "dft_at")
    return complex(out[0], out[1])


def fft(x, inverse: bool = False) -> np.ndarray:
    """Path 2, recursive radix-2 FFT; inverse via conj trick (:157-159)."""
    x = _c128(x)
    X = np.empty_like(x)
    _check(lib().oracle_fft1(x.size, x.ctypes.data, X.ctypes.data, int(inverse)), "fft")
    return X


def dft2_direct(p, inverse: bool = False) -> np.ndarray:
    """Brute-force double sum of 2D_DFT; tiny grids only."""
    p = _c128(p)
    if p.ndim != 2:
        raise OracleError("dft2_direct expects [ny, nx]")
    P = np.empty_like(p)
    _check(lib().oracle_dft2_direct(p.shape[1], p.shape[0], p.ctypes.data, P.ctypes.data,
                                    int(inverse)), "dft2_direct")
    return P


def fft2(p, inverse: bool = False, path: int = 2) -> np.ndarray:
    """2D transform by rows then columns; path 1 direct, path 2 FFT."""
    p, B, ny, nx = _grid(p)
    out = np.empty_like(p)
    _check(lib().oracle_fft2(nx, ny, B, p.ctypes.data, out.ctypes.data, int(inverse), path),
           "fft2")
    return out


def wavenumbers(n: int, L: float) -> np.ndarray:
    """k[a] = 2 pi fold(a)/L, Nyquist at +n/2."""
    k = np.empty(n)
    _check(lib().oracle_wavenumbers(n, float(L), k.ctypes.data), "wavenumbers")
    return k


def poisson(rho, Lx: float = 1.0, Ly: float = 1.0, path: int = 2) -> np.ndarray:
    """u = F^-1{-F{g}/|k|^2}, k=0 zeroed (eq:SolutionPoisson)."""
    rho, B, ny, nx = _grid(rho)
    u = np.empty_like(rho)
    _check(lib().oracle_poisson(nx, ny, B, Lx, Ly, rho.ctypes.data, u.ctypes.data, path),
           "poisson")
    return u


def diffuse(u0, D: float, dt: float, nsteps: int, Lx: float = 1.0, Ly: float = 1.0,
            collapsed: bool = False, path: int = 2) -> np.ndarray:
    """nsteps x (F, exp(-D|k|^2 dt), F^-1) (ec:solCalorFourier)."""
    u0, B, ny, nx = _grid(u0)
    u = np.empty_like(u0)
    _check(lib().oracle_diffuse(nx, ny, B, Lx, Ly, D, dt, int(nsteps), u0.ctypes.data,
                                u.ctypes.data, int(collapsed), path), "diffuse")
    return u


def wave(u, ut, c: float, dt: float, nsteps: int, Lx: float = 1.0, Ly: float = 1.0,
         collapsed: bool = False, path: int = 2):
    """Exact oscillator steps on (u^, v^) (eq:OmegaZero/NonZero).

    Returns new arrays (u, ut); the inputs are not modified."""
    u, B, ny, nx = _grid(u)
    ut = _c128(ut)
    if ut.shape != u.shape:
        raise OracleError("u and ut shapes differ")
    U = u.copy()
    V = ut.copy()
    _check(lib().oracle_wave(nx, ny, B, Lx, Ly, c, dt, int(nsteps), U.ctypes.data,
                             V.ctypes.data, int(collapsed), path), "wave")
    return U, V


def orbit_source(nx: int, ny: int, t: float, Lx: float = 4.0, Ly: float = 4.0, xmin: float = -2.0,
                 ymin: float = -2.0, A: float = 1.0, sigma: float = 0.1, Omega: float = 5.0,
                 gamma: float = 10.0, rs: float = 0.5) -> np.ndarray:
    """Orbiting Gaussian source s(t, x_j, y_k), [ny, nx] complex128."""
    out = np.empty((ny, nx), np.complex128)
    _check(lib().oracle_orbit_source(nx, ny, Lx, Ly, xmin, ymin, A, sigma, Omega, gamma, rs, t,
                                     out.ctypes.data), "orbit_source")
    return out


def wave_rk4(u, ut, dt: float, nsteps: int, c: float = 1.0, t0: float = 0.0, Lx: float = 4.0,
             Ly: float = 4.0, xmin: float = -2.0, ymin: float = -2.0, A: float = 1.0,
             sigma: float = 0.1, Omega: float = 5.0, gamma: float = 10.0, rs: float = 0.5):
    """RK4 on du^/dt = v^, dv^/dt = -(c|k|)^2 u^ + s^(t) with the orbiting source
    (PAPER.md:448-456, 516-523).  Returns (u, ut, means) at t0 + nsteps dt; means[n]
    is the grid mean of u at t0 + n dt."""
    u = _c128(u).copy()
    ut = _c128(ut).copy()
    if u.ndim != 2 or u.shape != ut.shape:
        raise OracleError("wave_rk4 expects two [ny, nx] fields")
    ny, nx = u.shape
    means = np.empty(nsteps + 1, np.complex128)
    _check(lib().oracle_wave_rk4(nx, ny, Lx, Ly, xmin, ymin, c, A, sigma, Omega, gamma, rs, t0, dt,
                                 nsteps, u.ctypes.data, ut.ctypes.data, means.ctypes.data), "wave_rk4")
    return u, ut, means


KOPS = {"laplacian": 0, "dx": 1, "dy": 2}


def kspace_apply(p, op: str, Lx: float = 1.0, Ly: float = 1.0) -> np.ndarray:
    """F^-1{m F{p}}, m = -|k|^2 (laplacian), -i kx (dx), -i ky (dy)."""
    p, B, ny, nx = _grid(p)
    out = np.empty_like(p)
    _check(lib().oracle_kspace_apply(nx, ny, B, Lx, Ly, KOPS[op], p.ctypes.data, out.ctypes.data),
           "kspace_apply")
    return out


def diffuse_source(u0, s, D: float, dt: float, nsteps: int, Lx: float = 1.0, Ly: float = 1.0) -> np.ndarray:
    """nsteps exact steps of u_t = D nabla^2 u + s, static s."""
    u, B, ny, nx = _grid(u0)
    u = u.copy()
    s, Bs, nys, nxs = _grid(s)
    if (Bs, nys, nxs) != (B, ny, nx):
        raise OracleError("diffuse_source: u0 and s shapes differ")
    _check(lib().oracle_diffuse_source(nx, ny, B, Lx, Ly, D, dt, nsteps, u.ctypes.data, s.ctypes.data),
           "diffuse_source")
    return u


def _vol(a):
    a = _c128(a)
    if a.ndim != 3:
        raise OracleError("expected a [nz, ny, nx] volume")
    return a, a.shape[2], a.shape[1], a.shape[0]


def fft3(p, inverse: bool = False) -> np.ndarray:
    """3D transform by sequential 1D transforms along x, y, z."""
    p, nx, ny, nz = _vol(p)
    out = np.empty_like(p)
    _check(lib().oracle_fft3(nx, ny, nz, p.ctypes.data, out.ctypes.data, int(inverse)), "fft3")
    return out


def poisson3(rho, Lx: float = 1.0, Ly: float = 1.0, Lz: float = 1.0) -> np.ndarray:
    """3D Poisson, -1/|k|^2 with k = 0 zeroed (eq:SolutionPoisson extended)."""
    u, nx, ny, nz = _vol(rho)
    u = u.copy()
    _check(lib().oracle_solve3(nx, ny, nz, Lx, Ly, Lz, 0, 0.0, 0.0, 1, u.ctypes.data), "poisson3")
    return u


def diffuse3(u0, D: float, dt: float, nsteps: int, Lx: float = 1.0, Ly: float = 1.0,
             Lz: float = 1.0) -> np.ndarray:
    """nsteps exact 3D diffusion steps exp(-D|k|^2 dt)."""
    u, nx, ny, nz = _vol(u0)
    u = u.copy()
    _check(lib().oracle_solve3(nx, ny, nz, Lx, Ly, Lz, 1, D, dt, nsteps, u.ctypes.data), "diffuse3")
    return u
