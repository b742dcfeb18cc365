"""Seeded synthetic inputs for the five BASELINE.json workloads (C1..C5).

This module is shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side.  It holds NONE of the method's arithmetic: it only draws random
numbers and samples analytic fields on the grid.  Both sides receive the same
bytes.  Recipe:

* generator ``numpy.random.Generator(PCG64(12308 + i))`` for config i = 1..5;
* grid ``x_j = j Lx/nx``, ``y_k = k Ly/ny`` on [0,1)^2, array index ``[k, j]``
  (vertex sampling; R15);
* Gaussians ``A exp(-d^2/sigma^2)`` -- the paper's form (PAPER.md:338, 392,
  492) -- with ``d`` the periodic minimum-image distance (R9);
* imaginary parts exactly 0 (R12).

The C4 source is white noise low-pass filtered to integer mode radius < 64
(R11); the filter is applied with ``numpy.fft`` as part of input
generation only (the mask is symmetric, so the library's sign convention is
irrelevant).  Sizes can be reduced (``n=...``) for tests; the recipe is the same.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 12308


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    op: str            # "poisson" | "diffuse" | "wave"
    nx: int
    ny: int
    batch: int
    dtype: str         # "c128" | "c64"
    nsteps: int = 1
    D: float = 0.0
    dt: float = 0.0
    c: float = 0.0
    Lx: float = 1.0
    Ly: float = 1.0
    nz: int = 1            # 3D workloads

    @property
    def points(self) -> int:
        return self.nx * self.ny * self.nz * self.batch


# BASELINE.json configs[0..4]
C1 = Workload("c1_poisson_64", "poisson", 64, 64, 1, "c128")
C2 = Workload("c2_diffusion_1024", "diffuse", 1024, 1024, 1, "c128", nsteps=200, D=1e-3, dt=0.01)
C3 = Workload("c3_wave_4096", "wave", 4096, 4096, 1, "c128", nsteps=500, c=1.0, dt=1e-4)
C4 = Workload("c4_batched_poisson_256x512", "poisson", 512, 512, 256, "c64")
C5 = Workload("c5_diffusion_32768", "diffuse", 32768, 32768, 1, "c128", nsteps=20, D=1e-4, dt=0.01)
WORKLOADS = {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c5": C5}

# SURVEY.md 8(f) row 1 (not a BASELINE config): the paper's orbiting-source wave run,
# D = [-2, 2]^2, dt = 0.25 h, t in [0, 2.5], and a B200-sized variant.
RK4 = Workload("rk4_orbit_256", "rk4", 256, 256, 1, "c128", nsteps=640, dt=0.25 * 4.0 / 256, c=1.0,
               Lx=4.0, Ly=4.0)
RK4_BIG = Workload("rk4_orbit_4096", "rk4", 4096, 4096, 1, "c128", nsteps=50, dt=0.25 * 4.0 / 4096, c=1.0,
                   Lx=4.0, Ly=4.0)
# SURVEY.md 8(f) row 2 (not a BASELINE config): diffusion with a static source, the C2
# grid and Gaussians as both the initial field and the source (exact integrator per step)
DSRC = Workload("dsrc_diffusion_1024", "dsrc", 1024, 1024, 1, "c128", nsteps=200, D=1e-3, dt=0.01)
# SURVEY.md 8(f) row 4 (not a BASELINE config): the 3D extension on 256^3
P3D = Workload("p3d_poisson_256", "poisson", 256, 256, 1, "c128", nz=256)
D3D = Workload("d3d_diffusion_256", "diffuse", 256, 256, 1, "c128", nsteps=20, D=1e-3, dt=0.01, nz=256)
# SURVEY.md 8(f) row 3 (not BASELINE configs): the C2 / C3 / C4 recipes on REAL storage
# (their data are real, R12), through the half-spectrum path
C2R = dataclasses.replace(C2, name="c2r_diffusion_1024_real", dtype="f64")
C3R = dataclasses.replace(C3, name="c3r_wave_4096_real", dtype="f64")
C4R = dataclasses.replace(C4, name="c4r_batched_poisson_256x512_real", dtype="f32")
EXTRA_WORKLOADS = {"rk4": RK4, "rk4big": RK4_BIG, "dsrc": DSRC, "p3d": P3D, "d3d": D3D,
                   "c2r": C2R, "c3r": C3R, "c4r": C4R}


def rng_for(config_index: int) -> np.random.Generator:
    """PCG64 stream for config i (1-based, BASELINE.json configs[i-1])."""
    return np.random.Generator(np.random.PCG64(SEED_BASE + config_index))


def axis(n: int, L: float = 1.0) -> np.ndarray:
    """Vertex-sampled coordinates x_j = j L/n, j = 0..n-1."""
    return np.arange(n, dtype=np.float64) * (L / n)


def min_image(x: np.ndarray, c: float, L: float = 1.0) -> np.ndarray:
    """Signed periodic minimum-image displacement x - c in [-L/2, L/2)."""
    return np.mod(x - c + 0.5 * L, L) - 0.5 * L


def gaussian_1d(n: int, c: float, sigma: float, L: float = 1.0) -> np.ndarray:
    d = min_image(axis(n, L), c, L)
    return np.exp(-(d * d) / (sigma * sigma))


def add_gaussian(field: np.ndarray, cx: float, cy: float, sigma: float, amp: float,
                 window: int | None = None) -> None:
    """field[k, j] += amp exp(-(dx^2 + dy^2)/sigma^2), evaluated separably.

    With ``window`` only the +-window points around the centre are touched
    (periodically wrapped); used for the 32768^2 C5 field where the Gaussian is
    below 1e-18 outside 6.5 sigma."""
    ny, nx = field.shape
    if window is None or 2 * window + 1 >= min(nx, ny):
        gx = gaussian_1d(nx, cx, sigma)
        gy = gaussian_1d(ny, cy, sigma)
        field += amp * np.outer(gy, gx)
        return
    jx = int(round(cx * nx))
    jy = int(round(cy * ny))
    ix = np.arange(jx - window, jx + window + 1) % nx
    iy = np.arange(jy - window, jy + window + 1) % ny
    dx = min_image(ix / nx, cx)
    dy = min_image(iy / ny, cy)
    gx = np.exp(-(dx * dx) / (sigma * sigma))
    gy = np.exp(-(dy * dy) / (sigma * sigma))
    field[np.ix_(iy, ix)] += amp * np.outer(gy, gx)


# ---------------------------------------------------------------------------
# C1: 2D Poisson on 64x64, rho = -8 pi^2 sin(2pi x) sin(2pi y) + 4 blobs, mean removed

@dataclasses.dataclass
class PoissonC1:
    rho: np.ndarray          # [n, n] complex128, mean subtracted
    rho_sin: np.ndarray      # sinusoid part alone (mean subtracted)
    rho_blobs: np.ndarray    # blob part alone (mean subtracted)
    centres: np.ndarray
    amps: np.ndarray
    sigma: float


def c1_inputs(n: int = 64) -> PoissonC1:
    rng = rng_for(1)
    centres = rng.random((4, 2))
    amps = rng.uniform(-1.0, 1.0, 4)
    sigma = 0.05
    x = axis(n)
    sin_part = -8.0 * math.pi ** 2 * np.outer(np.sin(2 * math.pi * x), np.sin(2 * math.pi * x))
    blobs = np.zeros((n, n))
    for (cx, cy), a in zip(centres, amps):
        add_gaussian(blobs, cx, cy, sigma, a)
    sin_part = sin_part - sin_part.mean()
    blobs = blobs - blobs.mean()
    rho = sin_part + blobs
    rho = rho - rho.mean()
    return PoissonC1(rho.astype(np.complex128), sin_part.astype(np.complex128),
                     blobs.astype(np.complex128), centres, amps, sigma)


# ---------------------------------------------------------------------------
# C2: diffusion, 16 Gaussians, sigma ~ U(0.01, 0.05), amplitudes U(0,1)

@dataclasses.dataclass
class GaussianField:
    u0: np.ndarray           # [n, n] complex128
    centres: np.ndarray      # [m, 2] (cx, cy)
    sigmas: np.ndarray
    amps: np.ndarray


def gaussian_params(config_index: int, m: int, sig_lo: float, sig_hi: float):
    rng = rng_for(config_index)
    centres = rng.random((m, 2))
    sigmas = rng.uniform(sig_lo, sig_hi, m)
    amps = rng.uniform(0.0, 1.0, m)
    return centres, sigmas, amps


def c2_inputs(n: int = 1024, m: int = 16, sig_lo: float = 0.01, sig_hi: float = 0.05) -> GaussianField:
    centres, sigmas, amps = gaussian_params(2, m, sig_lo, sig_hi)
    f = np.zeros((n, n))
    for (cx, cy), s, a in zip(centres, sigmas, amps):
        add_gaussian(f, cx, cy, s, a)
    return GaussianField(f.astype(np.complex128), centres, sigmas, amps)


# ---------------------------------------------------------------------------
# C3: wave, Gaussian pulse sigma = 0.02 (A = 1) + 1e-3 N(0,1) white noise, u_t = 0

@dataclasses.dataclass
class WaveC3:
    u: np.ndarray
    ut: np.ndarray
    centre: np.ndarray
    sigma: float
    noise: float


def c3_inputs(n: int = 4096, sigma: float = 0.02, noise: float = 1e-3) -> WaveC3:
    rng = rng_for(3)
    centre = rng.random(2)
    u = np.zeros((n, n))
    add_gaussian(u, centre[0], centre[1], sigma, 1.0)
    if noise:
        u += noise * rng.standard_normal((n, n))
    return WaveC3(u.astype(np.complex128), np.zeros((n, n), np.complex128), centre, sigma, noise)


# ---------------------------------------------------------------------------
# C4: 256 independent 512^2 sources: N(0,1) noise, integer mode radius < 64 kept,
# mean subtracted, cast to complex64.

def lowpass_mask(n: int, kmax: float = 64.0) -> np.ndarray:
    f = np.fft.fftfreq(n, d=1.0 / n)          # integer mode numbers, symmetric
    r2 = f[None, :] ** 2 + f[:, None] ** 2
    return r2 < kmax * kmax


def c4_inputs(n: int = 512, batch: int = 256, kmax: float = 64.0) -> np.ndarray:
    rng = rng_for(4)
    mask = lowpass_mask(n, kmax)
    out = np.empty((batch, n, n), np.complex64)
    for g in range(batch):
        w = rng.standard_normal((n, n))
        s = np.fft.ifft2(np.fft.fft2(w) * mask).real
        s -= s.mean()
        out[g] = s.astype(np.complex64)
    return out


# ---------------------------------------------------------------------------
# C5: 1024 Gaussians sigma ~ U(0.001, 0.01) on 32768^2 (windowed at 6.5 sigma)

def c5_params(m: int = 1024):
    return gaussian_params(5, m, 0.001, 0.01)


def c5_inputs(n: int = 32768, m: int = 1024, sig_lo: float = 0.001, sig_hi: float = 0.01) -> GaussianField:
    rng = rng_for(5)
    centres = rng.random((m, 2))
    sigmas = rng.uniform(sig_lo, sig_hi, m)
    amps = rng.uniform(0.0, 1.0, m)
    f = np.zeros((n, n))
    for (cx, cy), s, a in zip(centres, sigmas, amps):
        add_gaussian(f, cx, cy, s, a, window=int(math.ceil(6.5 * s * n)))
    return GaussianField(f.astype(np.complex128), centres, sigmas, amps)


def c5_field_torch(n: int = 32768, m: int = 1024, sig_lo: float = 0.001, sig_hi: float = 0.01,
                   device="cuda", dtype=None):
    """The C5 initial condition built directly in device memory (a 32768^2
    complex128 field is 16 GiB): the same PCG64 draws as c5_inputs, each
    Gaussian evaluated separably in fp64 by torch over its +-6.5 sigma window
    (periodically wrapped) and accumulated.  Returns (field, centres, sigmas, amps)."""
    import torch
    rng = rng_for(5)
    centres = rng.random((m, 2))
    sigmas = rng.uniform(sig_lo, sig_hi, m)
    amps = rng.uniform(0.0, 1.0, m)
    dtype = dtype or torch.complex128
    f = torch.zeros((n, n), dtype=torch.float64, device=device)
    for (cx, cy), s, a in zip(centres, sigmas, amps):
        w = int(math.ceil(6.5 * s * n))
        if 2 * w + 1 >= n:
            ix = torch.arange(n, device=device)
            iy = ix
        else:
            ix = torch.arange(int(round(cx * n)) - w, int(round(cx * n)) + w + 1, device=device) % n
            iy = torch.arange(int(round(cy * n)) - w, int(round(cy * n)) + w + 1, device=device) % n
        dx = torch.remainder(ix.to(torch.float64) / n - cx + 0.5, 1.0) - 0.5
        dy = torch.remainder(iy.to(torch.float64) / n - cy + 0.5, 1.0) - 0.5
        gx = torch.exp(-(dx * dx) / (s * s))
        gy = torch.exp(-(dy * dy) / (s * s))
        f.index_put_((iy[:, None].expand(-1, ix.numel()), ix[None, :].expand(iy.numel(), -1)),
                     a * torch.outer(gy, gx), accumulate=True)
    return f.to(dtype), centres, sigmas, amps


def white_noise(shape, seed: int, dtype=np.complex128, complex_valued: bool = True) -> np.ndarray:
    """Generic seeded complex test data (parity tests of the raw transforms)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape) if complex_valued else np.zeros(shape)
    return (re + 1j * im).astype(dtype)


def gaussians_3d(n: int = 256, m: int = 16, seed_index: int = 6) -> np.ndarray:
    """Sum of m seeded 3D Gaussians A exp(-d^2/sigma^2) on [0,1)^3 (minimum image,
    the C2 recipe extended to 3D), mean subtracted; [n, n, n] complex128."""
    rng = rng_for(seed_index)
    centres = rng.random((m, 3))
    sigmas = rng.uniform(0.02, 0.08, m)
    amps = rng.uniform(0.0, 1.0, m)
    f = np.zeros((n, n, n))
    for (cx, cy, cz), s, a in zip(centres, sigmas, amps):
        gx, gy, gz = gaussian_1d(n, cx, s), gaussian_1d(n, cy, s), gaussian_1d(n, cz, s)
        f += a * gz[:, None, None] * gy[None, :, None] * gx[None, None, :]
    f -= f.mean()
    return f.astype(np.complex128)
