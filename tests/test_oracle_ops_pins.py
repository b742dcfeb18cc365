"""Pins of the oracle's diagonal k-space operators and the sourced diffusion
integrator: closed forms on exact single modes, the
spectral derivative of a smooth periodic function, the Poisson residual
identity, the Nyquist reading (R24), and the exact exponential
integrator's closed forms and semigroup property.  CPU only."""
import math

import numpy as np

from oracle import oracle as O

RNG = np.random.default_rng(369)


def mode(nx, ny, p, q):
    j, k = np.arange(nx), np.arange(ny)
    return np.outer(np.exp(2j * np.pi * ((q * k) % ny) / ny), np.exp(2j * np.pi * ((p * j) % nx) / nx))


def test_derivatives_of_single_modes():
    # d/dx e^{2 pi i p x/Lx} = (2 pi i p/Lx) e^{...} (F{du/dx} = -i w F{u})
    for nx, ny, Lx, Ly in [(32, 32, 1.0, 1.0), (64, 16, 2.0, 0.5), (16, 128, 1.5, 3.0)]:
        for p, q in [(1, 0), (0, 1), (3, -2), (-5, 4), (nx // 2 - 1, -(ny // 2 - 1))]:
            m = mode(nx, ny, p, q)
            dx = O.kspace_apply(m, "dx", Lx, Ly)
            dy = O.kspace_apply(m, "dy", Lx, Ly)
            lap = O.kspace_apply(m, "laplacian", Lx, Ly)
            kx, ky = 2 * math.pi * p / Lx, 2 * math.pi * q / Ly
            assert np.max(np.abs(dx - 1j * kx * m)) <= 1e-12 * max(1, abs(kx)), (p, q)
            assert np.max(np.abs(dy - 1j * ky * m)) <= 1e-12 * max(1, abs(ky)), (p, q)
            assert np.max(np.abs(lap + (kx * kx + ky * ky) * m)) <= 1e-12 * max(1, kx * kx + ky * ky)


def test_nyquist_reading_for_odd_operators():
    # R24: the Nyquist bin sits at +N/2 (R2), so d/dx of the real mode (-1)^j is
    # -i (pi N/L) (-1)^j: the sampled values cannot tell e^{+i pi N x/L} from
    # e^{-i pi N x/L}, and the paper's folding picks the bin's +f_c wavenumber.
    n, L = 16, 2.0
    u = np.tile((-1.0) ** np.arange(n), (n, 1)) + 0j
    d = O.kspace_apply(u, "dx", L, L)
    assert np.max(np.abs(d - (-1j * math.pi * n / L) * u)) <= 1e-12
    # even operators see no ambiguity: the Laplacian of the Nyquist mode is real
    lap = O.kspace_apply(u, "laplacian", L, L)
    assert np.max(np.abs(lap + (math.pi * n / L) ** 2 * u)) <= 1e-10


def test_spectral_derivative_of_smooth_periodic_function():
    n = 64
    x = np.arange(n) / n
    f = np.exp(np.sin(2 * np.pi * x))
    u = np.tile(f, (n, 1)) + 0j
    d = O.kspace_apply(u, "dx")
    exact = np.tile(2 * np.pi * np.cos(2 * np.pi * x) * f, (n, 1))
    assert np.max(np.abs(d - exact)) <= 1e-11
    assert np.max(np.abs(O.kspace_apply(u, "dy"))) <= 1e-12       # no y dependence


def test_poisson_residual():
    # SPEC poisson_residual: nabla^2 u = s - s_bar for u = poisson(s)
    s = RNG.standard_normal((32, 64)) + 1j * RNG.standard_normal((32, 64))
    u = O.poisson(s, 2.0, 1.0)
    r = O.kspace_apply(u, "laplacian", 2.0, 1.0)
    assert np.max(np.abs(r - (s - s.mean()))) <= 1e-12 * np.max(np.abs(s))


def test_diffuse_source_closed_forms():
    nx, ny, Lx, Ly, D = 32, 16, 1.0, 0.5, 0.02
    dt, steps = 0.05, 40
    T = steps * dt
    # single-mode source from rest: u(T) = (1 - e^{-D k^2 T})/(D k^2) s
    for p, q in [(1, 0), (2, -3), (5, 4)]:
        s = mode(nx, ny, p, q)
        k2 = (2 * math.pi * p / Lx) ** 2 + (2 * math.pi * q / Ly) ** 2
        u = O.diffuse_source(np.zeros((ny, nx)), s, D, dt, steps, Lx, Ly)
        assert np.max(np.abs(u + math.expm1(-D * k2 * T) / (D * k2) * s)) <= 1e-13
    # k = 0: the mean grows linearly, u_bar = u0_bar + T s_bar
    u0 = np.full((ny, nx), 0.3 + 0.1j)
    s = np.full((ny, nx), -0.7 + 0.2j)
    u = O.diffuse_source(u0, s, D, dt, steps, Lx, Ly)
    assert np.max(np.abs(u - (u0 + T * s))) <= 1e-13
    # D = 0: pure accumulation u = u0 + T s for every mode
    u0 = RNG.standard_normal((ny, nx)) + 0j
    s = RNG.standard_normal((ny, nx)) + 0j
    u = O.diffuse_source(u0, s, 0.0, dt, steps, Lx, Ly)
    assert np.max(np.abs(u - (u0 + T * s))) <= 1e-12
    # the exact integrator is a semigroup: 40 steps of dt == 1 step of 40 dt
    u1 = O.diffuse_source(u0, s, D, dt, steps, Lx, Ly)
    u2 = O.diffuse_source(u0, s, D, T, 1, Lx, Ly)
    assert np.max(np.abs(u1 - u2)) <= 1e-12 * np.max(np.abs(u2))


def test_diffuse_source_steady_state():
    # as t -> inf (mean-free s): D nabla^2 u = -s, i.e. u -> -poisson(s)/D
    n, D = 32, 0.5
    s = RNG.standard_normal((n, n)) + 0j
    s -= s.mean()
    u = O.diffuse_source(np.zeros((n, n)), s, D, 10.0, 4)       # e^{-D (2 pi)^2 40} ~ 1e-343
    assert np.max(np.abs(u + O.poisson(s) / D)) <= 1e-13
