"""Pins of the oracle's 3D extension ("extended analogously";
SURVEY.md 8(f) row 4): the brute-force triple sum of the 3D DFT on tiny grids,
exact single modes under the forward sign +, round trip and Parseval, the 3D
Poisson and diffusion closed forms.  CPU only."""
import math

import numpy as np

from oracle import oracle as O

RNG = np.random.default_rng(275)


def rand_c(shape):
    return RNG.standard_normal(shape) + 1j * RNG.standard_normal(shape)


def mode3(nx, ny, nz, p, q, r):
    j, k, l = np.arange(nx), np.arange(ny), np.arange(nz)
    ex = np.exp(2j * np.pi * ((p * j) % nx) / nx)
    ey = np.exp(2j * np.pi * ((q * k) % ny) / ny)
    ez = np.exp(2j * np.pi * ((r * l) % nz) / nz)
    return ez[:, None, None] * ey[None, :, None] * ex[None, None, :]


def test_fft3_equals_brute_force_triple_sum():
    for nz, ny, nx in [(2, 4, 4), (4, 2, 8), (4, 4, 4)]:
        x = rand_c((nz, ny, nx))
        X = O.fft3(x)
        for c, b, a in [(0, 0, 0), (1, 1, 3), (nz - 1, ny - 1, nx - 1), (1, 0, 2)]:
            s = 0j
            for l in range(nz):
                for k in range(ny):
                    for j in range(nx):
                        s += x[l, k, j] * O.root(nx, a * j) * O.root(ny, b * k) * O.root(nz, c * l)
            assert abs(X[c, b, a] - s) <= 1e-12 * max(1, abs(s))


def test_fft3_mode_lands_in_bin_minus_p_and_round_trip():
    nz, ny, nx = 8, 16, 32
    X = O.fft3(mode3(nx, ny, nz, 3, -5, 2))
    # forward sign +: e^{+2 pi i p x} lands in bin -p (R1)
    expect = np.zeros((nz, ny, nx), complex)
    expect[(-2) % nz, 5 % ny, (-3) % nx] = nx * ny * nz
    assert np.max(np.abs(X - expect)) <= 1e-10
    x = rand_c((nz, ny, nx))
    X = O.fft3(x)
    assert np.max(np.abs(O.fft3(X, inverse=True) - x)) <= 1e-13
    assert abs(np.sum(np.abs(X) ** 2) / (nx * ny * nz) / np.sum(np.abs(x) ** 2) - 1) <= 1e-13   # Parseval


def test_poisson3_and_diffuse3_single_modes():
    nz, ny, nx, Lx, Ly, Lz = 16, 8, 32, 1.0, 0.5, 2.0
    for p, q, r in [(1, 0, 0), (2, -3, 1), (0, 0, 5), (-7, 2, -4)]:
        m = mode3(nx, ny, nz, p, q, r)
        k2 = (2 * math.pi) ** 2 * ((p / Lx) ** 2 + (q / Ly) ** 2 + (r / Lz) ** 2)
        u = O.poisson3(m, Lx, Ly, Lz)
        assert np.max(np.abs(u + m / k2)) <= 1e-13 / k2 * 10
        d = O.diffuse3(m, 1e-3, 0.01, 20, Lx, Ly, Lz)
        assert np.max(np.abs(d - math.exp(-1e-3 * k2 * 0.2) * m)) <= 1e-13
    # zero mode: Poisson ignores the mean, diffusion keeps it
    c = np.full((nz, ny, nx), 0.25 - 0.5j)
    assert np.max(np.abs(O.poisson3(c))) <= 1e-15
    assert np.max(np.abs(O.diffuse3(c, 0.1, 0.1, 5) - c)) <= 1e-15
    # a field independent of z reduces to the 2D solve on every slab
    s2 = rand_c((ny, nx))
    vol = np.broadcast_to(s2, (nz, ny, nx)).copy()
    assert np.max(np.abs(O.poisson3(vol, Lx, Ly, Lz) - O.poisson(s2, Lx, Ly)[None])) <= 1e-13
