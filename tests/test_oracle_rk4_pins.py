"""Pins of the oracle's time-dependent-source path:
the orbiting Gaussian source and the RK4 integration of the
Fourier-space first-order system (eq:SystemOfODEsForWaveEquation,
PAPER.md:448-454).  Every check is a closed form, an exact identity or the
paper's own convergence claim -- never the oracle against itself.  CPU only.
"""
import math

import numpy as np

from oracle import oracle as O

L, XMIN = 4.0, -2.0                  # D = [-2, 2]^2


def grid(n):
    return XMIN + np.arange(n) * (L / n)


def test_orbit_source_examples():
    n, sig = 128, 0.1
    h = L / n
    # cos(gamma t) = 0 -> identically zero (SPEC orbiting_source_eval example)
    s = O.orbit_source(n, n, math.pi / 20.0, gamma=10.0)
    assert np.max(np.abs(s)) <= 1e-15
    # r_s = 0, t = 0: centred Gaussian, peak A at the grid point x = y = 0, and the
    # grid sum is the integral pi sigma^2 (spectrally accurate for sigma/h = 3.2)
    s = O.orbit_source(n, n, 0.0, rs=0.0, A=1.7)
    assert s[n // 2, n // 2] == 1.7
    assert abs(s.real.sum() * h * h / (1.7 * math.pi * sig * sig) - 1) <= 1e-13
    assert np.all(s.imag == 0)
    # the centre follows x0 = r_s cos(Omega t), y0 = r_s sin(Omega t): at Omega t = pi/2
    # the peak sits at (0, r_s) = (0, 0.5) -> row (0.5 + 2)/h = 80, column 64
    s = O.orbit_source(n, n, math.pi / 10.0, Omega=5.0, gamma=0.0, rs=0.5)
    k, j = np.unravel_index(np.argmax(s.real), s.shape)
    assert (k, j) == (80, 64)
    # joint periodicity: t = 2 pi / Omega with gamma 2 pi / Omega = 4 pi -> s(t) = s(0)
    assert np.max(np.abs(O.orbit_source(n, n, 2 * math.pi / 5.0) - O.orbit_source(n, n, 0.0))) <= 1e-12
    # periodic minimum image: a centre at x0 = 1.95 is 0.05 from the node x = -2
    s = O.orbit_source(n, n, 0.0, rs=1.95, gamma=0.0, Omega=0.0)
    assert abs(s[n // 2, 0].real - math.exp(-(0.05 / sig) ** 2)) <= 1e-14   # 1.95, 0.05 inexact in binary


def test_rk4_free_modes_fourth_order():
    # s = 0: a single standing mode oscillates as cos(kappa t) (eq:OmegaNonZero);
    # the RK4 error falls by 2^4 per halving of dt (SPEC acceptance 13: [3.8, 4.2])
    n, c, T = 32, 1.0, 1.0
    x = grid(n)
    f = np.outer(np.cos(2 * np.pi * 2 * x / L), np.sin(2 * np.pi * 3 * x / L))
    kappa = c * 2 * np.pi * math.hypot(2, 3) / L
    errs = []
    for dt in (1 / 16, 1 / 32, 1 / 64):
        u, v, m = O.wave_rk4(f, np.zeros_like(f), dt, int(round(T / dt)), c=c, A=0.0)
        errs.append(np.max(np.abs(u - math.cos(kappa * T) * f)))
        assert np.max(np.abs(v + kappa * math.sin(kappa * T) * f)) <= 50 * errs[-1] * kappa
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(3.8 <= o <= 4.2 for o in orders), orders
    # RK4 on an oscillator: phase error ~ kappa (kappa dt)^4 / 120 per unit time
    dt = 1 / 64
    assert errs[-1] <= 2 * kappa * (kappa * dt) ** 4 / 120 * T


def test_rk4_static_source_matches_forced_oscillator():
    # gamma = Omega = 0: a static source; from rest the exact modal solution is
    # u^ = s^ (1 - cos kappa t)/kappa^2 (kappa > 0), s^ t^2/2 (kappa = 0)
    # (eq:OmegaZero / eq:OmegaNonZero with the +s^/omega^2 term).
    # SPEC acceptance 9: 1e-6 max-norm for u at dt = 0.25 h over t in [0, 2]; both
    # fields converge at fourth order as dt halves.
    n, c = 64, 1.0
    h = L / n
    s = O.orbit_source(n, n, 0.0, gamma=0.0, Omega=0.0, rs=0.5)
    k = 2 * np.pi * np.fft.fftfreq(n, d=h)
    kap2 = c * c * (k[None, :] ** 2 + k[:, None] ** 2)
    S = np.fft.fft2(s)                      # any sign convention: the factor is even in k
    errs = []
    for dt in (0.25 * h, 0.125 * h):
        steps = int(round(2.0 / dt))
        T = steps * dt
        with np.errstate(divide="ignore", invalid="ignore"):
            fac = np.where(kap2 > 0, (1 - np.cos(np.sqrt(kap2) * T)) / kap2, 0.5 * T * T)
            facv = np.where(kap2 > 0, np.sin(np.sqrt(kap2) * T) / np.sqrt(np.where(kap2 > 0, kap2, 1)), T)
        u_ex = np.fft.ifft2(fac * S)
        v_ex = np.fft.ifft2(facv * S)
        z = np.zeros((n, n))
        u, v, m = O.wave_rk4(z, z, dt, steps, c=c, gamma=0.0, Omega=0.0, rs=0.5)
        errs.append((np.max(np.abs(u - u_ex)), np.max(np.abs(v - v_ex))))
        # the mean obeys d^2 u_bar/dt^2 = s_bar (kappa = 0 mode), exactly quadratic in t
        tt = np.arange(steps + 1) * dt
        assert np.max(np.abs(m - 0.5 * tt ** 2 * s.mean())) <= 1e-14 * np.max(np.abs(m))
    assert errs[0][0] <= 1e-6
    for f in range(2):
        assert 3.8 <= math.log2(errs[0][f] / errs[1][f]) <= 4.2, errs


def test_rk4_self_convergence_factor_16():
    # Fig. 8 / eq:SCF: solutions at h, h/2, h/4 (N = 64, 128, 256,
    # dt = 0.25 h, D = [-2, 2]^2, A = 1, sigma_s = 0.1, Omega = 5, gamma = 10) give
    # (u2 - u1)/(u3 - u2) ~ 2^4 on the grid means; SPEC acceptance 11 band [10, 24].
    T0, T1 = 0.5, 2.5
    means = {}
    for n in (64, 128, 256):
        dt = 0.25 * L / n
        steps = int(round(T1 / dt))
        z = np.zeros((n, n))
        _, _, m = O.wave_rk4(z, z, dt, steps)
        stride = n // 64                     # common times: multiples of the coarse dt
        means[n] = m[::stride].real
    t = np.arange(means[64].size) * (0.25 * L / 64)
    win = (t >= T0) & (t <= T1)
    d1 = means[128][win] - means[64][win]
    d2 = means[256][win] - means[128][win]
    q_norm = np.linalg.norm(d1) / np.linalg.norm(d2)
    assert 10.0 <= q_norm <= 24.0, q_norm
    ok = np.abs(d2) > 1e-3 * np.max(np.abs(d2))
    q_med = float(np.median(d1[ok] / d2[ok]))
    assert 10.0 <= q_med <= 24.0, q_med
