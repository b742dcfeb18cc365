"""Pins of the fp64 CPU oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself: every check is a printed worked
example (tests/golden, cited), a closed form, an invariant, a brute-force sum
on tiny inputs, or a library routine for a special case.  A plausible mistake
in the oracle (dropped term, wrong sign or index, transposed operand, wrong
normalisation, Lx/Ly swap) fails at least one of these.  CPU only.
"""
import cmath
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_12308_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_dft_examples.json")
RNG = np.random.default_rng(2412)


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def cvec(pairs):
    return np.array([complex(r, i) for r, i in pairs])


def rand_c(shape):
    return RNG.standard_normal(shape) + 1j * RNG.standard_normal(shape)


def mode(nx, ny, p, q):
    """e^{2 pi i (p x/Lx + q y/Ly)} sampled at x_j = j Lx/nx, y_k = k Ly/ny with
    the phase reduced exactly in integers (no large-argument rounding)."""
    j, k = np.arange(nx), np.arange(ny)
    ex = np.exp(2j * np.pi * ((p * j) % nx) / nx)
    ey = np.exp(2j * np.pi * ((q * k) % ny) / ny)
    return np.outer(ey, ex)


# ---------------------------------------------------------------- 1D transforms

@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("fn", [O.dft, O.fft])
def test_spec_examples_forward(gold, fn):
    # SPEC.md:62-64 worked examples of eq:DFT, + sign.
    for case in gold["dft_forward"]:
        out = fn(cvec(case["in"]))
        assert np.max(np.abs(out - cvec(case["out"]))) <= 1e-15


@pytest.mark.parametrize("fn", [O.dft, O.fft])
def test_spec_examples_inverse(gold, fn):
    # SPEC.md:72-73, iDFT with 1/N.
    for case in gold["dft_inverse"]:
        out = fn(cvec(case["in"]), inverse=True)
        assert np.max(np.abs(out - cvec(case["out"]))) <= 1e-15


def test_roots_of_unity():
    # w_N = e^{2 pi i/N}: exact at quarter turns, unit modulus,
    # and equal to the library exponential to within 1 ulp-ish elsewhere.
    assert O.root(4, 1) == 1j and O.root(4, 2) == -1 and O.root(4, 3) == -1j
    assert O.root(8, 0) == 1 and O.root(8, -2) == -1j
    for n in [2, 3, 5, 8, 12, 64, 1000, 4096, 32768]:
        for m in RNG.integers(-3 * n, 3 * n, 20):
            w = O.root(n, int(m))
            # the library's argument 2 pi m/n is itself rounded, so allow a few ulp
            assert abs(w - cmath.exp(2j * math.pi * (int(m) % n) / n)) <= 2e-15
            assert abs(abs(w) - 1.0) <= 3e-16
    assert O.root(3, 1).real == -0.5 and O.root(6, 1).real == 0.5 and O.root(12, 1).imag == 0.5
    assert O.root(8, 1).real == O.root(8, 1).imag == math.sqrt(0.5)


def test_fourier_matrix_inverse():
    # W^{-1} = W^dagger / N: build W column by column from unit vectors.
    for n in [1, 2, 4, 7, 16, 32]:
        W = np.stack([O.dft(np.eye(n)[j]) for j in range(n)], axis=1)
        assert np.max(np.abs(W.conj().T @ W / n - np.eye(n))) <= 1e-12
        assert np.max(np.abs(W - W.T)) == 0.0                       # W_kj = w^{jk} symmetric


def test_direct_dft_matches_definition_entrywise():
    # eq:DFT written out with the library exponential, for a small odd size.
    n = 12
    x = rand_c(n)
    ref = np.array([sum(x[j] * cmath.exp(2j * math.pi * j * k / n) for j in range(n))
                    for k in range(n)])
    assert rel(O.dft(x), ref) <= 1e-14


@pytest.mark.parametrize("m", range(0, 13))
def test_fft_equals_direct_dft(m):
    # Path 2 (radix-2 recursion) vs path 1 (direct, eq:DFT).
    n = 2 ** m
    x = rand_c(n)
    assert rel(O.fft(x), O.dft(x)) <= 1e-13 * max(1, m)
    assert rel(O.fft(x, inverse=True), O.dft(x, inverse=True)) <= 1e-13 * max(1, m)


def test_numpy_crosscheck():
    # numpy's ifft uses e^{+2 pi i jk/n}/n, so the paper's forward = n * ifft,
    # the paper's inverse = fft / n  (R1, R3).
    for n in [1, 2, 8, 256, 4096]:
        x = rand_c(n)
        assert rel(O.fft(x), n * np.fft.ifft(x)) <= 1e-14
        assert rel(O.fft(x, inverse=True), np.fft.fft(x) / n) <= 1e-14


def test_roundtrip_parseval_linearity_symmetry():
    n = 1024
    x, y = rand_c(n), rand_c(n)
    X = O.fft(x)
    assert np.max(np.abs(O.fft(X, inverse=True) - x)) <= 1e-13                 # round trip
    assert abs(np.sum(abs(x) ** 2) - np.sum(abs(X) ** 2) / n) <= 1e-12 * np.sum(abs(x) ** 2)
    a, b = 0.3 - 1.1j, 2.0 + 0.5j
    assert rel(O.fft(a * x + b * y), a * X + b * O.fft(y)) <= 1e-14            # linearity
    r = RNG.standard_normal(n).astype(complex)
    R = O.fft(r)
    assert np.max(np.abs(R[1:] - np.conj(R[:0:-1]))) <= 1e-12                 # P_{N-k} = conj P_k


def test_periodicity():
    # P_{k+N} = P_k, by evaluating the eq:DFT sum at k + mN.
    n = 16
    x = rand_c(n)
    X = O.dft(x)
    for k in [0, 3, 9, 15]:
        for mm in [-2, 1, 3]:
            assert abs(O.dft_at(x, k + mm * n) - X[k]) <= 1e-13


def test_non_pow2_rejected():
    with pytest.raises(O.OracleError):
        O.fft(np.ones(12))
    with pytest.raises(O.OracleError):
        O.fft2(np.ones((6, 8)))
    assert O.dft(np.ones(12))[0] == 12          # the direct DFT handles any N


# ---------------------------------------------------------------- 2D transforms

@pytest.mark.parametrize("shape", [(1, 1), (1, 8), (2, 1), (4, 4), (8, 16), (16, 4), (16, 16)])
def test_fft2_matches_bruteforce_double_sum(shape):
    # 2D_DFT double sum vs rows-then-columns.
    p = rand_c(shape)
    P = O.dft2_direct(p)
    assert rel(O.fft2(p), P) <= 1e-13
    assert rel(O.fft2(p, path=1), P) <= 1e-13
    assert rel(O.fft2(P, inverse=True), p) <= 1e-13
    assert rel(O.dft2_direct(P, inverse=True), p) <= 1e-13


def test_fft2_bruteforce_entrywise_definition():
    # the double sum written out with the library exponential, 4x8 grid;
    # exponent a*j/Nx on x (fast index) and b*k/Ny on y.
    ny, nx = 4, 8
    p = rand_c((ny, nx))
    ref = np.zeros((ny, nx), complex)
    for b in range(ny):
        for a in range(nx):
            ref[b, a] = sum(p[k, j] * cmath.exp(2j * math.pi * (a * j / nx + b * k / ny))
                            for k in range(ny) for j in range(nx))
    assert rel(O.dft2_direct(p), ref) <= 1e-14
    assert rel(O.fft2(p), ref) <= 1e-14


def test_fft2_constant_grid(gold):
    # a constant c on 4x4 -> P(0,0) = 16c, all else 0.
    c = complex(*gold["fft2_constant_4x4"]["c"])
    P = O.fft2(np.full((4, 4), c))
    expect = np.zeros((4, 4), complex)
    expect[0, 0] = gold["fft2_constant_4x4"]["P00_factor"] * c
    assert np.max(np.abs(P - expect)) <= 1e-14


def test_fft2_properties():
    ny, nx = 64, 32
    p = rand_c((ny, nx))
    P = O.fft2(p)
    assert rel(P, nx * ny * np.fft.ifft2(p)) <= 1e-14                           # library special case
    assert rel(O.fft2(p, path=1), P) <= 1e-13                                  # path 1 vs path 2
    assert rel(O.fft2(p.T.copy()).T, P) <= 1e-14                               # axis-order independence
    assert abs(np.sum(abs(p) ** 2) - np.sum(abs(P) ** 2) / (nx * ny)) <= 1e-12 * np.sum(abs(p) ** 2)
    qx, qy = rand_c(nx), rand_c(ny)                                            # separability
    assert rel(O.fft2(np.outer(qy, qx)), np.outer(O.fft(qy), O.fft(qx))) <= 1e-13
    batch = rand_c((3, 8, 16))
    out = O.fft2(batch)
    for b in range(3):
        assert np.array_equal(out[b], O.fft2(batch[b]))


def test_wavenumbers(gold):
    # SPEC.md:219-220; k = 2 pi fold(a) / (n dx) with fold(n/2) = +n/2.
    for case in gold["wavenumbers"]:
        k = O.wavenumbers(case["n"], case["n"] * case["dx"])
        assert np.max(np.abs(k / math.pi - np.array(case["k_over_pi"]))) <= 1e-15
    k = O.wavenumbers(64, 2.0)
    assert k[0] == 0 and k[32] > 0 and np.allclose(k[33:], -k[31:0:-1])


def test_aliasing_beyond_nyquist():
    # A mode of index a + m n, sampled on n points, is indistinguishable from
    # mode a.  Under the + sign, e^{+2 pi i a x} lands in bin
    # n - a (R1).
    n, a = 64, 5
    j = np.arange(n)
    for m in [0, 1, 3]:
        x = np.exp(2j * np.pi * (a + m * n) * j / n)          # naive fp64 sampling
        X = O.fft(x)
        assert int(np.argmax(np.abs(X))) == n - a
        assert abs(X[n - a] - n) <= 1e-10 and np.sum(np.abs(X)) - abs(X[n - a]) <= 1e-9
    # Poisson of cos 2 pi (a + n) x returns the alias's solution
    xg = I.axis(n)
    s = np.tile(np.cos(2 * np.pi * (a + n) * xg), (n, 1))
    u = O.poisson(s)
    expect = -np.tile(np.cos(2 * np.pi * a * xg), (n, 1)) / (2 * np.pi * a) ** 2
    assert np.max(np.abs(u - expect)) <= 1e-12 * np.max(np.abs(expect))


# ---------------------------------------------------------------- Poisson

def test_poisson_single_modes_rectangular():
    # e^{2 pi i (p x/Lx + q y/Ly)} is an eigenfunction of nabla^2 with
    # eigenvalue -(2 pi)^2 (p^2/Lx^2 + q^2/Ly^2): u = -s / that.
    nx, ny, Lx, Ly = 32, 16, 2.0, 0.5
    for p, q in [(1, 0), (0, 1), (3, -2), (-5, 7), (16, 8), (2, 3)]:
        s = mode(nx, ny, p, q)
        lam = (2 * np.pi) ** 2 * (p * p / Lx ** 2 + q * q / Ly ** 2)
        for path in (1, 2):
            u = O.poisson(s, Lx, Ly, path=path)
            assert rel(u, -s / lam) <= 1e-13, (p, q, path)


def test_poisson_c1_sinusoid_closed_form():
    # BASELINE config 1: rho_sin = -8 pi^2 sin 2pi x sin 2pi y  =>  u = sin 2pi x sin 2pi y.
    d = I.c1_inputs(64)
    x = I.axis(64)
    expect = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x))
    assert rel(O.poisson(d.rho_sin), expect) <= 1e-14
    assert rel(O.poisson(d.rho_sin, path=1), expect) <= 1e-14


def test_poisson_zero_mode_and_mean():
    # k=0 zeroed (eq:Poisson2 equivalence): the input mean is
    # ignored and the output has zero mean.
    s = rand_c((32, 32))
    u1 = O.poisson(s)
    u2 = O.poisson(s - s.mean())
    u3 = O.poisson(s + 7.5 - 2j)
    assert abs(u1.mean()) <= 1e-15
    assert rel(u1, u2) <= 1e-14 and rel(u3, u1) <= 1e-14


def test_poisson_c1_blobs_paths_agree_and_linear():
    d = I.c1_inputs(64)
    ub1 = O.poisson(d.rho_blobs, path=1)
    ub2 = O.poisson(d.rho_blobs, path=2)
    assert rel(ub2, ub1) <= 1e-13
    assert rel(O.poisson(d.rho), O.poisson(d.rho_sin) + ub2) <= 1e-14


def test_poisson_fd_laplacian_residual():
    # Independent of any FFT: the 2nd-order 5-point Laplacian of the spectral
    # solution of a smooth source reproduces the source to O(h^2).
    errs = []
    for n in (64, 128):
        x = I.axis(n)
        s = np.zeros((n, n))
        I.add_gaussian(s, 0.4, 0.55, 0.1, 1.0)
        s -= s.mean()
        u = O.poisson(s).real
        h = 1.0 / n
        lap = (np.roll(u, 1, 0) + np.roll(u, -1, 0) + np.roll(u, 1, 1) + np.roll(u, -1, 1) - 4 * u) / h ** 2
        errs.append(np.max(np.abs(lap - s)) / np.max(np.abs(s)))
    assert errs[1] < 0.3 * errs[0] and errs[1] < 5e-3


# ---------------------------------------------------------------- diffusion

def heat_kernel(n, centres, sigmas, amps, D, T, images=2):
    """Exact periodic solution of u_t = D nabla^2 u for a sum of Gaussians
    A exp(-r^2/s^2): each becomes A s^2/(s^2+4DT) exp(-r^2/(s^2+4DT)), summed
    over periodic images."""
    x = I.axis(n)
    out = np.zeros((n, n))
    for (cx, cy), s, a in zip(centres, sigmas, amps):
        s2 = s * s + 4 * D * T
        gx = sum(np.exp(-(x - cx - m) ** 2 / s2) for m in range(-images, images + 1))
        gy = sum(np.exp(-(x - cy - m) ** 2 / s2) for m in range(-images, images + 1))
        out += a * (s * s / s2) * np.outer(gy, gx)
    return out


def test_diffusion_heat_kernel_closed_form():
    # C2 recipe at 256^2 (sigma range scaled so the grid resolves it), 200 steps.
    n, D, dt, steps = 256, 1e-3, 0.01, 200
    g = I.c2_inputs(n, sig_lo=0.02, sig_hi=0.05)
    u = O.diffuse(g.u0, D, dt, steps)
    exact = heat_kernel(n, g.centres, g.sigmas, g.amps, D, steps * dt)
    assert rel(u, exact) <= 1e-13
    assert np.max(np.abs(u.imag)) <= 1e-14
    uc = O.diffuse(g.u0, D, dt, steps, collapsed=True)                 # semigroup
    assert rel(uc, exact) <= 1e-13 and rel(u, uc) <= 1e-13


def test_diffusion_single_mode_and_mean():
    nx, ny, Lx, Ly, D, dt, steps = 32, 64, 1.5, 3.0, 0.02, 0.05, 7
    p, q = 3, -5
    f = mode(nx, ny, p, q)
    decay = math.exp(-D * (2 * np.pi) ** 2 * (p * p / Lx ** 2 + q * q / Ly ** 2) * dt * steps)
    assert rel(O.diffuse(f, D, dt, steps, Lx, Ly), decay * f) <= 1e-13
    g = rand_c((ny, nx)) + 3.0
    ug = O.diffuse(g, D, dt, steps, Lx, Ly)
    assert abs(ug.mean() / g.mean() - 1) <= 1e-14                    # Fig. 4
    assert np.array_equal(O.diffuse(g, D, dt, 0), g)                 # nsteps = 0 copies


# ---------------------------------------------------------------- wave

def test_wave_standing_modes():
    # sin 2 pi p x sin 2 pi q y is an eigenmode: u(T) = cos(wT) u0 for u_t(0) = 0,
    # u(T) = sin(wT)/w g for u(0) = 0, w = 2 pi c sqrt(p^2 + q^2).
    n, c, dt, steps = 64, 1.3, 1e-3, 40
    x = I.axis(n)
    for p, q in [(1, 1), (3, 5), (0, 2), (32, 1)]:
        m = np.outer(np.sin(2 * np.pi * q * x + 0.3), np.sin(2 * np.pi * p * x + 0.1))
        w = 2 * np.pi * c * math.hypot(p, q)
        T = steps * dt
        u, v = O.wave(m, np.zeros_like(m), c, dt, steps)
        assert np.max(np.abs(u - math.cos(w * T) * m)) <= 1e-13
        assert np.max(np.abs(v + w * math.sin(w * T) * m)) <= 1e-13 * max(1, w)
        u, v = O.wave(np.zeros_like(m), m, c, dt, steps)
        assert np.max(np.abs(u - math.sin(w * T) / w * m)) <= 1e-13
        assert np.max(np.abs(v - math.cos(w * T) * m)) <= 1e-13


def hankel_pulse(r, sigma, c, T):
    """Radial solution of u_tt = c^2 nabla^2 u, u(0) = exp(-r^2/sigma^2), u_t(0) = 0:
    u(r,T) = int_0^inf pi s^2 e^{-pi^2 s^2 rho^2} cos(2 pi rho c T) J0(2 pi rho r) 2 pi rho d rho."""
    from scipy import integrate, special
    f = lambda rho: (math.pi * sigma ** 2 * math.exp(-(math.pi * sigma * rho) ** 2)
                     * math.cos(2 * math.pi * rho * c * T) * special.j0(2 * math.pi * rho * r)
                     * 2 * math.pi * rho)
    top = 8.5 / (math.pi * sigma)
    val, err = integrate.quad(f, 0.0, top, limit=2000, epsabs=1e-15, epsrel=1e-13)
    return val


def test_wave_radial_pulse_hankel():
    n, sigma, c, dt, steps = 256, 0.05, 1.0, 2.5e-3, 40          # T = 0.1
    u0 = np.zeros((n, n))
    I.add_gaussian(u0, 0.5, 0.5, sigma, 1.0)
    u, _ = O.wave(u0, np.zeros_like(u0), c, dt, steps)
    T = steps * dt
    x = I.axis(n)
    for (k, j) in [(128, 128), (128, 140), (100, 150), (128, 160), (60, 128), (128, 190)]:
        r = math.hypot(x[j] - 0.5, x[k] - 0.5)
        assert abs(u[k, j].real - hankel_pulse(r, sigma, c, T)) <= 1e-12, (k, j)
    assert np.max(np.abs(u.imag)) <= 1e-14


def test_wave_mean_energy_reversibility():
    n, c, dt, steps = 64, 1.0, 1e-2, 50
    u0 = rand_c((n, n)) + 0.7
    v0 = rand_c((n, n)) - 0.2j
    u, v = O.wave(u0, v0, c, dt, steps)
    T = steps * dt
    assert abs(u.mean() - (u0.mean() + T * v0.mean())) <= 1e-13    # eq:OmegaZero mean law
    assert abs(v.mean() - v0.mean()) <= 1e-14
    k = O.wavenumbers(n, 1.0)
    kap2 = c * c * (k[None, :] ** 2 + k[:, None] ** 2)
    E = lambda uu, vv: np.sum(np.abs(np.fft.fft2(vv)) ** 2 + kap2 * np.abs(np.fft.fft2(uu)) ** 2)
    assert abs(E(u, v) / E(u0, v0) - 1) <= 1e-12                     # modal energy
    ub, vb = O.wave(u, v, c, -dt, steps)                             # time reversal
    # v carries kappa-amplified rounding of u (kappa up to 2 pi 45 on white noise)
    assert rel(ub, u0) <= 1e-13 and rel(vb, v0) <= 2e-12
    uc, vc = O.wave(u0, v0, c, dt, steps, collapsed=True)
    assert rel(uc, u) <= 1e-13 and rel(vc, v) <= 1e-12


def test_batched_equals_per_grid():
    b = rand_c((3, 16, 32))
    u = O.poisson(b)
    d = O.diffuse(b, 0.01, 0.1, 3)
    for i in range(3):
        assert np.array_equal(u[i], O.poisson(b[i]))
        assert np.array_equal(d[i], O.diffuse(b[i], 0.01, 0.1, 3))
