/*
 * fftpde_oracle.c -- plain, slow, fp64 CPU oracle for the 2D FFT-PDE hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2412_12308_b200/csrc) and neither side includes the other.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited by line):
 *   DFT      P_k = sum_j p_j w_N^{jk},  w_N = e^{+2 pi i/N}        eq:DFT
 *   iDFT     p_j = (1/N) sum_k P_k w_N^{-jk}
 *            = (1/N) conj(DFT(conj P))
 *   FFT      recursive radix-2 decimation in time:
 *            P_k = E_k + w_N^k O_k, P_{k+N/2} = E_k - w_N^k O_k     eq:FFTpairodd(_2) PAPER.md:188-224
 *   2D DFT   P_ab = sum_j sum_k p_jk e^{+2pi i aj/Nx} e^{+2pi i bk/Ny}   2D_DFT PAPER.md:246-249
 *            computed as Ny DFTs along x then Nx DFTs along y
 *   Poisson  u = F^{-1}{ -F{g} / w^2 },  k=0 mode zeroed           eq:SolutionPoisson PAPER.md:306-331
 *   Diffusion u^ = f^ e^{-w^2 t} (coefficient D per DESIGN.md R6)  solCalorFourier PAPER.md:376-386
 *   Wave     u^ = f^ cos(wt) + (g^/w) sin(wt);  w=0: u^ = g^ t + f^ eq:OmegaZero/NonZero PAPER.md:459-471
 *            v^ = d u^/dt
 *   3D transform, Poisson and diffusion (n-D extension)
 *   Diagonal operators  F^-1{(-i w)^k F{u}}: Laplacian, d/dx, d/dy
 *   Diffusion + static source: exact integrator of du^/dt = -D w^2 u^ + s^
 *   Wave with a time-dependent source: RK4 on du^/dt = v^,
 *            dv^/dt = -w^2 u^ + s^(t), orbiting Gaussian source
 *
 * Readings of silent / garbled points are DESIGN.md R1..R16:
 *   forward sign +, unnormalised; inverse 1/N per axis; natural order with
 *   fold(N/2) = +N/2; angular wavenumber k = 2 pi fold(a)/L; vertex sampling.
 *
 * Two independent transform paths:
 *   path 1: direct O(N^2) sums (eq:DFT and the conjugate-kernel iDFT sum)
 *   path 2: recursive radix-2 FFT (forward only) + the conj trick for the inverse.
 * Roots of unity are computed per index by exact integer reduction and an
 * octant-reduced argument in long double, never by recurrence.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math).
 * OpenMP is used only across independent rows, columns and batch members.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double re, im; } cplx;

static cplx c_add(cplx a, cplx b) { cplx r = { a.re + b.re, a.im + b.im }; return r; }
static cplx c_sub(cplx a, cplx b) { cplx r = { a.re - b.re, a.im - b.im }; return r; }
static cplx c_mul(cplx a, cplx b)
{
    cplx r = { a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re };
    return r;
}
static cplx c_conj(cplx a) { cplx r = { a.re, -a.im }; return r; }
static cplx c_scale(cplx a, double s) { cplx r = { a.re * s, a.im * s }; return r; }

static int is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

/* ------------------------------------------------------------------------ */
/* Roots of unity  w_n^m = exp(+2 pi i m / n)   (omega_N := e^{2 pi i/N}) */

/* Exact integer reduction: r = m mod n in [0,n).  The angle 2 pi r/n is split
 * into a quadrant q = floor(4r/n) and a remainder t = 4r - q n in [0,n), i.e.
 * angle = (pi/2)(q + t/n).  The remainder is folded to the first octant so
 * sin/cos are evaluated on an argument in [0, pi/4], in long double, then
 * rounded once to double.  Exact values (1, i, -1, -i) come out exact. */
static cplx root_of_unity(int64_t n, int64_t m)
{
    int64_t r = m % n;
    if (r < 0) r += n;
    int64_t q = (4 * r) / n;          /* quadrant 0..3 */
    int64_t t = 4 * r - q * n;        /* 0 <= t < n */
    long double c, s;
    const long double half_pi = 1.570796326794896619231321691639751442L;
    if (2 * t <= n) {
        long double phi = half_pi * (long double)t / (long double)n;
        c = cosl(phi); s = sinl(phi);
    } else {                           /* complement: phi = pi/2 - phi' */
        long double phi = half_pi * (long double)(n - t) / (long double)n;
        c = sinl(phi); s = cosl(phi);
    }
    double cd = (double)c, sd = (double)s;
    cplx w;
    switch (q) {                       /* rotate by q quarter turns: multiply by i^q */
    case 0:  w.re =  cd; w.im =  sd; break;
    case 1:  w.re = -sd; w.im =  cd; break;
    case 2:  w.re = -cd; w.im = -sd; break;
    default: w.re =  sd; w.im = -cd; break;
    }
    return w;
}

/* table w[m] = w_n^m, m = 0..n-1, each entry computed directly */
static cplx *root_table(int64_t n)
{
    cplx *w = (cplx *)malloc(sizeof(cplx) * (size_t)n);
    for (int64_t m = 0; m < n; ++m) w[m] = root_of_unity(n, m);
    return w;
}

int oracle_root(int64_t n, int64_t m, double *out2)
{
    if (n < 1 || !out2) return -1;
    cplx w = root_of_unity(n, m);
    out2[0] = w.re; out2[1] = w.im;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Path 1: direct sums.                                                      */

/* X_k = sum_j x_j w_n^{jk}  (eq:DFT) for sign=+1;
 * x_j = (1/n) sum_k X_k w_n^{-jk} (iDFT) for sign=-1.
 * Elements are read/written with strides so columns can be transformed too. */
static void dft_direct(int64_t n, const cplx *x, int64_t xs, cplx *X, int64_t Xs,
                       int sign, const cplx *w)
{
    for (int64_t k = 0; k < n; ++k) {
        cplx acc = { 0.0, 0.0 };
        for (int64_t j = 0; j < n; ++j) {
            int64_t e = (j * k) % n;                    /* exact index product */
            cplx wk = w[e];
            if (sign < 0) wk = c_conj(wk);               /* w_n^{-jk} */
            acc = c_add(acc, c_mul(x[j * xs], wk));
        }
        if (sign < 0) acc = c_scale(acc, 1.0 / (double)n);
        X[k * Xs] = acc;
    }
}

int oracle_dft1(int64_t n, const double *x, double *X, int inverse)
{
    if (n < 1 || !x || !X) return -1;
    cplx *w = root_table(n);
    cplx *tmp = (cplx *)malloc(sizeof(cplx) * (size_t)n);
    dft_direct(n, (const cplx *)x, 1, tmp, 1, inverse ? -1 : +1, w);
    memcpy(X, tmp, sizeof(cplx) * (size_t)n);
    free(tmp); free(w);
    return 0;
}

/* The DFT sum of eq:DFT evaluated at an arbitrary integer k (any sign, any
 * size): used to check the periodicity P_{k+N} = P_k. */
int oracle_dft1_at(int64_t n, const double *x, int64_t k, double *out2)
{
    if (n < 1 || !x || !out2) return -1;
    const cplx *xc = (const cplx *)x;
    cplx acc = { 0.0, 0.0 };
    for (int64_t j = 0; j < n; ++j) {
        int64_t e = (j * k) % n;
        acc = c_add(acc, c_mul(xc[j], root_of_unity(n, e)));
    }
    out2[0] = acc.re; out2[1] = acc.im;
    return 0;
}

/* Brute-force 2D double sum, 2D_DFT, O((nx ny)^2).
 * p[k][j] = p_{jk} (x index j fastest).  inverse: conjugate kernel and
 * 1/(nx ny) (per-axis iDFT). */
int oracle_dft2_direct(int64_t nx, int64_t ny, const double *p, double *P, int inverse)
{
    if (nx < 1 || ny < 1 || !p || !P) return -1;
    const cplx *pc = (const cplx *)p;
    cplx *wx = root_table(nx), *wy = root_table(ny);
    cplx *out = (cplx *)malloc(sizeof(cplx) * (size_t)(nx * ny));
    for (int64_t b = 0; b < ny; ++b)
        for (int64_t a = 0; a < nx; ++a) {
            cplx acc = { 0.0, 0.0 };
            for (int64_t k = 0; k < ny; ++k)
                for (int64_t j = 0; j < nx; ++j) {
                    cplx ex = wx[(a * j) % nx], ey = wy[(b * k) % ny];
                    if (inverse) { ex = c_conj(ex); ey = c_conj(ey); }
                    acc = c_add(acc, c_mul(pc[k * nx + j], c_mul(ex, ey)));
                }
            if (inverse) acc = c_scale(acc, 1.0 / ((double)nx * (double)ny));
            out[b * nx + a] = acc;
        }
    memcpy(P, out, sizeof(cplx) * (size_t)(nx * ny));
    free(out); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Path 2: recursive radix-2 decimation-in-time FFT, forward (+) sign.       */

/* X[0..n) <- FFT_n of x[0], x[s], x[2s], ...  (n a power of two).
 * w is the root table of the top-level length N; w_n^k = w_N^{k N/n}.
 * If n == 1 return x.  Otherwise E = FFT(even), O = FFT(odd)
 * are written into X[0..n/2) and X[n/2..n), then combined with
 * P_k = E_k + w_n^k O_k and P_{k+n/2} = E_k - w_n^k O_k. */
static void fft_rec(int64_t n, const cplx *x, int64_t s, cplx *X,
                    const cplx *w, int64_t N)
{
    if (n == 1) { X[0] = x[0]; return; }
    int64_t h = n / 2;
    fft_rec(h, x, 2 * s, X, w, N);          /* even-indexed points  -> E */
    fft_rec(h, x + s, 2 * s, X + h, w, N);  /* odd-indexed points   -> O */
    int64_t step = N / n;
    for (int64_t k = 0; k < h; ++k) {
        cplx e = X[k];
        cplx o = c_mul(w[k * step], X[k + h]);
        X[k] = c_add(e, o);
        X[k + h] = c_sub(e, o);
    }
}

/* 1D forward (+) or inverse transform of n contiguous points, path 2.
 * inverse = (1/n) conj(FFT(conj(X))). */
static void fft1_path2(int64_t n, const cplx *in, cplx *out, int inverse,
                       const cplx *w, cplx *tmp)
{
    if (!inverse) {
        fft_rec(n, in, 1, out, w, n);
        return;
    }
    for (int64_t j = 0; j < n; ++j) tmp[j] = c_conj(in[j]);
    fft_rec(n, tmp, 1, out, w, n);
    double s = 1.0 / (double)n;
    for (int64_t j = 0; j < n; ++j) out[j] = c_scale(c_conj(out[j]), s);
}

int oracle_fft1(int64_t n, const double *x, double *X, int inverse)
{
    if (n < 1 || !x || !X) return -1;
    if (!is_pow2(n)) return -2;
    cplx *w = root_table(n);
    cplx *tmp = (cplx *)malloc(sizeof(cplx) * (size_t)n);
    cplx *out = (cplx *)malloc(sizeof(cplx) * (size_t)n);
    fft1_path2(n, (const cplx *)x, out, inverse, w, tmp);
    memcpy(X, out, sizeof(cplx) * (size_t)n);
    free(out); free(tmp); free(w);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* 2D transform by sequential 1D transforms: every row (x axis, length nx)    */
/* then every column (y axis, length ny).                 */

/* path = 1: separable direct sums; path = 2: radix-2 FFT.  In place on g. */
static void transform2d(int64_t nx, int64_t ny, cplx *g, int inverse, int path,
                        const cplx *wx, const cplx *wy)
{
    /* rows */
    #pragma omp parallel
    {
        cplx *a = (cplx *)malloc(sizeof(cplx) * (size_t)nx);
        cplx *b = (cplx *)malloc(sizeof(cplx) * (size_t)nx);
        cplx *t = (cplx *)malloc(sizeof(cplx) * (size_t)nx);
        #pragma omp for schedule(static)
        for (int64_t k = 0; k < ny; ++k) {
            memcpy(a, g + k * nx, sizeof(cplx) * (size_t)nx);
            if (path == 1) dft_direct(nx, a, 1, b, 1, inverse ? -1 : +1, wx);
            else fft1_path2(nx, a, b, inverse, wx, t);
            memcpy(g + k * nx, b, sizeof(cplx) * (size_t)nx);
        }
        free(a); free(b); free(t);
    }
    /* columns: copy each to a contiguous buffer, transform, copy back */
    #pragma omp parallel
    {
        cplx *a = (cplx *)malloc(sizeof(cplx) * (size_t)ny);
        cplx *b = (cplx *)malloc(sizeof(cplx) * (size_t)ny);
        cplx *t = (cplx *)malloc(sizeof(cplx) * (size_t)ny);
        #pragma omp for schedule(static)
        for (int64_t j = 0; j < nx; ++j) {
            for (int64_t k = 0; k < ny; ++k) a[k] = g[k * nx + j];
            if (path == 1) dft_direct(ny, a, 1, b, 1, inverse ? -1 : +1, wy);
            else fft1_path2(ny, a, b, inverse, wy, t);
            for (int64_t k = 0; k < ny; ++k) g[k * nx + j] = b[k];
        }
        free(a); free(b); free(t);
    }
}

static int check_grid(int64_t nx, int64_t ny, int64_t batch, int path)
{
    if (nx < 1 || ny < 1 || batch < 1) return -1;
    if (path == 2 && (!is_pow2(nx) || !is_pow2(ny))) return -2;
    if (path != 1 && path != 2) return -1;
    return 0;
}

int oracle_fft2(int64_t nx, int64_t ny, int64_t batch, const double *in, double *out,
                int inverse, int path)
{
    int rc = check_grid(nx, ny, batch, path);
    if (rc) return rc;
    if (!in || !out) return -1;
    cplx *wx = root_table(nx), *wy = root_table(ny);
    size_t plane = (size_t)(nx * ny);
    if (out != in) memcpy(out, in, sizeof(cplx) * plane * (size_t)batch);
    for (int64_t b = 0; b < batch; ++b)
        transform2d(nx, ny, (cplx *)out + b * plane, inverse, path, wx, wy);
    free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Wavenumbers: k[a] = 2 pi fold(a) / L,  fold(a) = a (a <= n/2) else a - n.  */
/* Frequency grid PAPER.md:106-109, 253-258; shifting of k > N/2 PAPER.md:175; */
/* omega = 2 pi f (R4), Nyquist bin at +n/2 (R2).        */

static int64_t fold(int64_t a, int64_t n) { return (2 * a <= n) ? a : a - n; }

int oracle_wavenumbers(int64_t n, double L, double *k)
{
    if (n < 1 || !(L > 0.0) || !k) return -1;
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t a = 0; a < n; ++a) k[a] = two_pi * (double)fold(a, n) / L;
    return 0;
}

/* |k|^2 = kx[a]^2 + ky[b]^2 (R4) */
static double *ksq_table(int64_t nx, int64_t ny, double Lx, double Ly)
{
    double *kx = (double *)malloc(sizeof(double) * (size_t)nx);
    double *ky = (double *)malloc(sizeof(double) * (size_t)ny);
    oracle_wavenumbers(nx, Lx, kx);
    oracle_wavenumbers(ny, Ly, ky);
    double *k2 = (double *)malloc(sizeof(double) * (size_t)(nx * ny));
    for (int64_t b = 0; b < ny; ++b)
        for (int64_t a = 0; a < nx; ++a)
            k2[b * nx + a] = kx[a] * kx[a] + ky[b] * ky[b];
    free(kx); free(ky);
    return k2;
}

/* ------------------------------------------------------------------------ */
/* Poisson  nabla^2 u = s  (eq:Poisson PAPER.md:286-291):                     */
/*   g = s - mean(s) (eq:Poisson2) is the same as zeroing   */
/*   the k = 0 mode of F{s}; u = F^{-1}{ -F{g} / |k|^2 } (eq:SolutionPoisson, */
/*   PAPER.md:329-331), with the k = 0 mode of u set to 0 (R5).    */
int oracle_poisson(int64_t nx, int64_t ny, int64_t batch, double Lx, double Ly,
                   const double *rho, double *u, int path)
{
    int rc = check_grid(nx, ny, batch, path);
    if (rc) return rc;
    if (!rho || !u || !(Lx > 0.0) || !(Ly > 0.0)) return -1;
    cplx *wx = root_table(nx), *wy = root_table(ny);
    double *k2 = ksq_table(nx, ny, Lx, Ly);
    size_t plane = (size_t)(nx * ny);
    if (u != rho) memcpy(u, rho, sizeof(cplx) * plane * (size_t)batch);
    for (int64_t bi = 0; bi < batch; ++bi) {
        cplx *g = (cplx *)u + bi * plane;
        transform2d(nx, ny, g, 0, path, wx, wy);              /* F{s} */
        for (size_t i = 0; i < plane; ++i) {
            if (k2[i] == 0.0) { g[i].re = 0.0; g[i].im = 0.0; }   /* k = 0 zeroed */
            else g[i] = c_scale(g[i], -1.0 / k2[i]);           /* -F{g}/|k|^2 */
        }
        transform2d(nx, ny, g, 1, path, wx, wy);              /* F^{-1} */
    }
    free(k2); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Diffusion u_t = D nabla^2 u (ec:EcuacionDeCalor with s = 0, coefficient D, */
/* DESIGN.md R6): u^(t+dt) = u^(t) exp(-D |k|^2 dt) for |k| > 0, u^ unchanged */
/* at k = 0 (ec:solCalorFourier).                            */
/* Stepped: nsteps x (forward 2D, multiply, inverse 2D).  Collapsed (a pin,    */
/* DESIGN.md R8): one forward, multiply by exp(-D |k|^2 T), T = nsteps dt, one */
/* inverse.                                                                    */
int oracle_diffuse(int64_t nx, int64_t ny, int64_t batch, double Lx, double Ly,
                   double D, double dt, int64_t nsteps, const double *u0, double *u,
                   int collapsed, int path)
{
    int rc = check_grid(nx, ny, batch, path);
    if (rc) return rc;
    if (!u0 || !u || nsteps < 0 || !(Lx > 0.0) || !(Ly > 0.0)) return -1;
    size_t plane = (size_t)(nx * ny);
    if (u != u0) memcpy(u, u0, sizeof(cplx) * plane * (size_t)batch);
    if (nsteps == 0) return 0;
    cplx *wx = root_table(nx), *wy = root_table(ny);
    double *k2 = ksq_table(nx, ny, Lx, Ly);
    double tstep = collapsed ? (double)nsteps * dt : dt;
    int64_t reps = collapsed ? 1 : nsteps;
    double *m = (double *)malloc(sizeof(double) * plane);
    for (size_t i = 0; i < plane; ++i)
        m[i] = (k2[i] == 0.0) ? 1.0 : exp(-D * k2[i] * tstep);
    for (int64_t bi = 0; bi < batch; ++bi) {
        cplx *g = (cplx *)u + bi * plane;
        for (int64_t s = 0; s < reps; ++s) {
            transform2d(nx, ny, g, 0, path, wx, wy);
            for (size_t i = 0; i < plane; ++i) g[i] = c_scale(g[i], m[i]);
            transform2d(nx, ny, g, 1, path, wx, wy);
        }
    }
    free(m); free(k2); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Wave u_tt = c^2 nabla^2 u, s = 0 (eq:wave_equation PAPER.md:417-424).      */
/* First-order system du^/dt = v^, dv^/dt = -kappa^2 u^,   */
/* kappa = c|k|.  Exact step of length dt (eq:OmegaNonZero PAPER.md:466-471,  */
/* eq:OmegaZero PAPER.md:459-464, and v^ = du^/dt, R7):             */
/*   u^' = C u^ + S1 v^,   v^' = S2 u^ + C v^                                  */
/*   C = cos(kappa dt), S1 = sin(kappa dt)/kappa, S2 = -kappa sin(kappa dt);   */
/*   kappa = 0: C = 1, S1 = dt, S2 = 0.                                        */
/* Stepped: nsteps x (forward both fields, 2x2 update, inverse both).          */
/* Collapsed: the same with dt -> T = nsteps dt, once.  In place on (u, ut).   */
int oracle_wave(int64_t nx, int64_t ny, int64_t batch, double Lx, double Ly,
                double c, double dt, int64_t nsteps, double *u, double *ut,
                int collapsed, int path)
{
    int rc = check_grid(nx, ny, batch, path);
    if (rc) return rc;
    if (!u || !ut || nsteps < 0 || !(Lx > 0.0) || !(Ly > 0.0) || c < 0.0) return -1;
    if (nsteps == 0) return 0;
    size_t plane = (size_t)(nx * ny);
    cplx *wx = root_table(nx), *wy = root_table(ny);
    double *k2 = ksq_table(nx, ny, Lx, Ly);
    double tstep = collapsed ? (double)nsteps * dt : dt;
    int64_t reps = collapsed ? 1 : nsteps;
    double *C = (double *)malloc(sizeof(double) * plane);
    double *S1 = (double *)malloc(sizeof(double) * plane);
    double *S2 = (double *)malloc(sizeof(double) * plane);
    for (size_t i = 0; i < plane; ++i) {
        double kappa = c * sqrt(k2[i]);
        if (kappa == 0.0) { C[i] = 1.0; S1[i] = tstep; S2[i] = 0.0; }
        else {
            double sn = sin(kappa * tstep);
            C[i] = cos(kappa * tstep);
            S1[i] = sn / kappa;
            S2[i] = -kappa * sn;
        }
    }
    for (int64_t bi = 0; bi < batch; ++bi) {
        cplx *U = (cplx *)u + bi * plane;
        cplx *V = (cplx *)ut + bi * plane;
        for (int64_t s = 0; s < reps; ++s) {
            transform2d(nx, ny, U, 0, path, wx, wy);
            transform2d(nx, ny, V, 0, path, wx, wy);
            for (size_t i = 0; i < plane; ++i) {
                cplx uh = U[i], vh = V[i];
                U[i] = c_add(c_scale(uh, C[i]), c_scale(vh, S1[i]));
                V[i] = c_add(c_scale(uh, S2[i]), c_scale(vh, C[i]));
            }
            transform2d(nx, ny, U, 1, path, wx, wy);
            transform2d(nx, ny, V, 1, path, wx, wy);
        }
    }
    free(C); free(S1); free(S2); free(k2); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* 3D: the n-D extension of the 2D recipe, "extended analogously" to further  */
/* dimensions: sequential 1D transforms along x (rows), y and  */
/* z.  Grid [nz][ny][nx], x fastest.  Forward sign +, inverse 1/N per axis.   */
static void transform3d(int64_t nx, int64_t ny, int64_t nz, cplx *g, int inverse,
                        const cplx *wx, const cplx *wy, const cplx *wz)
{
    size_t plane = (size_t)(nx * ny);
    for (int64_t z = 0; z < nz; ++z) transform2d(nx, ny, g + (size_t)z * plane, inverse, 2, wx, wy);
    #pragma omp parallel
    {
        cplx *a = (cplx *)malloc(sizeof(cplx) * (size_t)nz);
        cplx *b = (cplx *)malloc(sizeof(cplx) * (size_t)nz);
        cplx *t = (cplx *)malloc(sizeof(cplx) * (size_t)nz);
        #pragma omp for schedule(static)
        for (int64_t c = 0; c < nx * ny; ++c) {
            for (int64_t z = 0; z < nz; ++z) a[z] = g[(size_t)z * plane + c];
            fft1_path2(nz, a, b, inverse, wz, t);
            for (int64_t z = 0; z < nz; ++z) g[(size_t)z * plane + c] = b[z];
        }
        free(a); free(b); free(t);
    }
}

int oracle_fft3(int64_t nx, int64_t ny, int64_t nz, const double *in, double *out, int inverse)
{
    int rc = check_grid(nx, ny, nz, 2);
    if (rc) return rc;
    if (!is_pow2(nz)) return -2;
    if (!in || !out) return -1;
    cplx *wx = root_table(nx), *wy = root_table(ny), *wz = root_table(nz);
    if (out != in) memcpy(out, in, sizeof(cplx) * (size_t)(nx * ny * nz));
    transform3d(nx, ny, nz, (cplx *)out, inverse, wx, wy, wz);
    free(wx); free(wy); free(wz);
    return 0;
}

/* 3D Poisson (op 0: m = -1/|k|^2, k = 0 zeroed, eq:SolutionPoisson PAPER.md: */
/* 329-331) and exact diffusion steps (op 1: m = exp(-D |k|^2 dt), PAPER.md:  */
/* 378-386, stepped nsteps times materialising u, R8), |k|^2 = kx^2 + ky^2 +  */
/* kz^2.  In place on u.                                                       */
int oracle_solve3(int64_t nx, int64_t ny, int64_t nz, double Lx, double Ly, double Lz, int op,
                  double D, double dt, int64_t nsteps, double *u)
{
    int rc = check_grid(nx, ny, nz, 2);
    if (rc) return rc;
    if (!is_pow2(nz)) return -2;
    if (!u || !(Lx > 0.0) || !(Ly > 0.0) || !(Lz > 0.0) || op < 0 || op > 1 || nsteps < 0) return -1;
    size_t plane = (size_t)(nx * ny), vol = plane * (size_t)nz;
    cplx *wx = root_table(nx), *wy = root_table(ny), *wz = root_table(nz);
    double *kx = (double *)malloc(sizeof(double) * (size_t)nx);
    double *ky = (double *)malloc(sizeof(double) * (size_t)ny);
    double *kz = (double *)malloc(sizeof(double) * (size_t)nz);
    oracle_wavenumbers(nx, Lx, kx);
    oracle_wavenumbers(ny, Ly, ky);
    oracle_wavenumbers(nz, Lz, kz);
    double *m = (double *)malloc(sizeof(double) * vol);
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double k2 = kx[x] * kx[x] + ky[y] * ky[y] + kz[z] * kz[z];
                size_t i = (size_t)z * plane + (size_t)y * (size_t)nx + (size_t)x;
                if (op == 0) m[i] = k2 == 0.0 ? 0.0 : -1.0 / k2;
                else m[i] = exp(-D * k2 * dt);
            }
    int64_t reps = op == 0 ? 1 : nsteps;
    cplx *g = (cplx *)u;
    for (int64_t s = 0; s < reps; ++s) {
        transform3d(nx, ny, nz, g, 0, wx, wy, wz);
        for (size_t i = 0; i < vol; ++i) g[i] = c_scale(g[i], m[i]);
        transform3d(nx, ny, nz, g, 1, wx, wy, wz);
    }
    free(m); free(kx); free(ky); free(kz); free(wx); free(wy); free(wz);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Diagonal k-space operators:  out = F^-1{ m F{in} }  */
/* with F{d^k u/dx^k} = (-i omega)^k F{u} under the forward */
/* sign + (R1); omega = 2 pi fold(a)/L, Nyquist bin +N/2 (R2, R24): */
/*   op 0  Laplacian      m = -(kx^2 + ky^2)                                  */
/*   op 1  d/dx           m = -i kx                                            */
/*   op 2  d/dy           m = -i ky                                            */
int oracle_kspace_apply(int64_t nx, int64_t ny, int64_t batch, double Lx, double Ly, int op,
                        const double *in, double *out)
{
    int rc = check_grid(nx, ny, batch, 2);
    if (rc) return rc;
    if (!in || !out || !(Lx > 0.0) || !(Ly > 0.0) || op < 0 || op > 2) return -1;
    size_t plane = (size_t)(nx * ny);
    cplx *wx = root_table(nx), *wy = root_table(ny);
    double *kx = (double *)malloc(sizeof(double) * (size_t)nx);
    double *ky = (double *)malloc(sizeof(double) * (size_t)ny);
    oracle_wavenumbers(nx, Lx, kx);
    oracle_wavenumbers(ny, Ly, ky);
    if (out != in) memcpy(out, in, sizeof(cplx) * plane * (size_t)batch);
    for (int64_t bi = 0; bi < batch; ++bi) {
        cplx *g = (cplx *)out + bi * plane;
        transform2d(nx, ny, g, 0, 2, wx, wy);
        for (int64_t b = 0; b < ny; ++b)
            for (int64_t a = 0; a < nx; ++a) {
                cplx v = g[b * nx + a], r;
                if (op == 0) {
                    r = c_scale(v, -(kx[a] * kx[a] + ky[b] * ky[b]));
                } else {
                    double k = op == 1 ? kx[a] : ky[b];
                    r.re = k * v.im;                      /* (-i k) (x + i y) = k y - i k x */
                    r.im = -k * v.re;
                }
                g[b * nx + a] = r;
            }
        transform2d(nx, ny, g, 1, 2, wx, wy);
    }
    free(kx); free(ky); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Diffusion with a static source, u_t = D nabla^2 u + s (eq. EcuacionDeCalor */
/* PAPER.md:355-367; coefficient D per R6).  In Fourier space                 */
/* du^/dt = -D w^2 u^ + s^ (eq:DiffusionIVPFS PAPER.md:369-376), integrated   */
/* exactly over each step (the closed form of solCalorFourier extended by the */
/* constant forcing):                                                          */
/*   u^(t + dt) = E u^(t) + Phi s^,   E = exp(-D w^2 dt),                      */
/*   Phi = -expm1(-D w^2 dt) / (D w^2)   (w != 0, D > 0),   Phi = dt otherwise.*/
/* Stepped: nsteps x (forward u, update, inverse) materialising u (R8); s^ is */
/* the transform of the source, computed once.  In place on u.                 */
int oracle_diffuse_source(int64_t nx, int64_t ny, int64_t batch, double Lx, double Ly, double D,
                          double dt, int64_t nsteps, double *u, const double *src)
{
    int rc = check_grid(nx, ny, batch, 2);
    if (rc) return rc;
    if (!u || !src || nsteps < 0 || !(Lx > 0.0) || !(Ly > 0.0) || D < 0.0 || dt < 0.0) return -1;
    size_t plane = (size_t)(nx * ny);
    cplx *wx = root_table(nx), *wy = root_table(ny);
    double *k2 = ksq_table(nx, ny, Lx, Ly);
    cplx *S = (cplx *)malloc(sizeof(cplx) * plane);
    for (int64_t bi = 0; bi < batch; ++bi) {
        cplx *U = (cplx *)u + bi * plane;
        memcpy(S, (const cplx *)src + bi * plane, sizeof(cplx) * plane);
        transform2d(nx, ny, S, 0, 2, wx, wy);
        for (int64_t n = 0; n < nsteps; ++n) {
            transform2d(nx, ny, U, 0, 2, wx, wy);
            for (size_t i = 0; i < plane; ++i) {
                double x = D * k2[i] * dt;
                double E = exp(-x);
                double Phi = x > 0.0 ? -expm1(-x) / (D * k2[i]) : dt;
                U[i] = c_add(c_scale(U[i], E), c_scale(S[i], Phi));
            }
            transform2d(nx, ny, U, 1, 2, wx, wy);
        }
    }
    free(S); free(k2); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Orbiting Gaussian source ("Example with Source"):        */
/*   s(t,x,y) = A exp(-[(x - x0)^2 + (y - y0)^2] / sigma^2) cos(gamma t),     */
/*   x0 = rs cos(Omega t),  y0 = rs sin(Omega t),                             */
/* sampled at x_j = xmin + j Lx/nx, y_k = ymin + k Ly/ny; on the periodic     */
/* domain x - x0 and y - y0 are minimum images in [-L/2, L/2) (R21).*/
static double min_image(double d, double L) { return d - L * floor(d / L + 0.5); }

int oracle_orbit_source(int64_t nx, int64_t ny, double Lx, double Ly, double xmin, double ymin,
                        double A, double sigma, double Omega, double gamma, double rs, double t,
                        double *out)
{
    if (nx < 1 || ny < 1 || !out || !(Lx > 0.0) || !(Ly > 0.0) || !(sigma > 0.0)) return -1;
    double x0 = rs * cos(Omega * t), y0 = rs * sin(Omega * t);
    double amp = A * cos(gamma * t);
    cplx *o = (cplx *)out;
    for (int64_t k = 0; k < ny; ++k) {
        double y = ymin + (double)k * Ly / (double)ny;
        double dy = min_image(y - y0, Ly);
        for (int64_t j = 0; j < nx; ++j) {
            double x = xmin + (double)j * Lx / (double)nx;
            double dx = min_image(x - x0, Lx);
            o[k * nx + j].re = amp * exp(-(dx * dx + dy * dy) / (sigma * sigma));
            o[k * nx + j].im = 0.0;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Wave equation with a time-dependent source, u_tt = c^2 nabla^2 u + s      */
/* (eq:wave_equation PAPER.md:417-424), in Fourier space the first-order     */
/* system (eq:SystemOfODEsForWaveEquation PAPER.md:448-454)                   */
/*   du^/dt = v^,   dv^/dt = -kappa^2 u^ + s^(t),   kappa = c|k|,             */
/* integrated with the classical Runge-Kutta 4 scheme (stages   */
/* combined as (k1 + 2 k2 + 2 k3 + k4)/6), the source re-sampled and           */
/* transformed (path 2) at each stage time t, t + dt/2, t + dt (DESIGN.md     */
/* R22).  u, ut: physical fields at t0 on entry, at t0 + nsteps dt on exit    */
/* (inverse transforms).  means (nsteps + 1 complex, may be */
/* NULL): the grid mean of u at t0 + n dt, = u^(0,0) / (nx ny).               */
int oracle_wave_rk4(int64_t nx, int64_t ny, double Lx, double Ly, double xmin, double ymin, double c,
                    double A, double sigma, double Omega, double gamma, double rs,
                    double t0, double dt, int64_t nsteps, double *u, double *ut, double *means)
{
    int rc = check_grid(nx, ny, 1, 2);
    if (rc) return rc;
    if (!u || !ut || nsteps < 0 || !(Lx > 0.0) || !(Ly > 0.0) || c < 0.0 || !(sigma > 0.0)) return -1;
    size_t plane = (size_t)(nx * ny);
    cplx *wx = root_table(nx), *wy = root_table(ny);
    double *k2 = ksq_table(nx, ny, Lx, Ly);
    cplx *U = (cplx *)u, *V = (cplx *)ut;
    cplx *s0 = (cplx *)malloc(sizeof(cplx) * plane);
    cplx *sh = (cplx *)malloc(sizeof(cplx) * plane);
    cplx *s1 = (cplx *)malloc(sizeof(cplx) * plane);
    double inv_area = 1.0 / ((double)nx * (double)ny);
    transform2d(nx, ny, U, 0, 2, wx, wy);                   /* u^ = F{f} */
    transform2d(nx, ny, V, 0, 2, wx, wy);                   /* v^ = F{g} */
    if (means) { means[0] = U[0].re * inv_area; means[1] = U[0].im * inv_area; }
    for (int64_t n = 0; n < nsteps; ++n) {
        double t = t0 + (double)n * dt;
        oracle_orbit_source(nx, ny, Lx, Ly, xmin, ymin, A, sigma, Omega, gamma, rs, t, (double *)s0);
        oracle_orbit_source(nx, ny, Lx, Ly, xmin, ymin, A, sigma, Omega, gamma, rs, t + 0.5 * dt, (double *)sh);
        oracle_orbit_source(nx, ny, Lx, Ly, xmin, ymin, A, sigma, Omega, gamma, rs, t + dt, (double *)s1);
        transform2d(nx, ny, s0, 0, 2, wx, wy);
        transform2d(nx, ny, sh, 0, 2, wx, wy);
        transform2d(nx, ny, s1, 0, 2, wx, wy);
        for (size_t i = 0; i < plane; ++i) {
            double w2 = c * c * k2[i];                        /* kappa^2 */
            cplx u0 = U[i], v0 = V[i];
            /* k1 = f(t, y) */
            cplx k1u = v0;
            cplx k1v = c_add(c_scale(u0, -w2), s0[i]);
            /* k2 = f(t + dt/2, y + dt/2 k1) */
            cplx u2 = c_add(u0, c_scale(k1u, 0.5 * dt)), v2 = c_add(v0, c_scale(k1v, 0.5 * dt));
            cplx k2u = v2;
            cplx k2v = c_add(c_scale(u2, -w2), sh[i]);
            /* k3 = f(t + dt/2, y + dt/2 k2) */
            cplx u3 = c_add(u0, c_scale(k2u, 0.5 * dt)), v3 = c_add(v0, c_scale(k2v, 0.5 * dt));
            cplx k3u = v3;
            cplx k3v = c_add(c_scale(u3, -w2), sh[i]);
            /* k4 = f(t + dt, y + dt k3) */
            cplx u4 = c_add(u0, c_scale(k3u, dt)), v4 = c_add(v0, c_scale(k3v, dt));
            cplx k4u = v4;
            cplx k4v = c_add(c_scale(u4, -w2), s1[i]);
            /* y(t + dt) = y + dt/6 (k1 + 2 k2 + 2 k3 + k4) */
            cplx su = c_add(c_add(k1u, c_scale(k2u, 2.0)), c_add(c_scale(k3u, 2.0), k4u));
            cplx sv = c_add(c_add(k1v, c_scale(k2v, 2.0)), c_add(c_scale(k3v, 2.0), k4v));
            U[i] = c_add(u0, c_scale(su, dt / 6.0));
            V[i] = c_add(v0, c_scale(sv, dt / 6.0));
        }
        if (means) { means[2 * (n + 1)] = U[0].re * inv_area; means[2 * (n + 1) + 1] = U[0].im * inv_area; }
    }
    transform2d(nx, ny, U, 1, 2, wx, wy);
    transform2d(nx, ny, V, 1, 2, wx, wy);
    free(s0); free(sh); free(s1); free(k2); free(wx); free(wy);
    return 0;
}

/* ------------------------------------------------------------------------ */
int oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

int oracle_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
