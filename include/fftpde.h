/*
 * fftpde.h -- C ABI of the B200-native 2D FFT-PDE hot path (arXiv 2412.12308).
 *
 * Every compute call runs hand-written sm_100a CUDA kernels (libfftpde.so);
 * there is no CPU fallback and no cuFFT.  PAPER.md below is the paper's LaTeX
 * source, cited by line; R1..R16 are the
 * readings of its silent or garbled points.
 *
 * Conventions (all calls)
 * -----------------------
 * Grids: [batch][ny][nx], C-contiguous, x fastest, interleaved complex
 *   (FFTPDE_C128: double re,im = 16 B/pt; FFTPDE_C64: float re,im = 8 B/pt).
 *   Element (b,k,j) is p_{jk} at x_j = j Lx/nx, y_k = k Ly/ny.
 * Spectra: natural order, index a <-> fold(a) = a (a <= n/2) else a - n
 *   (R2).  Angular wavenumber k_a = 2 pi fold(a)/Lx (R4).
 * Forward transform: P_ab = sum_jk p_jk e^{+2 pi i aj/nx} e^{+2 pi i bk/ny},
 *   unnormalised (2D_DFT; eq:DFT PAPER.md:119-124; R1, R3).
 * Inverse transform: conjugate kernel times 1/(nx ny).
 * Axis lengths: powers of two, 1 <= n <= 32768 per axis.
 *   Axes up to 8192 use one-CTA transforms; 16384 and 32768 use two-level
 *   cluster passes, which for columns need nx >= 128 B / element size (8
 *   columns for complex128, 16 for complex64); otherwise FFTPDE_ERR_UNSUPPORTED.
 *   With two-level column passes (ny >= 2048 and such nx) the plain
 *   transforms need the default grid stride nx*ny.
 *
 * Ownership: the caller owns every device buffer -- inputs, outputs and the
 *   workspace of fftpde_workspace_size() bytes (allocate it with torch).  The
 *   plan owns host-side state only and never calls cudaMalloc.
 * Execution: compute calls are asynchronous on the plan's stream (set with
 *   fftpde_set_stream; default: the legacy default stream).  Argument checks
 *   are synchronous and happen before anything is enqueued.  Launch errors
 *   are returned as FFTPDE_ERR_CUDA; device faults surface at the caller's
 *   next synchronisation.
 * Aliasing: in == out is allowed everywhere; inputs are otherwise not written.
 * Alignment: device pointers must be aligned to one complex element
 *   (16 B for FFTPDE_C128, 8 B for FFTPDE_C64); complex64 plans with
 *   nx >= 2048 (rows loaded by one bulk copy each) need 16-byte aligned
 *   pointers and, for batch > 1, a batch stride of an even number of
 *   elements.  Violations return FFTPDE_ERR_INVALID_ARG before any launch.
 * Threads: one host thread per plan at a time; distinct plans are independent.
 */
#ifndef FFTPDE_H
#define FFTPDE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fftpde_plan_s *fftpde_plan;

typedef enum { FFTPDE_C64 = 0, FFTPDE_C128 = 1 } fftpde_dtype;

typedef enum {
    FFTPDE_OK = 0,
    FFTPDE_ERR_INVALID_ARG = 1,  /* null pointer, bad dtype, non-finite/non-positive L, dt<0 (diffuse), nsteps<0, misaligned, stride < nx*ny */
    FFTPDE_ERR_EMPTY = 2,        /* a zero-sized axis or batch ("rejects empty input") */
    FFTPDE_ERR_NOT_POW2_X = 3,   /* nx not a power of two (radix-2 restriction) */
    FFTPDE_ERR_NOT_POW2_Y = 4,   /* ny not a power of two */
    FFTPDE_ERR_UNSUPPORTED = 5,  /* axis longer than this build supports, or batch outside the plan */
    FFTPDE_ERR_WORKSPACE = 6,    /* workspace missing or smaller than fftpde_workspace_size() */
    FFTPDE_ERR_CUDA = 7,         /* a CUDA runtime call or kernel launch failed */
    FFTPDE_ERR_NCCL = 8,         /* NCCL missing or failed (sharded plans) */
    FFTPDE_ERR_NOT_POW2_Z = 9    /* nz not a power of two (3D plans) */
} fftpde_status;

/* Create a plan for batch grids of ny x nx points on the periodic domain
 * [0,Lx) x [0,Ly) with complex dtype `dtype` on CUDA device
 * `device`.  Validates the arguments and builds the host tables (twiddles
 * w_n^m = e^{+2 pi i m/n} per index in fp64, kx^2, ky^2).  *plan is NULL on
 * error. */
fftpde_status fftpde_plan_2d(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t batch,
                             fftpde_dtype dtype, double Lx, double Ly, int device);

/* Real-field plan: real [batch][ny][nx] fields (FFTPDE_C128
 * plans take double data, FFTPDE_C64 plans float), whose spectra are Hermitian,
 * X_{n-a} = conj(X_a), so only a <= nx/2 is stored: fftpde_forward returns the half
 * spectrum [batch][ny][nx/2 + 1] (complex of the plan's precision, natural order,
 * + sign, unnormalised), fftpde_inverse takes it back to real (x 1/(nx ny));
 * fftpde_poisson, fftpde_diffuse and fftpde_wave_step act on real fields with the
 * same operators as the complex plans, moving half the bytes.  A real row of nx
 * values is transformed as nx/2 complex pairs and untangled with the even/odd split
 * of eq:FFTpairodd.  16 <= nx <= 16384 (complex128) /
 * 32 <= nx <= 16384 (complex64); ny as fftpde_plan_2d; whole-plan calls only
 * (the *_batched calls and the other operators return FFTPDE_ERR_UNSUPPORTED). */
fftpde_status fftpde_plan_2d_r2c(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t batch, fftpde_dtype dtype,
                                 double Lx, double Ly, int device);

/* Sharded plans: the slab decomposition over `nranks`
 * processes (one GPU each), NCCL inside the library.  Every rank calls the plan
 * constructor collectively with the same sizes, dtype, L and the same 128-byte
 * NCCL unique id (from fftpde_nccl_unique_id on rank 0, broadcast by the caller,
 * e.g. over the torch process group).
 *
 * 2D (fftpde_plan_2d_sharded): rank r owns rows [r ny/P, (r+1) ny/P) (its "row
 * slab", [ny/P][nx]).  Per step: rows -> pack -> grouped ncclSend/ncclRecv (an
 * all-to-all over NVLink) -> column-slab pass (forward along y, multiplier at the
 * global wavenumbers, inverse) -> all-to-all -> unpack -> inverse rows.
 * fftpde_forward: row slab -> the rank's spectral column slab [ny][nx/P]
 * (columns a in [r nx/P, (r+1) nx/P)), in != out; fftpde_inverse: column slab ->
 * row slab (x 1/(nx ny)).  P must divide nx and ny, (nx/P) * element size must be
 * a multiple of 16 bytes, and for ny > 8192 nx/P at least one 128-byte block.
 * fftpde_diffuse on nx = ny = 32768 complex128 with P a power of two <= 32 runs
 * the distributed four-step instead (R28; the four-step split of
 * PAPER.md:262-273 applied inside each axis, N = 1024 x 32): rank r holds the
 * field's rows with (y mod 1024) in [r M, r M + M) ("Y-part", M = 1024/P) or its
 * columns with (x mod 1024) in that range ("X-part"), both as [P][32][M][32][M];
 * per solve step the x-axis 1024-point diffusion pass on the Y-part, ONE
 * all-to-all (Y-part <-> X-part), the y-axis pass on the X-part and the combined
 * high-index pass that writes the physical field and starts the next step (the
 * parts alternate step by step).  The caller's row slabs are converted on entry
 * and exit (a permutation pass, an all-to-all and a block swap each way).
 * Same results on every P, bit for bit (tests/test_gpu_sharded.py).
 *
 * 3D (fftpde_plan_3d_sharded, SURVEY.md 8(f) row 4 on several GPUs): rank r owns
 * z-planes [r nz/P, (r+1) nz/P) (its "z-slab", [nz/P][ny][nx]).  Per step: x- and
 * y-passes of the local planes -> pack -> all-to-all -> z-pass with the multiplier
 * on the "y-slab" [nz][ny/P][nx] (rows [r ny/P, (r+1) ny/P) of every plane) ->
 * all-to-all -> unpack -> inverse y- and x-passes.  fftpde_forward returns the
 * y-slab of the spectrum, fftpde_inverse takes it back (x 1/(nx ny nz)).  P must
 * divide nz and ny.  One all-to-all per transform: a slab, not a pencil,
 * decomposition (needs nz >= P; fftpde_plan_3d_pencil lifts that).
 *
 * Whole-plan calls on a sharded plan (fftpde_forward / _inverse / _poisson /
 * _diffuse) are collective, in the same order on every rank; u0 == u allowed.
 * Loopback: nccl_unique_id = NULL and rank = FFTPDE_SHARDED_LOOPBACK builds one
 * plan that runs all P ranks on its device in a single process (each phase for
 * every rank in turn, the all-to-all as block copies): the caller's buffers then
 * hold the P slabs back to back (for row and z-slabs: the natural full field).  It
 * exercises the same per-rank kernels and index arithmetic as the NCCL path and is
 * what single-GPU tests use.
 * Errors: FFTPDE_ERR_INVALID_ARG for rank/nranks/id combinations other than the
 * two above; FFTPDE_ERR_UNSUPPORTED when P does not divide the sliced axes;
 * FFTPDE_ERR_NCCL when libnccl.so.2 cannot be loaded (dlopen) or
 * ncclCommInitRank fails. */
#define FFTPDE_SHARDED_LOOPBACK (-1)
fftpde_status fftpde_nccl_unique_id(void *out_128_bytes);
fftpde_status fftpde_plan_2d_sharded(fftpde_plan *plan, int64_t nx, int64_t ny, fftpde_dtype dtype, double Lx,
                                     double Ly, int device, const void *nccl_unique_id, int rank, int nranks);
fftpde_status fftpde_plan_3d_sharded(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t nz, fftpde_dtype dtype,
                                     double Lx, double Ly, double Lz, int device, const void *nccl_unique_id,
                                     int rank, int nranks);

/* 3D pencil plan ("3D extension with pencil decomposition";
 * the n-D extension of PAPER.md:275, whose per-axis transforms PAPER.md:262-273
 * apply along x, y and z in turn).  P = pz * py ranks on a pz x py process grid;
 * rank r = i py + j (i < pz, j < py) owns the x-pencil [nz/pz][ny/py][nx]: planes
 * [i nz/pz, (i+1) nz/pz), rows [j ny/py, (j+1) ny/py), every x.  Per transform:
 * x-pass -> all-to-all inside the row group (the py ranks of z-block i) -> the
 * y-pencil [nz/pz][ny][nx/py] (x-block j) -> y-pass -> all-to-all inside the
 * column group (the pz ranks of x-block j) -> the z-pencil [nz][ny/pz][nx/py]
 * (rows [i ny/pz, (i+1) ny/pz) of x-block j) -> z-pass with the multiplier ->
 * the same back.  Two all-to-alls per 3D transform over sub-groups of sizes py
 * and pz, so P may exceed nz (the z-slab plan needs P <= nz).
 * fftpde_forward: x-pencil -> this rank's z-pencil of the spectrum (in != out);
 * fftpde_inverse: z-pencil -> x-pencil (x 1/(nx ny nz)); fftpde_poisson /
 * fftpde_diffuse act on x-pencils.  Requires pz | nz, py | ny, py | nx, pz | ny
 * and (nx/py) * element size a multiple of 16 bytes (else
 * FFTPDE_ERR_UNSUPPORTED); nccl_unique_id / rank / loopback as for
 * fftpde_plan_3d_sharded (one NCCL communicator over all P ranks: each group
 * exchange is a grouped send/recv with the group's ranks).  Loopback: the
 * caller's buffers hold the P x-pencils (or z-pencils) back to back in rank
 * order -- not the natural [nz][ny][nx] field. */
fftpde_status fftpde_plan_3d_pencil(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t nz, fftpde_dtype dtype,
                                    double Lx, double Ly, double Lz, int device, const void *nccl_unique_id,
                                    int rank, int pz, int py);

/* 3D plan (the n-D extension): [nz][ny][nx] grids on
 * [0,Lx) x [0,Ly) x [0,Lz), x fastest.  Transforms are sequential 1D passes
 * along x, y and z; the whole-plan calls fftpde_forward / fftpde_inverse /
 * fftpde_poisson (-1/|k|^2, k = 0 zeroed) / fftpde_diffuse (exp(-D|k|^2 dt),
 * |k|^2 = kx^2 + ky^2 + kz^2) act on the volume; fftpde_wave_step, the
 * *_batched calls and the other operators return FFTPDE_ERR_UNSUPPORTED.
 * nz <= 32768: up to 1024 a single-level z-pass, beyond it the two-level
 * column pass (nz = P Q, one 128-byte block of adjacent lines per cluster), which
 * needs nx*ny * element size to be a multiple of 128 bytes (else
 * FFTPDE_ERR_UNSUPPORTED; the sharded and pencil plans check their own line
 * counts the same way); nx, ny as fftpde_plan_2d.
 * Errors as fftpde_plan_2d, plus FFTPDE_ERR_NOT_POW2_Z. */
fftpde_status fftpde_plan_3d(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t nz, fftpde_dtype dtype,
                             double Lx, double Ly, double Lz, int device);

/* Bytes of device workspace the plan needs (tables + operator tables). */
size_t fftpde_workspace_size(fftpde_plan plan);

/* Hand the plan a device workspace of >= fftpde_workspace_size() bytes,
 * 256-byte aligned; the plan uploads its tables into it on its stream.  The
 * caller keeps it alive until fftpde_destroy. */
fftpde_status fftpde_set_workspace(fftpde_plan plan, void *dev_ptr, size_t bytes);

/* Stream for all subsequent calls (a cudaStream_t, e.g. torch's
 * torch.cuda.current_stream().cuda_stream); NULL = legacy default stream. */
fftpde_status fftpde_set_stream(fftpde_plan plan, void *cuda_stream);

fftpde_status fftpde_destroy(fftpde_plan plan);
const char *fftpde_status_string(fftpde_status status);

/* Number of CUDA kernels the library enqueued since the plan was created
 * (instrumentation for bench.py's gpu_launches). */
int64_t fftpde_launch_count(fftpde_plan plan);

/* Per-kernel timing (instrumentation for bench.py's roofline).  While enabled,
 * every launch is bracketed by CUDA events on the plan's stream.
 * fftpde_read_profile synchronises on the recorded events, returns the summed
 * device time (ms) and launch count of one kernel class since the last read,
 * and resets them. */
#define FFTPDE_KERNEL_ROW 0       /* row pass (forward or inverse along x) */
#define FFTPDE_KERNEL_COL 1       /* column pass (transform, or forward + operator + inverse along y) */
#define FFTPDE_KERNEL_WAVE_COL 2  /* wave column pass (both fields) */
#define FFTPDE_KERNEL_SMALL 3     /* single-CTA whole-grid solve */
#define FFTPDE_KERNEL_POINTWISE 4 /* pointwise k-space / source kernels (RK4 path) */
#define FFTPDE_KERNEL_AA 5        /* four-step high-index pass (32768^2 complex128 diffusion) */
#define FFTPDE_KERNEL_CLASSES 6
fftpde_status fftpde_set_profiling(fftpde_plan plan, int enable);
fftpde_status fftpde_read_profile(fftpde_plan plan, int kernel_class, double *total_ms, int64_t *launches);

/* ---- transforms ------------------------------------------------------------
 * fftpde_forward: out = DFT2(in), + sign, unnormalised, natural order
 *   (2D_DFT PAPER.md:246-249, computed as row transforms then column
 *   transforms).
 * fftpde_inverse: out = iDFT2(in) = conj kernel x 1/(nx ny).
 * Both act on the plan's whole batch. */
fftpde_status fftpde_forward(fftpde_plan plan, const void *in, void *out);
fftpde_status fftpde_inverse(fftpde_plan plan, const void *in, void *out);

/* ---- solvers ---------------------------------------------------------------
 * fftpde_poisson: solve nabla^2 u = rho (eq:Poisson PAPER.md:286-291):
 *   u = iDFT2( m .* DFT2(rho) ), m = -1/|k|^2, m(0,0) = 0
 *   (eq:SolutionPoisson PAPER.md:329-331; zeroing k=0 == subtracting the mean,
 *   eq:Poisson2 PAPER.md:308-325; R5).  The input mean is ignored and u has
 *   zero mean.
 * fftpde_diffuse: nsteps exact steps of u_t = D nabla^2 u from u0
 *   (ec:solCalorFourier PAPER.md:376-386, coefficient D per R6): each step is
 *   DFT2, multiply by exp(-D |k|^2 dt), iDFT2, and materialises u (R8).  The
 *   multiplier is separable, exp(-D kx^2 dt) exp(-D ky^2 dt), so a step is
 *   computed as the 1D diffusion of every row followed by that of every column
 *   (the same operator, R26; one read and one write of u per axis).
 *   Single-grid complex128 32768 x 32768 plans split both axes four-step
 *   (N = 1024 x 32, R27): per step one pass of the high-index DFTs
 *   (which also writes u), then the 1024-point row and column diffusions; the
 *   intermediate lives in the workspace scratch.
 *   D >= 0, dt >= 0, nsteps >= 0 (0 copies u0 to u).  k = 0 is kept.
 * fftpde_wave_step: nsteps exact steps of u_tt = c^2 nabla^2 u (s = 0,
 *   eq:wave_equation PAPER.md:417-424) on the state (u, ut) in place: with
 *   kappa = c|k|, (U,V) <- (C U + S1 V, S2 U + C V), C = cos(kappa dt),
 *   S1 = sin(kappa dt)/kappa, S2 = -kappa sin(kappa dt); at kappa = 0,
 *   S1 = dt, S2 = 0 (eq:OmegaZero/OmegaNonZero PAPER.md:459-471; R7).
 *   Any finite dt (negative reverses time), c >= 0, nsteps >= 0.
 *   The propagator tables are computed on the host in fp64 for each new
 *   (c, dt) and uploaded into the workspace on the plan's stream. */
fftpde_status fftpde_poisson(fftpde_plan plan, const void *rho, void *u);
fftpde_status fftpde_diffuse(fftpde_plan plan, const void *u0, void *u,
                             double D, double dt, int64_t nsteps);
fftpde_status fftpde_wave_step(fftpde_plan plan, void *u, void *ut,
                               double c, double dt, int64_t nsteps);

/* ---- batched variants -------------------------------------------------------
 * Same semantics over `batch` grids (1 <= batch <= the plan's batch) whose
 * starts are `stride` elements apart (stride >= nx*ny). */
fftpde_status fftpde_forward_batched(fftpde_plan plan, const void *in, void *out,
                                     int64_t batch, int64_t stride);
fftpde_status fftpde_inverse_batched(fftpde_plan plan, const void *in, void *out,
                                     int64_t batch, int64_t stride);
fftpde_status fftpde_poisson_batched(fftpde_plan plan, const void *rho, void *u,
                                     int64_t batch, int64_t stride);
fftpde_status fftpde_diffuse_batched(fftpde_plan plan, const void *u0, void *u,
                                     int64_t batch, int64_t stride,
                                     double D, double dt, int64_t nsteps);
fftpde_status fftpde_wave_step_batched(fftpde_plan plan, void *u, void *ut,
                                       int64_t batch, int64_t stride,
                                       double c, double dt, int64_t nsteps);

/* ---- diagonal k-space operators ------------------------
 * fftpde_apply: out = iDFT2( m .* DFT2(in) ) over the plan's batch, with
 *   F{d^k u/dx^k} = (-i w)^k F{u} under the forward sign + (R1):
 *   FFTPDE_KOP_LAPLACIAN  m = -(kx^2 + ky^2)
 *   FFTPDE_KOP_DX         m = -i kx          (spectral d/dx)
 *   FFTPDE_KOP_DY         m = -i ky          (spectral d/dy)
 *   kx = 2 pi fold(a)/Lx with the Nyquist bin at +nx/2 (R2): odd operators see
 *   that choice (R24).  in == out allowed.  Unknown op:
 *   FFTPDE_ERR_INVALID_ARG.
 * fftpde_diffuse_source: nsteps exact steps of u_t = D nabla^2 u + s with a static
 *   source s (coefficient D per R6): per step u^ <- E u^ + Phi s^,
 *   E = exp(-D|k|^2 dt), Phi = (1 - E)/(D|k|^2) (k != 0, D > 0) or dt, each step
 *   materialising u (R8).  u0, s, u: [batch][ny][nx] (u0 == u allowed); scratch:
 *   >= fftpde_diffuse_source_scratch_size() bytes of device memory (two spectra
 *   per grid), caller-owned.  D >= 0, dt >= 0, nsteps >= 0 (0 copies u0). */
#define FFTPDE_KOP_LAPLACIAN 0
#define FFTPDE_KOP_DX 1
#define FFTPDE_KOP_DY 2
fftpde_status fftpde_apply(fftpde_plan plan, const void *in, void *out, int op);
size_t fftpde_diffuse_source_scratch_size(fftpde_plan plan);
fftpde_status fftpde_diffuse_source(fftpde_plan plan, const void *u0, const void *s, void *u, double D,
                                    double dt, int64_t nsteps, void *scratch, size_t scratch_bytes);

/* ---- time-dependent source: RK4 ------------------------
 * fftpde_wave_rk4: nsteps RK4 steps of dt (dt > 0) of the wave equation with the
 *   paper's orbiting Gaussian source, u_tt = c^2 nabla^2 u + s(t, x, y),
 *     s = A exp(-[(x - x0)^2 + (y - y0)^2]/sigma^2) cos(gamma t),
 *     x0 = rs cos(Omega t), y0 = rs sin(Omega t),
 *   sampled at x_j = xmin + j Lx/nx, y_k = ymin + k Ly/ny with periodic minimum
 *   images (R21), integrated in Fourier space as the first-order
 *   system du^/dt = v^, dv^/dt = -c^2|k|^2 u^ + s^(t) (eq:SystemOfODEsForWaveEquation,
 *   PAPER.md:448-454) with classical RK4, the source re-sampled and
 *   transformed at t, t + dt/2, t + dt of every step (R22).
 *   u, ut: the plan's grid (batch 1), physical fields at t0 on entry and at
 *   t0 + nsteps dt on exit (in place).  means: NULL or nsteps + 1 complex
 *   elements of the plan's dtype on the device, means[n] = grid mean of u at
 *   t0 + n dt (= u^(0,0)/(nx ny); the quantity of the paper's self-convergence
 *   test, eq:SCF PAPER.md:533-553).  scratch: >= fftpde_wave_rk4_scratch_size()
 *   bytes of device memory (5 spectra), caller-owned.
 *   Errors: FFTPDE_ERR_UNSUPPORTED for a batched plan; FFTPDE_ERR_INVALID_ARG for
 *   dt <= 0, nsteps < 0, c < 0, sigma <= 0, non-finite parameters, u == ut;
 *   FFTPDE_ERR_WORKSPACE if scratch is missing or too small. */
size_t fftpde_wave_rk4_scratch_size(fftpde_plan plan);
fftpde_status fftpde_wave_rk4(fftpde_plan plan, void *u, void *ut, double c,
                              double xmin, double ymin, double A, double sigma, double Omega,
                              double gamma, double rs, double t0, double dt, int64_t nsteps,
                              void *means, void *scratch, size_t scratch_bytes);

/* ---- slab (sharded) building blocks ------------------------------------------
 * The slab decomposition of SURVEY.md 8(e): rank r of P owns rows
 * [r ny/P, (r+1) ny/P); one step is rows -> all-to-all -> column slab pass ->
 * all-to-all -> inverse rows.  These calls are the per-rank pieces; the
 * exchange is done by the caller (torch.distributed / NCCL).
 *
 * fftpde_rows: transforms of `nrows` contiguous rows of length nx (any
 *   nrows >= 1) along x; inverse != 0 selects the conjugate kernel (unscaled).
 * fftpde_cols_slab: the column pass of a column slab: in/out hold the ncols
 *   columns col0 .. col0+ncols-1 of all ny rows, row-major with row length
 *   ncols (in == out allowed).  op = FFTPDE_OP_POISSON or FFTPDE_OP_DIFFUSE:
 *   forward along y, the multiplier at the GLOBAL wavenumbers (k_x of column
 *   col0 + c), inverse along y, 1/(nx ny) folded in (D, dt used by DIFFUSE).
 *   ncols must be a power of two dividing nx; col0 a multiple of ncols.
 * fftpde_pack_blocks: direction 0: [nrows][nblocks][bw] -> [nblocks][nrows][bw]
 *   (row slab -> per-peer send blocks); direction 1: the inverse.  bw in
 *   elements, bw * element size a multiple of 16 bytes.
 * fftpde_rows and fftpde_cols_slab take a plain complex 2D plan (fftpde_plan_2d);
 * 3D, real-field and sharded plans return FFTPDE_ERR_UNSUPPORTED. */
/* fftpde_peer_transpose: the exchange step itself as direct stores into the
 *   other ranks' buffers over NVLink (the fused alternative to
 *   fftpde_pack_blocks + an all-to-all): one kernel per rank, local coalesced
 *   reads, contiguous bw-element runs written to peer memory.
 *   direction 0: src = this rank's row-slab spectrum [R][P bw] (P bw = nx);
 *     columns [q bw, (q+1) bw) of row k go to peers[q] at row rank R + k of its
 *     column slab [P R][bw] (P R = ny).
 *   direction 1: src = this rank's column slab [P R][bw]; rows [s R, (s+1) R)
 *     go to peers[s]'s row slab [R][P bw] at columns [rank bw, (rank+1) bw).
 *   peers: host array of npeers (= P, <= 16) device pointers the calling device
 *   can store to (torch symmetric memory, CUDA IPC, or one device's buffers in a
 *   single-process emulation); rank < npeers; bw * element size a multiple of 16
 *   bytes.  Asynchronous on the plan's stream; the caller orders the phases across
 *   ranks with a stream-ordered barrier (every rank's stores complete before any
 *   rank reads its slab). */
fftpde_status fftpde_peer_transpose(fftpde_plan plan, const void *src, void *const *peers, int npeers, int rank,
                                    int64_t R, int64_t bw, int direction);

/* The distributed four-step of the 32768^2 complex128 diffusion (R28;
 * the four-step split N = 1024 x 32 of each axis, PAPER.md:262-273 applied inside
 * the axis) as per-rank pieces, for callers that run their own ranks and exchanges
 * (sharded.FusedFourStepSolver: torch symmetric memory, the exchange fused into
 * the B passes).  plan: a plain 2D plan of the whole 32768 x 32768 complex128
 * grid (batch 1); anything else returns FFTPDE_ERR_UNSUPPORTED.  nranks = P, a
 * power of two <= 32; M = 1024 / P.  A rank's PART is an array of 2^30 / P
 * complex128 in the layout [P][32][M][32][M]:
 *   Y-part (xmode 0) of rank r: element (blk q, a, m1_l, b, n1_l) is grid point
 *     y = (r M + m1_l) + 1024 a, x = (q M + n1_l) + 1024 b;
 *   X-part (xmode 1) of rank q: element (blk r, a, m1_l, b, n1_l) is the same
 *     point (r M + m1_l) + 1024 a, (q M + n1_l) + 1024 b;
 * (in the AA domain a, b are the high-index wavenumbers l1, k1).  So block q of
 * rank r's Y-part and block r of rank q's X-part hold the same points in the same
 * order: the Y <-> X transpose is an all-to-all of whole blocks.
 * fftpde_fs_part_aa: op 0 AA (physical part -> AA domain), 1 AA^-1 (-> physical,
 *   x 1 / N^2 from the B passes' factors), 2 MID (AA^-1 -> phys, then AA -> out);
 *   in == out allowed; phys only for op 2.
 * fftpde_fs_part_b: the 1024-point diffusion of the part's local axis (xmode 0: x
 *   on a Y-part, xmode 1: y on an X-part) with e^{-D k^2 dt}/32768, in place when
 *   peers == NULL; with peers (npeers == nranks device pointers, peer-mapped:
 *   torch symmetric memory, CUDA IPC, or one device's buffers in a single-process
 *   emulation) the result is stored straight into the OTHER part of every rank
 *   (block q -> peers[q] at block `rank`; xmode 1 needs nranks <= 8), f is left
 *   unchanged, and the caller orders the phase against the peers with a
 *   stream-ordered barrier.
 * fftpde_fs_part_perm: direction 0: a rank's row slab (rows [r 32768/P, ..)) ->
 *   [P][P][32/P][M][32][M] (block r = the part of the slab Y-part rank r owns,
 *   in its order); direction 1 the inverse (in != out).
 * Pointers 16-byte aligned, on the plan's device; asynchronous on its stream. */
fftpde_status fftpde_fs_part_aa(fftpde_plan plan, int op, int nranks, int rank, int xmode, const void *in, void *out,
                                void *phys);
fftpde_status fftpde_fs_part_b(fftpde_plan plan, int xmode, int nranks, int rank, void *f, double D, double dt,
                               void *const *peers, int npeers);
fftpde_status fftpde_fs_part_perm(fftpde_plan plan, int nranks, const void *in, void *out, int direction);

/* fftpde_rows_to_peers: the row pass of this rank's slab with the exchange fused
 *   into its epilogue: the output element a of row k is
 *   stored straight into peers[a / bw] at row rank R + k, column a mod bw, of
 *   that rank's column slab [npeers R][bw], bw = nx / npeers (a power of two).
 *   plan: the plain complex 2D plan of the whole grid (ny = npeers R); in: the
 *   row slab [R][nx] on the plan's device; peers: npeers peer-mapped device
 *   pointers (<= 16; symmetric memory, CUDA IPC, or one device's buffers in a
 *   single-process emulation).  op: FFTPDE_ROWS_FWD (forward transform along x,
 *   PAPER.md:262-266) or FFTPDE_ROWS_DIFFUSE (forward, times
 *   exp(-D kx^2 dt)/(nx ny), inverse: the x factor of the separable diffusion
 *   step, R26; D, dt used).  Asynchronous on the plan's stream; the caller orders
 *   it against the peers' next phase with a stream-ordered barrier. */
#define FFTPDE_ROWS_FWD 0
#define FFTPDE_ROWS_DIFFUSE 3
fftpde_status fftpde_rows_to_peers(fftpde_plan plan, const void *in, void *const *peers, int npeers, int rank,
                                   int64_t R, int op, double D, double dt);

/* fftpde_cols_to_peers: the column pass of this rank's column slab [npeers R][bw]
 *   (global columns rank bw .. rank bw + bw - 1) with the return exchange fused
 *   into its epilogue: the output element of slab row y, local column c, is
 *   stored straight into peers[y / R] at row y mod R, column rank bw + c, of that
 *   rank's row slab [R][nx].  op: FFTPDE_OP_POISSON, FFTPDE_OP_DIFFUSE (the 2D
 *   multiplier at the global wavenumbers) or FFTPDE_OP_DIFFUSE_Y (the y factor of
 *   the separable step, R26).  The slab is used as the pass's scratch (its contents
 *   are not preserved).  Same plan, peers and ordering rules as
 *   fftpde_rows_to_peers. */
fftpde_status fftpde_cols_to_peers(fftpde_plan plan, void *colslab, void *const *peers, int npeers, int rank,
                                   int64_t R, int op, double D, double dt);

#define FFTPDE_OP_POISSON 2
#define FFTPDE_OP_DIFFUSE 3
#define FFTPDE_OP_DIFFUSE_Y 5     /* cols_slab: the y factor exp(-D ky^2 dt) alone (R26) */
fftpde_status fftpde_rows(fftpde_plan plan, const void *in, void *out, int64_t nrows, int inverse);
fftpde_status fftpde_cols_slab(fftpde_plan plan, const void *in, void *out, int64_t col0, int64_t ncols,
                               int op, double D, double dt);
fftpde_status fftpde_pack_blocks(fftpde_plan plan, const void *in, void *out, int64_t nrows,
                                 int64_t nblocks, int64_t bw, int direction);

#ifdef __cplusplus
}
#endif
#endif /* FFTPDE_H */
