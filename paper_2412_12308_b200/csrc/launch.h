// launch.h -- host-side launchers of the pass kernels (internal to libfftpde.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fftpde {

// Peer pointers of the slab exchange (pack.cu), passed by value.
constexpr int kMaxPeers = 16;
constexpr int kFsMaxPeerMaps = 8;   // distributed four-step By peer stores: one tensor map per peer (R28)
struct PeerPtrs {
    void *p[kMaxPeers];
};
// Pass output scattered straight into the peers' slabs (the exchanges of the slab
// decomposition fused into the pass epilogues).  Row passes:
// element a of output row k goes to p[a >> bwlog] at row rank R + k, column
// a & (bw - 1), of a [P R][bw] column slab.  Column passes (on this rank's column
// slab [P R][bw]): element y of local column c goes to p[y / R] at row y mod R,
// column rank bw + c, of an [R][nx] row slab.  p[0] == nullptr: the ordinary store.
struct PeerOut {
    void *p[kMaxPeers] = {};
    int rank = 0;
    int bwlog = 0;
    int64_t R = 0;
    int64_t nx = 0;          // row-slab length (column passes)
};
#ifdef __CUDACC__
template <typename C> __device__ __forceinline__ C *peer_row_dst(const PeerOut &po, int64_t k, int64_t a)
{
    const int64_t bw = (int64_t)1 << po.bwlog;
    return reinterpret_cast<C *>(po.p[a >> po.bwlog]) + ((int64_t)po.rank * po.R + k) * bw + (a & (bw - 1));
}
template <typename C> __device__ __forceinline__ C *peer_col_dst(const PeerOut &po, int64_t y, int64_t c)
{
    const int64_t r = y / po.R;
    return reinterpret_cast<C *>(po.p[r]) + (y - r * po.R) * po.nx + ((int64_t)po.rank << po.bwlog) + c;
}
#endif

enum ColOp { COL_FWD = 0, COL_INV = 1, COL_POISSON = 2, COL_DIFFUSE = 3 };   // == PipeOp

// Device tables of the k-space multipliers; every multiplier includes the
// 1/(nx ny) of the inverse transform (exact: a power of two).
template <typename T> struct OpTables {
    const T *kx2, *ky2;      // |k|^2 per axis: (2 pi fold(a)/L)^2          (Poisson)
    const T *ex, *ey;        // exp(-D kx^2 dt)/(nx ny), exp(-D ky^2 dt)    (diffusion)
    const T *wC, *wS1, *wS2; // wave quadrant tables [qa][qb], scale folded in
    int64_t qpitch;          // ny/2 + 1
    int64_t nfold;           // x length for the quadrant index qa = min(a, nfold - a) (nx; real plans
                             // run the column passes over a padded half spectrum, so not the column count)
    T scale;                 // 1/(nx ny)
    // optional 2D row factor of the four-step passes (fourstep.cuh): the element
    // factor of line class cls is ey2d[cls * N + element], cls = line % ey2d_mod
    // (rows) or the batch index (columns); ex is then not applied
    const T *ey2d = nullptr;
    int64_t ey2d_mod = 1;
};

constexpr int64_t kMaxLen = 8192;    // single-CTA (one pass) axis length limit
constexpr int64_t kMaxLen2 = 32768;  // two-level (cluster) axis length limit

// radix (elements per thread) of the sub-transforms of the two-level column pass;
// the host builds its P and Q twiddle tables for the same factorisation
// row2d (long rows): points per thread / radix of its in-register stages
#ifndef FFTPDE_R2D_E
#define FFTPDE_R2D_E 16
#endif
#ifndef FFTPDE_COL2_EMAX
#define FFTPDE_COL2_EMAX 8
#endif

// Row transforms of `batch` grids: length n along x, ny rows per grid, grids
// `stride` elements apart.  dir: ROW_FWD, ROW_INV (unscaled), or ROW_MID (inverse
// stored to out2, then forward stored to out).
// ROW_DIFF: forward transform, times the per-wavenumber multiplier mul[a] (the x
// factor of a separable operator, 1/(nx ny) folded in), inverse transform, in
// one pass; `ones` is a table of 1s over the row index (the operator slot of the
// line kernels is (line, element)-separable).
enum RowDir { ROW_FWD = 0, ROW_DIFF = 3, ROW_INV = 4, ROW_MID = 5 };   // == PipeOp values
struct ColTw;
struct RowMul {
    const void *mul = nullptr;    // [nx] multiplier over the row's wavenumber index
    const void *ones = nullptr;   // [>= ny] ones
    const void *mul2d = nullptr;  // optional [mod][nx]: the factor of row r is mul2d[r % mod] (OpTables::ey2d)
    int64_t mod = 1;
};
template <typename T>
cudaError_t launch_rows(int64_t n, const void *in, void *out, void *out2, int64_t ny, int64_t stride,
                        int64_t batch, int dir, const ColTw &tw, cudaStream_t st, RowMul rm = {},
                        PeerOut po = {});

// Twiddle tables of the column axis: the single-level stage table of ny, and for
// the two-level (cluster) column pass the stage tables of P and Q (ny = P Q)
// plus the plain table w_ny^m, m < ny.
struct ColTw {
    const void *tw;      // stage table of the axis (radix 16)
    const void *twP, *twQ, *twN;
    const void *tw8;     // stage table of the axis (radix 8, line_kernel E = 8)
    const void *tw32 = nullptr;   // stage table of the axis (radix 32)
};

// Split ny = P * Q used by the two-level column pass (P = Q = 0: not used).
void col2_split(int64_t ny, int64_t nx, int elem_bytes, int64_t &P, int64_t &Q);
// Split nx = P * Q of the two-level row pass (rows longer than kMaxLen).
void row2_split(int64_t nx, int64_t &P, int64_t &Q);

// Long-row pass (nx = P Q > kMaxLen, row2d.cuh): dir = ROW_FWD, ROW_INV
// (unscaled) or ROW_MID (inverse -> out2, then forward -> out).  Tables (ColTw):
// twP, twQ = radix-16 stage tables of P and Q; twN = split inter-phase table.
template <typename T>
cudaError_t launch_rows2(int64_t nx, const void *in, void *out, void *out2, int64_t ny, int64_t stride,
                         int64_t batch, int dir, const ColTw &tw, cudaStream_t st, RowMul rm = {},
                         PeerOut po = {});

// Column pass along y (length ny) over nx columns, op in ColOp.
template <typename T>
cudaError_t launch_cols(int64_t ny, const void *in, void *out, int64_t nx, int64_t stride,
                        int64_t batch, int op, const ColTw &tw, const OpTables<T> &tab,
                        cudaStream_t st, PeerOut po = {});

// Wave column pass: both fields, in place.
template <typename T>
cudaError_t launch_wave_cols(int64_t ny, void *U, void *V, int64_t nx, int64_t stride,
                             int64_t batch, const ColTw &tw, const OpTables<T> &tab,
                             cudaStream_t st);

// Wave solve on a transposed internal spectrum T[kx][y] (wavet.cuh): complex128,
// nx, ny in {2048, 4096}, one grid.  Rows: op 0 physical -> T (forward), 1 T ->
// physical + T (inverse, materialise, forward), 2 T -> physical (inverse); in place
// on T.  Columns: the oscillator step of both fields on their transposed spectra.
enum WaveTOp { WT_FWD = 0, WT_MID = 1, WT_INV = 2 };
bool wave_t_supported(int64_t nx, int64_t ny);
cudaError_t launch_wave_t_rows(int op, void *T, const void *phys_in, void *phys_out, int64_t nx, int64_t ny,
                               const void *twx32, cudaStream_t st);
cudaError_t launch_wave_t_cols(void *TU, void *TV, int64_t nx, int64_t ny, const void *twy32,
                               const OpTables<double> &tab, cudaStream_t st);

// Single-CTA whole-grid solve (small square grids).
template <typename T> bool small_supported(int64_t nx, int64_t ny);
template <typename T>
cudaError_t launch_small(int64_t nx, int64_t ny, const void *in, void *out, int64_t stride,
                         int64_t batch, int op, const void *twx, const void *twy,
                         const OpTables<T> &tab, cudaStream_t st);

// ---- time-dependent source path (rk4.cu) ----
// Orbiting Gaussian source at one time t: the host evaluates
// x0 = rs cos(Omega t), y0 = rs sin(Omega t), amp = A cos(gamma t) in fp64.
struct SrcParams {
    double xmin, ymin, Lx, Ly;   // grid x_j = xmin + j Lx/nx, y_k = ymin + k Ly/ny
    double x0, y0, amp, sigma;
};
template <typename T>
cudaError_t launch_source(void *s, int64_t nx, int64_t ny, const SrcParams &p, cudaStream_t st);
// One RK4 step of du^/dt = v^, dv^/dt = -c^2 |k|^2 u^ + s^ on every mode, given
// s^ at t, t + dt/2, t + dt; optional mean_out <- u^(0,0)/(nx ny) after the step.
template <typename T>
cudaError_t launch_rk4(void *U, void *V, const void *S0, const void *Sh, const void *S1, int64_t nx, int64_t ny,
                       const void *kx2, const void *ky2, double c, double dt, void *mean_out, cudaStream_t st);
template <typename T>
cudaError_t launch_mean(const void *U, void *out, int64_t nx, int64_t ny, cudaStream_t st);

// ---- real-to-complex row passes (rc.cu) ----
// RC_DIFF: real row -> half spectrum, times mul[a], -> real row (the x factor of
// a separable operator), in one pass
enum RcOp { RC_FWD = 0, RC_INV = 1, RC_MID = 2, RC_DIFF = 3 };
template <typename T>
cudaError_t launch_rc_rows(int64_t nx, const void *in, void *out, void *out2, int64_t nrows, int64_t pitch, int op,
                           const void *tw, const void *twr, cudaStream_t st, const void *mul = nullptr);

// ---- diagonal k-space operators (kspace.cu) ----
enum KOp { KOP_LAPLACIAN = 0, KOP_DX = 1, KOP_DY = 2, KOP_DIFFSRC = 3 };
template <typename T>
cudaError_t launch_kop(void *X, const void *S, int64_t nx, int64_t ny, int64_t batch, int64_t stride, int op,
                       const void *kx, const void *ky, const void *kx2, const void *ky2, double D, double dt,
                       cudaStream_t st);

cudaError_t launch_peer_transpose(const void *src, const PeerPtrs &peers, int P, int rank, int64_t R,
                                  int64_t bw_bytes, int direction, cudaStream_t st);

// ---- four-step (Bailey) passes of the 32768^2 complex128 diffusion (fourstep.cu) ----
// op: 0 = AA (in -> out), 1 = AA^-1 (in -> out), 2 = MID (AA^-1 -> phys, then AA -> out).
// tw = w_32768^{a b}, a < 1024, b < 32.  The B passes are launch_rows / launch_cols
// over 1024-point lines with the 2D factors (OpTables::ey2d).
bool fourstep_supported(int64_t nx, int64_t ny, int64_t batch, int elem_bytes);
cudaError_t launch_aa(int op, const void *in, void *out, void *phys, const void *tw, cudaStream_t st);
// the distributed four-step of sharded plans (R28, fourstep.cu / pack.cu)
bool fs_dist_supported(int P);
cudaError_t launch_aa_part(int op, int P, int rank, int xmode, const void *in, void *out, void *phys, const void *tw,
                           cudaStream_t st);
cudaError_t launch_fs_b_part(bool cols, int P, int rank, void *f, const void *tw32, const double *m2d, cudaStream_t st,
                             const PeerPtrs *peers = nullptr);   // peers: store into the peers' other part
cudaError_t launch_fs_perm(const void *in, void *out, int P, int direction, cudaStream_t st);
cudaError_t launch_fs_bb(void *f, const void *tw32, const double *mx2d, const double *my2d, void *sync,
                         cudaStream_t st);
bool fs_bb_enabled();
cudaError_t launch_fs_b(bool cols, void *f, const void *tw32, const void *tw16, const OpTables<double> &tab,
                        cudaStream_t st);

// Block transpose of the sharded path (pack.cu); bw_bytes a multiple of 16.
cudaError_t launch_pack(const void *in, void *out, int64_t nrows, int64_t nblocks, int64_t bw_bytes,
                        int direction, cudaStream_t st);

} // namespace fftpde
