// fftpde_api.cu -- the C ABI (include/fftpde.h): plans, host tables, dispatch.
//
// Host-side responsibilities (everything on the device is in kernels.cuh):
//   * argument validation (synchronous, before anything is enqueued);
//   * fp64 tables: twiddles w_n^m = e^{+2 pi i m/n} per index (eq:DFT,
//     PAPER.md:124), |k|^2 per axis with k = 2 pi fold(a)/L (PAPER.md:106-109,
//     175, 253-258, 296-303; R2, R4), the diffusion factors
//     exp(-D k^2 dt) (ec:solCalorFourier PAPER.md:378-386) and the wave
//     propagator quadrant (eq:OmegaZero/NonZero PAPER.md:459-471);
//   * the pass sequence of each call (3 passes per solve step).
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <type_traits>
#include <utility>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: NCCL is loaded at run time (dlopen), not linked

#include "../../include/fftpde.h"
#include "launch.h"

using namespace fftpde;

struct fftpde_plan_s {
    int64_t nx = 0, ny = 0, batch = 0;
    fftpde_dtype dtype = FFTPDE_C128;
    double Lx = 1.0, Ly = 1.0;
    int device = 0;
    cudaStream_t stream = nullptr;
    unsigned char *ws = nullptr;
    size_t ws_bytes = 0;
    // workspace offsets (bytes)
    size_t o_one = 0, o_twx = 0, o_twy = 0, o_twx8 = 0, o_twy8 = 0, o_twx32 = 0, o_twy32 = 0, o_kx = 0, o_ky = 0, o_kx2 = 0, o_ky2 = 0, o_ex = 0, o_ey = 0, o_wc = 0, o_ws1 = 0, o_ws2 = 0;
    size_t o_twP = 0, o_twQ = 0, o_twN = 0;   // two-level column pass tables (P, Q > 0)
    size_t o_scr = 0;                          // scratch: row spectra of 2 fields (multi-step solves)
    int64_t colP = 0, colQ = 0;
    std::vector<double> twP, twQ, twN;
    size_t o_rtwP = 0, o_rtwQ = 0, o_rtwN = 0;   // two-level row pass tables (nx > kMaxLen)
    int64_t rowP = 0, rowQ = 0;
    std::vector<double> rtwP, rtwQ, rtwN;   // row2d: radix-16 stage tables of P, Q; split inter-phase table
    // four-step diffusion passes (fourstep.cuh; 32768^2 complex128 single grids, R27)
    bool fs = false;
    bool fsd = false;   // sharded 32768^2 complex128 plan: the distributed four-step (R28) with the fs tables
    std::vector<double> fs_tw, fs_tw32, fs_tw16;   // w_N^{ab} (a < 1024, b < 32); radix-32 / -16 stage tables of 1024
    size_t o_fs_tw = 0, o_fs_tw32 = 0, o_fs_tw16 = 0, o_fs_mx = 0, o_fs_my = 0, o_fs_sync = 0;
    size_t need = 0;
    int64_t qx = 0, qy = 0;   // quadrant extents nx/2+1, ny/2+1
    // host tables (fp64)
    std::vector<double> twx, twy;   // interleaved re, im (radix-16 stage tables)
    std::vector<double> twx8, twy8; // radix-8 stage tables (line_kernel E = 8)
    std::vector<double> twx32, twy32; // radix-32 stage tables
    std::vector<double> kx2, ky2;
    std::vector<double> kx, ky;     // signed 2 pi fold(a)/L (odd operators)
    bool diff_valid = false;
    double diff_D = 0, diff_dt = 0;
    bool wave_valid = false;
    double wave_c = 0, wave_dt = 0;
    int64_t launches = 0;
    // 3D plans (fftpde_plan_3d): the 2D machinery runs with batch = nz slabs; the
    // z-pass is a column pass of length nz over the nx*ny lines of the volume
    // sharded plans (fftpde_plan_2d_sharded): this rank's row slab [R][nx], R = ny/P
    bool sharded = false;
    int P = 1, rank = 0;
    bool loopback = false;                     // all P ranks in this one plan (single-process emulation)
    bool nccl_failed = false;                  // an NCCL call of the last exchange did not return ncclSuccess
    ncclComm_t comm = nullptr;
    int64_t R = 0, BW = 0, nzl = 0, slab_elems = 0;
    // 3D pencil plans (fftpde_plan_3d_pencil): P = Pz x Py ranks, rank r = i Py + j owns
    // the x-pencil [nzl][nyl][nx] (z-block i, y-block j); the y-pencil [nzl][ny][nxl]
    // (x-block j) after the row-group exchange; the z-pencil [nz][nyl2][nxl] (y-block i
    // of ny/Pz) after the column-group exchange
    bool pencil = false;
    int Pz = 1, Py = 1;
    int64_t nyl = 0, nxl = 0, nyl2 = 0;
    size_t o_shA = 0, o_shB = 0, o_shC = 0;
    bool is3d = false;
    // real plans (fftpde_plan_2d_r2c): half spectrum [batch][ny][pitch], pitch = nx/2 + LPP
    bool is_real = false;
    int64_t pitch = 0;
    std::vector<double> twm, twr;   // radix-16 stage table of nx/2; w_nx^a, a <= nx/2
    size_t o_twm = 0, o_twr = 0;
    int64_t nz = 1;
    double Lz = 1.0;
    std::vector<double> twz, twz8, kz2, kxy2;
    int64_t zP = 0, zQ = 0;                    // nz > 1024: the z-pass is the two-level col2 pass, nz = zP zQ
    std::vector<double> twPz, twQz, twNz;
    size_t o_twPz = 0, o_twQz = 0, o_twNz = 0;
    size_t o_twz = 0, o_twz8 = 0, o_kz2 = 0, o_kxy2 = 0, o_exy = 0, o_ez = 0, o_zscale = 0;
    bool diff3_valid = false;
    double diff3_D = 0, diff3_dt = 0;
    // optional per-launch timing (fftpde_set_profiling): event pairs per kernel class
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[FFTPDE_KERNEL_CLASSES];
    std::vector<cudaEvent_t> event_pool;
    double prof_ms[FFTPDE_KERNEL_CLASSES] = {0};
    int64_t prof_n[FFTPDE_KERNEL_CLASSES] = {0};
    // CUDA graphs of multi-step solves (one host launch per solve instead of 3 per step)
    struct Graph {
        std::array<uint64_t, 6> key;
        cudaGraphExec_t exec;
        int64_t launches;
        // profiling graphs: the event pairs recorded around each kernel node
        std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof;
    };
    bool capturing = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> cap_prof;
    std::vector<Graph> graphs;
    cudaStream_t cap_stream = nullptr;
    bool use_graphs = true;
};

namespace {

bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// w_n^m = exp(+2 pi i m/n).  m is reduced exactly modulo n, the angle is
// folded by symmetry into [0, pi/4] and evaluated in long double, then
// rounded once; quarter-turn values are exact.
void unit_root(int64_t n, int64_t m, double &re, double &im)
{
    int64_t r = m % n;
    if (r < 0) r += n;
    bool conj = false;
    if (2 * r > n) { r = n - r; conj = true; }            // e^{-i t} = conj e^{i t}
    bool mirror = false;                                    // angle in (pi/2, pi]: pi - t
    if (4 * r > n) { r = n - 2 * r; mirror = true; } else { r = 2 * r; }
    // now angle = pi * r / n  with r in [0, n/2] (units of pi/n)
    bool swap = false;                                      // angle in (pi/4, pi/2]: pi/2 - t
    if (4 * r > n) { r = n - 2 * r; swap = true; } else { r = 2 * r; }
    // now angle = (pi/2) r / n, r in [0, n/2] -> angle in [0, pi/4]
    const long double phi = (long double)r / (long double)n * 1.5707963267948966192313216916397514L;
    long double c = cosl(phi), s = sinl(phi);
    if (swap) { long double t = c; c = s; s = t; }
    if (mirror) c = -c;
    if (conj) s = -s;
    re = (double)c;
    im = (double)s;
}

// Stage-major twiddle table of the Stockham factorisation n = E^s * R used by
// the kernels (fft_core.cuh Shape<n>): per middle stage (Ns = E, E^2, ...)
// w_{Ns E}^{m k} at [m Ns + k]; then the last stage w_n^{m j} at [m Ns_last + j].
// Each entry is w_M^q = w_n^{q n / M}, evaluated directly from its index.
void build_twiddles(int64_t n, std::vector<double> &tw, int64_t emax = 16)
{
    const int64_t E = n < emax ? n : emax;
    tw.clear();
    auto put = [&](int64_t M, int64_t q) {
        double re, im;
        unit_root(M, q, re, im);
        tw.push_back(re);
        tw.push_back(im);
    };
    int64_t ns = 1;
    while (ns * E < n) {
        if (ns > 1)
            for (int64_t m = 0; m < E; ++m)
                for (int64_t k = 0; k < ns; ++k) put(ns * E, m * k);
        ns *= E;
    }
    if (ns > 1)
        for (int64_t m = 0; m < n / ns; ++m)
            for (int64_t j = 0; j < ns; ++j) put(n, m * j);
    if (tw.empty()) { tw.push_back(1.0); tw.push_back(0.0); }
}

// 2 pi fold(a) / L, fold(a) = a for a <= n/2 else a - n (Nyquist at +n/2, R2)
void build_k(int64_t n, double L, std::vector<double> &k)
{
    k.resize((size_t)n);
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t a = 0; a < n; ++a) k[(size_t)a] = two_pi * (double)((2 * a <= n) ? a : a - n) / L;
}

// (2 pi fold(a) / L)^2, fold(a) = a for a <= n/2 else a - n
void build_k2(int64_t n, double L, std::vector<double> &k2)
{
    k2.resize((size_t)n);
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t a = 0; a < n; ++a) {
        const int64_t f = (2 * a <= n) ? a : a - n;
        const double k = two_pi * (double)f / L;
        k2[(size_t)a] = k * k;
    }
}

// Plain table w_n^m, m < n (the inter-phase twiddles w_N^{n1 k1} of the two-level pass).
void build_plain_twiddles(int64_t n, std::vector<double> &tw)
{
    tw.resize(2 * (size_t)n);
    for (int64_t m = 0; m < n; ++m) unit_root(n, m, tw[2 * m], tw[2 * m + 1]);
}

// Inter-phase twiddles w_N^{n1 k1} of the four-step row pass (row2d.cuh), as
// products of two small tables, every entry rounded once from its exact angle:
// S1[n1][l] = w^{n1 l}, S2[n1][h] = w^{16 n1 h}, U1[k1][l] = w^{k1 l}, U2[k1][h] = w^{16 k1 h}.
void build_split_twiddles(int64_t n, int64_t P, int64_t Q, std::vector<double> &tw)
{
    tw.clear();
    auto put = [&](int64_t m) {
        double re, im;
        unit_root(n, m, re, im);
        tw.push_back(re);
        tw.push_back(im);
    };
    for (int64_t a = 0; a < P; ++a)
        for (int64_t l = 0; l < 16; ++l) put(a * l);
    for (int64_t a = 0; a < P; ++a)
        for (int64_t h = 0; h < Q / 16; ++h) put(16 * a * h);
    for (int64_t k = 0; k < Q; ++k)
        for (int64_t l = 0; l < 16; ++l) put(k * l);
    for (int64_t k = 0; k < Q; ++k)
        for (int64_t h = 0; h < P / 16; ++h) put(16 * k * h);
}

// Tables of the four-step passes (fourstep.cuh, N = 1024 x 32 on both axes):
// tw[a][b] = w_N^{a b}, a < 1024, b < 32; the radix-32 stage table of 1024 (line passes).
void build_fourstep_tables(int64_t n, std::vector<double> &tw, std::vector<double> &tw32, std::vector<double> &tw16)
{
    tw.clear();
    double re, im;
    for (int64_t a = 0; a < 1024; ++a)
        for (int64_t b = 0; b < 32; ++b) {
            unit_root(n, a * b, re, im);
            tw.push_back(re);
            tw.push_back(im);
        }
    build_twiddles(1024, tw32, 32);
    build_twiddles(1024, tw16, 16);
}

// The factor m(k) of an axis in the four-step B-pass order [k1][k2], k = k1 + 32 k2.
std::vector<double> fourstep_mul_order(const std::vector<double> &m)
{
    std::vector<double> o(m.size());
    for (size_t k1 = 0; k1 < 32; ++k1)
        for (size_t k2 = 0; k2 < 1024; ++k2) o[k1 * 1024 + k2] = m[k1 + 32 * k2];
    return o;
}

template <typename T> std::vector<T> cast_vec(const std::vector<double> &v)
{
    std::vector<T> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = (T)v[i];
    return o;
}

size_t elem_real(const fftpde_plan p) { return p->dtype == FFTPDE_C128 ? 8 : 4; }
size_t elem_cplx(const fftpde_plan p) { return 2 * elem_real(p); }

fftpde_status cuda_status(cudaError_t e) { return e == cudaSuccess ? FFTPDE_OK : FFTPDE_ERR_CUDA; }

// Upload a double host vector as the plan's real type.
fftpde_status upload(fftpde_plan p, size_t off, const std::vector<double> &v)
{
    cudaError_t e;
    if (p->dtype == FFTPDE_C128) {
        e = cudaMemcpyAsync(p->ws + off, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice,
                            p->stream);
    } else {
        std::vector<float> f = cast_vec<float>(v);
        e = cudaMemcpyAsync(p->ws + off, f.data(), f.size() * sizeof(float), cudaMemcpyHostToDevice,
                            p->stream);
        // pageable source: the call returns after staging, so f may be freed
    }
    return cuda_status(e);
}

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

template <typename T> OpTables<T> tables(fftpde_plan p)
{
    OpTables<T> t;
    t.kx2 = (const T *)(p->ws + p->o_kx2);
    t.ky2 = (const T *)(p->ws + p->o_ky2);
    t.ex = (const T *)(p->ws + p->o_ex);
    t.ey = (const T *)(p->ws + p->o_ey);
    t.wC = (const T *)(p->ws + p->o_wc);
    t.wS1 = (const T *)(p->ws + p->o_ws1);
    t.wS2 = (const T *)(p->ws + p->o_ws2);
    t.qpitch = p->qy;
    t.nfold = p->nx;
    t.scale = (T)(1.0 / ((double)p->nx * (double)p->ny));
    return t;
}

// element-aligned device pointer (16 B for complex128, 8 B for complex64)
// Rows of >= 2048 points are loaded by one cp.async.bulk per row (pipe.cuh BULK),
// which needs a 16-byte aligned global address: for complex64 plans with such
// rows the buffers (and the batch stride in bytes) must be 16-byte aligned too,
// otherwise the copy would fault and poison the context (fftpde.h "Alignment").
static bool needs_bulk_alignment(fftpde_plan p) { return elem_cplx(p) < 16 && p->nx >= 2048; }

fftpde_status check_ptr(fftpde_plan p, const void *ptr)
{
    if (!ptr) return FFTPDE_ERR_INVALID_ARG;
    if (((uintptr_t)ptr % elem_cplx(p)) != 0) return FFTPDE_ERR_INVALID_ARG;
    if (needs_bulk_alignment(p) && ((uintptr_t)ptr % 16) != 0) return FFTPDE_ERR_INVALID_ARG;
    return FFTPDE_OK;
}

fftpde_status check_call(fftpde_plan p, int64_t batch, int64_t stride)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->is3d || p->is_real || p->sharded) return FFTPDE_ERR_UNSUPPORTED;   // whole-plan entry points only
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    if (batch == 0) return FFTPDE_ERR_EMPTY;
    if (batch < 0 || stride < p->nx * p->ny) return FFTPDE_ERR_INVALID_ARG;
    if (needs_bulk_alignment(p) && batch > 1 && (stride * (int64_t)elem_cplx(p)) % 16 != 0)
        return FFTPDE_ERR_INVALID_ARG;
    if (batch > p->batch) return FFTPDE_ERR_UNSUPPORTED;
    return FFTPDE_OK;
}

cudaEvent_t pool_event(fftpde_plan p)
{
    if (!p->event_pool.empty()) {
        cudaEvent_t e = p->event_pool.back();
        p->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Launch `f` counting it, and bracket it with events when profiling.
template <typename F> cudaError_t launch(fftpde_plan p, int cls, F &&f)
{
    ++p->launches;
    if (!p->profiling) return f();
    cudaEvent_t a = pool_event(p), b = pool_event(p);
    // inside a stream capture, External records become event-record nodes of the graph
    const unsigned flags = p->capturing ? cudaEventRecordExternal : 0u;
    cudaEventRecordWithFlags(a, p->stream, flags);
    cudaError_t e = f();
    cudaEventRecordWithFlags(b, p->stream, flags);
    if (p->capturing) p->cap_prof.push_back({cls, {a, b}});
    else p->pending[cls].emplace_back(a, b);
    return e;
}

// ---- pass sequences --------------------------------------------------------
// ---- NCCL, loaded at run time (the process's libnccl, e.g. the one torch loaded) --
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};
const NcclApi &nccl()
{
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
        a.send = (decltype(a.send))dlsym(h, "ncclSend");
        a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.groupStart && a.groupEnd && a.send && a.recv;
        return a;
    }();
    return api;
}

template <typename T> struct Passes {
    using Real = T;
    fftpde_plan p;
    int64_t batch, stride;
    const void *twx() const { return p->ws + p->o_twx; }
    const void *twy() const { return p->ws + p->o_twy; }
    // the z-pass tables (3D): single-level stage tables, + the col2 tables when nz > 1024
    ColTw ztw() const
    {
        return ColTw{p->ws + p->o_twz, p->zP ? p->ws + p->o_twPz : nullptr, p->zP ? p->ws + p->o_twQz : nullptr,
                     p->zP ? p->ws + p->o_twNz : nullptr, p->ws + p->o_twz8};
    }
    ColTw rtw() const
    {
        return ColTw{twx(), p->ws + p->o_rtwP, p->ws + p->o_rtwQ, p->ws + p->o_rtwN, p->ws + p->o_twx8,
                     p->ws + p->o_twx32};
    }
    cudaError_t rows(const void *in, void *out, int inverse)
    {
        return launch(p, FFTPDE_KERNEL_ROW, [&] {
            if (p->rowP)   // long rows: DSMEM four-step cluster pass
                return launch_rows2<T>(p->nx, in, out, nullptr, p->ny, stride, batch, inverse ? ROW_INV : ROW_FWD,
                                       rtw(), p->stream);
            return launch_rows<T>(p->nx, in, out, nullptr, p->ny, stride, batch, inverse ? ROW_INV : ROW_FWD,
                                  rtw(), p->stream);
        });
    }
    // inverse rows of step s (physical field -> phys) + forward rows of step s+1 (-> spec)
    cudaError_t rows_mid(const void *in, void *spec, void *phys)
    {
        return launch(p, FFTPDE_KERNEL_ROW, [&] {
            if (p->rowP)
                return launch_rows2<T>(p->nx, in, spec, phys, p->ny, stride, batch, ROW_MID, rtw(), p->stream);
            return launch_rows<T>(p->nx, in, spec, phys, p->ny, stride, batch, ROW_MID, rtw(), p->stream);
        });
    }
    void *scratch(int field) const
    {
        return p->ws + p->o_scr + (size_t)field * (size_t)(p->batch * p->nx * p->ny) * elem_cplx(p);
    }
    ColTw ctw() const
    {
        return ColTw{twy(), p->ws + p->o_twP, p->ws + p->o_twQ, p->ws + p->o_twN, p->ws + p->o_twy8,
                     p->ws + p->o_twy32};
    }
    cudaError_t cols(const void *in, void *out, int op)
    {
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->nx, stride, batch, op, ctw(), tables<T>(p), p->stream);
        });
    }
    cudaError_t wave_cols(void *U, void *V)
    {
        return launch(p, FFTPDE_KERNEL_WAVE_COL, [&] {
            return launch_wave_cols<T>(p->ny, U, V, p->nx, stride, batch, ctw(), tables<T>(p), p->stream);
        });
    }
    bool small() const { return small_supported<T>(p->nx, p->ny); }
    cudaError_t small_op(const void *in, void *out, int op)
    {
        return launch(p, FFTPDE_KERNEL_SMALL, [&] {
            return launch_small<T>(p->nx, p->ny, in, out, stride, batch, op, twx(), twy(), tables<T>(p),
                                   p->stream);
        });
    }
    // one step of a diagonal k-space operator: DFT2 -> multiply -> iDFT2
    cudaError_t solve_step(const void *in, void *out, int op)
    {
        if (small()) return small_op(in, out, op);
        cudaError_t e = rows(in, out, 0);
        if (e == cudaSuccess) e = cols(out, out, op);
        if (e == cudaSuccess) e = rows(out, out, 1);
        return e;
    }
    // plain transforms; the two-level column pass is out of place through the scratch
    cudaError_t forward(const void *in, void *out)
    {
        if (small()) return small_op(in, out, COL_FWD);
        if (p->colP) {
            void *S = scratch(0);
            cudaError_t e = rows(in, S, 0);
            return e == cudaSuccess ? cols(S, out, COL_FWD) : e;
        }
        cudaError_t e = rows(in, out, 0);
        if (e == cudaSuccess) e = cols(out, out, COL_FWD);
        return e;
    }
    cudaError_t inverse(const void *in, void *out)
    {
        if (small()) return small_op(in, out, COL_INV);
        if (p->colP) {
            void *S = scratch(0);
            cudaError_t e = cols(in, S, COL_INV);
            return e == cudaSuccess ? rows(S, out, 1) : e;
        }
        cudaError_t e = cols(in, out, COL_INV);
        if (e == cudaSuccess) e = rows(out, out, 1);
        return e;
    }
    // nsteps diffusion steps: the row spectrum lives in the workspace scratch;
    // between column passes one fused row pass writes the physical field of
    // step s (materialised in u) and the row spectrum of step s+1.
    // Separable diffusion (R17, R26): exp(-D|k|^2 dt) = ex(a) ey(b), so one
    // step is the 1D diffusion of every row (forward, times ex / (nx ny), inverse)
    // followed by that of every column (times ey): two passes of one read and one
    // write each, in place, u materialised after every step.
    RowMul rowmul() const { return RowMul{p->ws + p->o_ex, p->ws + p->o_one}; }
    cudaError_t rows_diff(const void *in, void *out)
    {
        return launch(p, FFTPDE_KERNEL_ROW, [&] {
            if (p->rowP)
                return launch_rows2<T>(p->nx, in, out, nullptr, p->ny, stride, batch, ROW_DIFF, rtw(), p->stream,
                                       rowmul());
            return launch_rows<T>(p->nx, in, out, nullptr, p->ny, stride, batch, ROW_DIFF, rtw(), p->stream,
                                  rowmul());
        });
    }
    cudaError_t cols_diff_y(const void *in, void *out)
    {
        OpTables<T> t = tables<T>(p);
        t.ex = (const T *)(p->ws + p->o_one);               // the x factor was applied by the rows
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->nx, stride, batch, COL_DIFFUSE, ctw(), t, p->stream);
        });
    }
    cudaError_t diffuse(const void *u0, void *u, int64_t nsteps)
    {
        if (small()) {
            cudaError_t e = cudaSuccess;
            for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k)
                e = small_op(k == 0 ? u0 : u, u, COL_DIFFUSE);
            return e;
        }
        if (stride != p->nx * p->ny) {          // custom grid stride: in place, 3 passes per step
            cudaError_t e = cudaSuccess;
            for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) e = solve_step(k == 0 ? u0 : u, u, COL_DIFFUSE);
            return e;
        }
        cudaError_t e = cudaSuccess;
        if (p->fs && batch == 1 && nsteps > 0) {   // R27: the four-step passes, field W in the scratch
            void *Wf = scratch(0);
            e = fs_aa(0, u0, Wf, nullptr);
            for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
                if (fs_bb_enabled()) {
                    e = fs_bb(Wf);
                } else {
                    e = fs_bx(Wf);
                    if (e == cudaSuccess) e = fs_by(Wf);
                }
                if (e == cudaSuccess) e = k + 1 < nsteps ? fs_aa(2, Wf, Wf, u) : fs_aa(1, Wf, u, nullptr);
            }
            return e;
        }
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            e = rows_diff(k == 0 ? u0 : u, u);
            if (e == cudaSuccess) e = cols_diff_y(u, u);
        }
        return e;
    }
    // four-step passes (fourstep.cuh): AA (op 0), AA^-1 (op 1), MID (op 2: AA^-1 -> phys, AA -> out)
    cudaError_t fs_aa(int op, const void *in, void *out, void *phys)
    {
        return launch(p, FFTPDE_KERNEL_AA, [&] { return launch_aa(op, in, out, phys, p->ws + p->o_fs_tw, p->stream); });
    }
    // Bx + By fused over L2-resident 1024 x 1024 blocks (bb_kernel)
    cudaError_t fs_bb(void *Wf)
    {
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_fs_bb(Wf, p->ws + p->o_fs_tw32, (const double *)(p->ws + p->o_fs_mx),
                                (const double *)(p->ws + p->o_fs_my), p->ws + p->o_fs_sync, p->stream);
        });
    }
    // Bx: the 1024-point row segments of fixed k1 (32 per row): line class = segment % 32
    cudaError_t fs_bx(void *Wf)
    {
        OpTables<double> t{};
        t.ey2d = (const double *)(p->ws + p->o_fs_mx);
        t.ey2d_mod = 32;
        return launch(p, FFTPDE_KERNEL_ROW, [&] { return launch_fs_b(false, Wf, p->ws + p->o_fs_tw32, p->ws + p->o_fs_tw16, t, p->stream); });
    }
    // By: the 1024-row column blocks of fixed l1 (32 per column): class = block l1
    cudaError_t fs_by(void *Wf)
    {
        OpTables<double> t{};
        t.ey2d = (const double *)(p->ws + p->o_fs_my);
        return launch(p, FFTPDE_KERNEL_COL, [&] { return launch_fs_b(true, Wf, p->ws + p->o_fs_tw32, p->ws + p->o_fs_tw16, t, p->stream); });
    }
    // complex128 4096^2-class grids (C3): the spectra between the passes are stored
    // transposed (wavet.cuh), so the column pass moves whole contiguous columns
    cudaError_t wave_t(void *U, void *V, void *SU, void *SV, int64_t nsteps)
    {
        const void *twx = p->ws + p->o_twx32, *twy = p->ws + p->o_twy32;
        auto rows_t = [&](int op, void *S, const void *in, void *out) {
            return launch(p, FFTPDE_KERNEL_ROW, [&] {
                return launch_wave_t_rows(op, S, in, out, p->nx, p->ny, twx, p->stream);
            });
        };
        cudaError_t e = rows_t(WT_FWD, SU, U, nullptr);
        if (e == cudaSuccess) e = rows_t(WT_FWD, SV, V, nullptr);
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            e = launch(p, FFTPDE_KERNEL_WAVE_COL, [&] {
                return launch_wave_t_cols(SU, SV, p->nx, p->ny, twy, tables<double>(p), p->stream);
            });
            const int op = k + 1 < nsteps ? WT_MID : WT_INV;
            if (e == cudaSuccess) e = rows_t(op, SU, nullptr, U);
            if (e == cudaSuccess) e = rows_t(op, SV, nullptr, V);
        }
        return e;
    }
    cudaError_t wave(void *U, void *V, int64_t nsteps)
    {
        if (stride != p->nx * p->ny) {          // custom grid stride: in place, 5 launches per step
            cudaError_t e = cudaSuccess;
            for (int64_t s = 0; s < nsteps && e == cudaSuccess; ++s) {
                e = rows(U, U, 0);
                if (e == cudaSuccess) e = rows(V, V, 0);
                if (e == cudaSuccess) e = wave_cols(U, V);
                if (e == cudaSuccess) e = rows(U, U, 1);
                if (e == cudaSuccess) e = rows(V, V, 1);
            }
            return e;
        }
        void *SU = scratch(0), *SV = scratch(1);
        if constexpr (sizeof(T) == 8) {
            if (batch == 1 && wave_t_supported(p->nx, p->ny)) return wave_t(U, V, SU, SV, nsteps);
        }
        cudaError_t e = rows(U, SU, 0);
        if (e == cudaSuccess) e = rows(V, SV, 0);
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            e = wave_cols(SU, SV);
            if (e != cudaSuccess) break;
            if (k + 1 < nsteps) {
                e = rows_mid(SU, SU, U);
                if (e == cudaSuccess) e = rows_mid(SV, SV, V);
            } else {
                e = rows(SU, U, 1);
                if (e == cudaSuccess) e = rows(SV, V, 1);
            }
        }
        return e;
    }
    // ---- sharded plans: the slab decomposition ----------------------
    // 2D: rank r owns rows [r R, (r+1) R); after the exchange, spectral columns
    // [r BW, (r+1) BW) of all ny rows.  3D: rank r owns z-planes [r nzl, (r+1) nzl)
    // ("z-slab" [nzl][ny][nx]); after the exchange, all nz planes of rows
    // [r R, (r+1) R) ("y-slab" [nz][R][nx]).  With NCCL the plan runs its own rank
    // (grouped point-to-point send/recv = the all-to-all); in loopback mode one plan
    // runs all P ranks on one device, every phase for every rank in turn, the
    // exchange as block copies, and the caller's buffers hold the P slabs back to back.
    int nloc() const { return p->loopback ? p->P : 1; }
    int rk(int i) const { return p->loopback ? i : p->rank; }
    size_t slab_bytes() const { return (size_t)p->slab_elems * elem_cplx(p); }
    void *at(const void *base, int i) const { return (unsigned char *)base + (p->loopback ? (size_t)i * slab_bytes() : 0); }
    void *shA(int i) const { return at(p->ws + p->o_shA, i); }
    void *shB(int i) const { return at(p->ws + p->o_shB, i); }
    void *shC(int i) const { return at(p->ws + p->o_shC, i); }
    // rows (the x-pass) of one rank's slab: R rows (2D) or nzl planes of ny rows (3D)
    cudaError_t rows_sh(const void *in, void *out, int inverse)
    {
        const int64_t nrows = p->pencil ? p->nzl * p->nyl : p->is3d ? p->ny : p->R;
        const int64_t nb = p->is3d && !p->pencil ? p->nzl : 1, st = nrows * p->nx;
        return launch(p, FFTPDE_KERNEL_ROW, [&] {
            if (p->rowP)
                return launch_rows2<T>(p->nx, in, out, nullptr, nrows, st, nb, inverse ? ROW_INV : ROW_FWD, rtw(),
                                       p->stream);
            return launch_rows<T>(p->nx, in, out, nullptr, nrows, st, nb, inverse ? ROW_INV : ROW_FWD, rtw(),
                                  p->stream);
        });
    }
    // [nrows][P][blk] <-> [P][nrows][blk]: 2D rows of R x BW blocks; 3D planes of R x nx blocks
    cudaError_t pack_sh(const void *in, void *out, int direction)
    {
        ++p->launches;
        const int64_t nrows = p->is3d ? p->nzl : p->R, bw = p->is3d ? p->R * p->nx : p->BW;
        return launch_pack(in, out, nrows, p->P, bw * (int64_t)elem_cplx(p), direction, p->stream);
    }
    // 2D: the column pass of column slab r ([ny][BW], global wavenumbers r BW + c)
    cudaError_t cols_sh(const void *in, void *out, int op, int r)
    {
        OpTables<T> t = tables<T>(p);
        t.kx2 += r * p->BW;
        t.ex += r * p->BW;
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->BW, p->ny * p->BW, 1, op, ctw(), t, p->stream);
        });
    }
    // 3D: the y-pass of one z-slab (nzl planes), forward or unscaled inverse
    cudaError_t ypass_sh(const void *in, void *out, int op)
    {
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->nx, p->nx * p->ny, p->nzl, op, ctw(), tables3<false>((T)1),
                                  p->stream);
        });
    }
    // 3D: the z-pass of y-slab r: lines x + nx j (j < R) of length nz, global row r R + j
    cudaError_t zpass_sh(const void *in, void *out, int op, int r)
    {
        OpTables<T> t = tables3<true>(scale3());
        t.kx2 += r * p->R * p->nx;
        t.ex += r * p->R * p->nx;
        const ColTw ztw = this->ztw();
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->nz, in, out, p->R * p->nx, p->nz * p->R * p->nx, 1, op, ztw, t, p->stream);
        });
    }
    // the all-to-all: block q of rank r's send buffer -> block r of rank q's receive buffer
    cudaError_t exchange(void *(Passes::*send)(int) const, void *(Passes::*recv)(int) const)
    {
        const size_t blk = slab_bytes() / (size_t)p->P;
        if (p->loopback) {
            for (int r = 0; r < p->P; ++r)
                for (int q = 0; q < p->P; ++q) {
                    cudaError_t e = cudaMemcpyAsync((unsigned char *)(this->*recv)(q) + r * blk,
                                                    (const unsigned char *)(this->*send)(r) + q * blk, blk,
                                                    cudaMemcpyDeviceToDevice, p->stream);
                    if (e != cudaSuccess) return e;
                }
            return cudaSuccess;
        }
        const NcclApi &n = nccl();
        const size_t count = blk / sizeof(T);                          // complex = 2 reals
        const ncclDataType_t ty = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
        const unsigned char *sb = (const unsigned char *)(this->*send)(0);
        unsigned char *rb = (unsigned char *)(this->*recv)(0);
        // every enqueue is checked; groupEnd is still called after a failed one so the
        // group is closed, and the failure surfaces as FFTPDE_ERR_NCCL (dispatch)
        ncclResult_t first = n.groupStart();
        if (first != ncclSuccess) {
            p->nccl_failed = true;
            return cudaErrorUnknown;
        }
        for (int q = 0; q < p->P; ++q) {
            const ncclResult_t rs = n.send(sb + q * blk, count, ty, q, p->comm, p->stream);
            if (first == ncclSuccess) first = rs;
            const ncclResult_t rr = n.recv(rb + q * blk, count, ty, q, p->comm, p->stream);
            if (first == ncclSuccess) first = rr;
        }
        const ncclResult_t re = n.groupEnd();
        if (first == ncclSuccess) first = re;
        if (first != ncclSuccess) {
            p->nccl_failed = true;
            return cudaErrorUnknown;
        }
        return cudaGetLastError();
    }
    template <typename F> cudaError_t each(F &&f)
    {
        for (int i = 0; i < nloc(); ++i) {
            cudaError_t e = f(i);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    // ---- pencils (fftpde_plan_3d_pencil) ----
    int pi(int r) const { return r / p->Py; }
    int pj(int r) const { return r % p->Py; }
    cudaError_t pack_pen(const void *in, void *out, int64_t nrows, int nblocks, int64_t blk_elems, int direction)
    {
        ++p->launches;
        return launch_pack(in, out, nrows, nblocks, blk_elems * (int64_t)elem_cplx(p), direction, p->stream);
    }
    // the all-to-all inside a group: kind 0 = the Py ranks of z-block i (row group),
    // kind 1 = the Pz ranks of x-block j (column group).  Block g of rank r's send
    // buffer goes to the group's g-th rank, at the position of r within the group.
    cudaError_t exchange_pen(void *(Passes::*send)(int) const, void *(Passes::*recv)(int) const, int kind)
    {
        const int G = kind ? p->Pz : p->Py;
        const size_t blk = slab_bytes() / (size_t)G;
        auto peer = [&](int r, int g) { return kind ? g * p->Py + pj(r) : pi(r) * p->Py + g; };
        auto pos = [&](int r) { return kind ? pi(r) : pj(r); };
        if (p->loopback) {
            for (int r = 0; r < p->P; ++r)
                for (int g = 0; g < G; ++g) {
                    const int q = peer(r, g);
                    cudaError_t e = cudaMemcpyAsync((unsigned char *)(this->*recv)(q) + (size_t)pos(r) * blk,
                                                    (const unsigned char *)(this->*send)(r) + (size_t)g * blk, blk,
                                                    cudaMemcpyDeviceToDevice, p->stream);
                    if (e != cudaSuccess) return e;
                }
            return cudaSuccess;
        }
        const NcclApi &n = nccl();
        const size_t count = blk / sizeof(T);
        const ncclDataType_t ty = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
        const unsigned char *sb = (const unsigned char *)(this->*send)(0);
        unsigned char *rb = (unsigned char *)(this->*recv)(0);
        ncclResult_t first = n.groupStart();
        if (first != ncclSuccess) {
            p->nccl_failed = true;
            return cudaErrorUnknown;
        }
        for (int g = 0; g < G; ++g) {      // the group's g-th rank sends me its block at my position
            const int q = peer(p->rank, g);
            const ncclResult_t rs = n.send(sb + (size_t)g * blk, count, ty, q, p->comm, p->stream);
            if (first == ncclSuccess) first = rs;
            const ncclResult_t rr = n.recv(rb + (size_t)g * blk, count, ty, q, p->comm, p->stream);
            if (first == ncclSuccess) first = rr;
        }
        const ncclResult_t re = n.groupEnd();
        if (first == ncclSuccess) first = re;
        if (first != ncclSuccess) {
            p->nccl_failed = true;
            return cudaErrorUnknown;
        }
        return cudaGetLastError();
    }
    // x-pencil in -> z-pencils shC: x-pass, pack by x-block, row-group exchange,
    // unpack to [nzl][ny][nxl], y-pass, pack by y-block of ny/Pz, column-group exchange
    cudaError_t to_zpencils(const void *in)
    {
        const int64_t nzl = p->nzl, nyl = p->nyl, nxl = p->nxl, nyl2 = p->nyl2;
        // a group of one rank exchanges nothing: py = 1 makes the x-pencil the
        // y-pencil, pz = 1 the y-pencil the z-pencil (no pack, no copy)
        cudaError_t e = each([&](int i) { return rows_sh(at(in, i), shA(i), 0); });
        if (p->Py > 1) {
            if (e == cudaSuccess) e = each([&](int i) { return pack_pen(shA(i), shB(i), nzl * nyl, p->Py, nxl, 0); });
            if (e == cudaSuccess) e = exchange_pen(&Passes::shB, &Passes::shC, 0);
            if (e == cudaSuccess) e = each([&](int i) { return pack_pen(shC(i), shA(i), nzl, p->Py, nyl * nxl, 1); });
        }
        if (p->Pz == 1) return e == cudaSuccess ? each([&](int i) { return ypass_pen(shA(i), shC(i), COL_FWD); }) : e;
        if (e == cudaSuccess) e = each([&](int i) { return ypass_pen(shA(i), shB(i), COL_FWD); });
        if (e == cudaSuccess) e = each([&](int i) { return pack_pen(shB(i), shA(i), nzl, p->Pz, nyl2 * nxl, 0); });
        if (e == cudaSuccess) e = exchange_pen(&Passes::shA, &Passes::shC, 1);
        return e;
    }
    // z-pencils shC -> x-pencil out: the reverse, with the unscaled inverse y- and x-passes
    cudaError_t from_zpencils(void *out)
    {
        const int64_t nzl = p->nzl, nyl = p->nyl, nxl = p->nxl, nyl2 = p->nyl2;
        cudaError_t e = cudaSuccess;
        if (p->Pz > 1) {
            e = exchange_pen(&Passes::shC, &Passes::shA, 1);
            if (e == cudaSuccess) e = each([&](int i) { return pack_pen(shA(i), shB(i), nzl, p->Pz, nyl2 * nxl, 1); });
            if (e == cudaSuccess) e = each([&](int i) { return ypass_pen(shB(i), shA(i), COL_INV); });
        } else {
            e = each([&](int i) { return ypass_pen(shC(i), shA(i), COL_INV); });
        }
        if (p->Py > 1) {
            if (e == cudaSuccess) e = each([&](int i) { return pack_pen(shA(i), shB(i), nzl, p->Py, nyl * nxl, 0); });
            if (e == cudaSuccess) e = exchange_pen(&Passes::shB, &Passes::shC, 0);
            if (e == cudaSuccess) e = each([&](int i) { return pack_pen(shC(i), shA(i), nzl * nyl, p->Py, nxl, 1); });
        }
        if (e == cudaSuccess) e = each([&](int i) { return rows_sh(shA(i), at(out, i), 1); });
        return e;
    }
    // y-pass of a y-pencil [nzl][ny][nxl]: nxl columns per plane (forward or unscaled inverse)
    cudaError_t ypass_pen(const void *in, void *out, int op)
    {
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->nxl, p->ny * p->nxl, p->nzl, op, ctw(), tables3<false>((T)1),
                                  p->stream);
        });
    }
    // z-pass of z-pencil r: lines l = yl2 nxl + xl of length nz; the plan's (x, y)
    // line tables are stored in pencil order (rank-major), so rank r's lines start at r nyl2 nxl
    cudaError_t zpass_pen(const void *in, void *out, int op, int r)
    {
        OpTables<T> t = tables3<true>(scale3());
        const int64_t nl = p->nyl2 * p->nxl;
        t.kx2 += r * nl;
        t.ex += r * nl;
        const ColTw ztw = this->ztw();
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->nz, in, out, nl, p->nz * nl, 1, op, ztw, t, p->stream);
        });
    }
    // slab in -> slabs shC (2D: column slabs [ny][BW] of the x-spectrum; 3D: y-slabs [nz][R][nx] of the xy-spectrum)
    cudaError_t to_columns(const void *in)
    {
        if (p->pencil) return to_zpencils(in);
        cudaError_t e = each([&](int i) { return rows_sh(at(in, i), shA(i), 0); });
        if (p->is3d) {
            if (e == cudaSuccess) e = each([&](int i) { return ypass_sh(shA(i), shB(i), COL_FWD); });
            if (e == cudaSuccess) e = each([&](int i) { return pack_sh(shB(i), shA(i), 0); });
            if (e == cudaSuccess) e = exchange(&Passes::shA, &Passes::shC);
            return e;
        }
        if (e == cudaSuccess) e = each([&](int i) { return pack_sh(shA(i), shB(i), 0); });
        if (e == cudaSuccess) e = exchange(&Passes::shB, &Passes::shC);
        return e;
    }
    // slabs shC -> slab out (inverse x-pass, and for 3D the inverse y-pass first)
    cudaError_t from_columns(void *out)
    {
        if (p->pencil) return from_zpencils(out);
        cudaError_t e = exchange(&Passes::shC, &Passes::shB);
        if (e == cudaSuccess) e = each([&](int i) { return pack_sh(shB(i), shA(i), 1); });
        if (p->is3d) {
            if (e == cudaSuccess) e = each([&](int i) { return ypass_sh(shA(i), shB(i), COL_INV); });
            if (e == cudaSuccess) e = each([&](int i) { return rows_sh(shB(i), at(out, i), 1); });
            return e;
        }
        if (e == cudaSuccess) e = each([&](int i) { return rows_sh(shA(i), at(out, i), 1); });
        return e;
    }
    cudaError_t colpass_sh(const void *in, void *out, int op)
    {
        return each([&](int i) {
            if (p->pencil) return zpass_pen(at(in, i), at(out, i), op, rk(i));
            return p->is3d ? zpass_sh(at(in, i), at(out, i), op, rk(i)) : cols_sh(at(in, i), at(out, i), op, rk(i));
        });
    }
    // 2D diffusion step in the separable form (R26): x diffusion of the row slab,
    // exchange, y diffusion of the column slab, exchange back (one row pass per step
    // instead of a forward and an inverse one)
    cudaError_t diff_step_sh(const void *in, void *out)
    {
        cudaError_t e = each([&](int i) {
            return launch(p, FFTPDE_KERNEL_ROW, [&] {
                if (p->rowP)
                    return launch_rows2<T>(p->nx, at(in, i), shA(i), nullptr, p->R, p->R * p->nx, 1, ROW_DIFF, rtw(),
                                           p->stream, rowmul());
                return launch_rows<T>(p->nx, at(in, i), shA(i), nullptr, p->R, p->R * p->nx, 1, ROW_DIFF, rtw(),
                                      p->stream, rowmul());
            });
        });
        if (e == cudaSuccess) e = each([&](int i) { return pack_sh(shA(i), shB(i), 0); });
        if (e == cudaSuccess) e = exchange(&Passes::shB, &Passes::shC);
        if (e == cudaSuccess)
            e = each([&](int i) {
                OpTables<T> t = tables<T>(p);
                t.ex = (const T *)(p->ws + p->o_one);
                return launch(p, FFTPDE_KERNEL_COL, [&] {
                    return launch_cols<T>(p->ny, shC(i), shC(i), p->BW, p->ny * p->BW, 1, COL_DIFFUSE, ctw(), t,
                                          p->stream);
                });
            });
        if (e == cudaSuccess) e = exchange(&Passes::shC, &Passes::shB);
        if (e == cudaSuccess) e = each([&](int i) { return pack_sh(shB(i), at(out, i), 1); });
        return e;
    }
    // ---- the distributed four-step diffusion (R28; 32768^2 complex128, P | 32) ----
    // Rank r's Y-part (rows of m1 in [r M, r M + M)) and X-part (columns of n1 in
    // [r M, r M + M)) share the 5D layout [blk][Q][M][Q][M] (fourstep.cuh FsPart), so
    // the Y -> X and X -> Y transposes are the plain all-to-all `exchange` of equal
    // blocks.  Per step: the B pass of the part the field is in, the exchange, the B
    // pass of the other axis, then MID (AA^-1 of this step -> the physical field, AA
    // of the next) in that part: 3 passes and one exchange per step, the parts
    // alternating.  The caller's row slabs enter and leave through one permutation
    // pass, one all-to-all and one block transpose each way.
    cudaError_t fsd_aa(int op, int xmode, int i, const void *in, void *out, void *phys)
    {
        return launch(p, FFTPDE_KERNEL_AA, [&] {
            if (p->P == 1) return launch_aa(op, in, out, phys, p->ws + p->o_fs_tw, p->stream);   // = the plain layout
            return launch_aa_part(op, p->P, rk(i), xmode, in, out, phys, p->ws + p->o_fs_tw, p->stream);
        });
    }
    cudaError_t fsd_b(bool cols, int i, void *f)
    {
        return launch(p, cols ? FFTPDE_KERNEL_COL : FFTPDE_KERNEL_ROW, [&] {
            if (p->P == 1) {                               // both parts are the single-GPU layout
                OpTables<double> t{};
                t.ey2d = (const double *)(p->ws + (cols ? p->o_fs_my : p->o_fs_mx));
                t.ey2d_mod = 32;
                return launch_fs_b(cols, f, p->ws + p->o_fs_tw32, p->ws + p->o_fs_tw16, t, p->stream);
            }
            return launch_fs_b_part(cols, p->P, rk(i), f, p->ws + p->o_fs_tw32,
                                    (const double *)(p->ws + (cols ? p->o_fs_my : p->o_fs_mx)), p->stream);
        });
    }
    // [P][P][X] -> [P][P][X] with the two block indices swapped (X = a rank's slab / P^2)
    cudaError_t fsd_swap(const void *in, void *out)
    {
        ++p->launches;
        return launch_pack(in, out, p->P, p->P, slab_bytes() / ((size_t)p->P * p->P), 0, p->stream);
    }
    cudaError_t fsd_perm(const void *in, void *out, int direction)
    {
        ++p->launches;
        return launch_fs_perm(in, out, p->P, direction, p->stream);
    }
    cudaError_t diffuse_fsd(const void *u0, void *u, int64_t nsteps)
    {
        const bool one = p->P == 1;                        // both parts are the plain layout, no exchange
        cudaError_t e;
        if (one) {
            e = fsd_aa(0, 0, 0, u0, shA(0), nullptr);
        } else {                                           // row slab -> Y-part in shA
            e = each([&](int i) { return fsd_perm(at(u0, i), shB(i), 0); });
            if (e == cudaSuccess) e = exchange(&Passes::shB, &Passes::shC);
            if (e == cudaSuccess) e = each([&](int i) { return fsd_swap(shC(i), shA(i)); });
            if (e == cudaSuccess) e = each([&](int i) { return fsd_aa(0, 0, i, shA(i), shA(i), nullptr); });
        }
        int x = 0;                                         // the part the AA-domain field is in
        auto W = [&](int i) { return x && !one ? shC(i) : shA(i); };
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            e = each([&](int i) { return fsd_b(x != 0, i, W(i)); });
            if (e == cudaSuccess && !one) e = x ? exchange(&Passes::shC, &Passes::shA) : exchange(&Passes::shA, &Passes::shC);
            x ^= 1;
            if (e == cudaSuccess) e = each([&](int i) { return fsd_b(x != 0, i, W(i)); });
            if (e != cudaSuccess) break;
            if (k + 1 < nsteps) e = each([&](int i) { return fsd_aa(2, x, i, W(i), W(i), one ? at(u, i) : shB(i)); });
            else e = each([&](int i) { return fsd_aa(1, x, i, W(i), one ? at(u, i) : shB(i), nullptr); });
        }
        if (e != cudaSuccess || one) return e;
        // the physical field (shB, part x) -> Y-part -> the caller's row slabs
        if (x) {
            e = exchange(&Passes::shB, &Passes::shA);
            if (e == cudaSuccess) e = each([&](int i) { return fsd_swap(shA(i), shB(i)); });
        } else {
            e = each([&](int i) { return fsd_swap(shB(i), shA(i)); });
        }
        if (e == cudaSuccess) e = x ? exchange(&Passes::shB, &Passes::shC) : exchange(&Passes::shA, &Passes::shC);
        if (e == cudaSuccess) e = each([&](int i) { return fsd_perm(shC(i), at(u, i), 1); });
        return e;
    }
    // one step: slab -> exchange -> column-slab pass with the operator -> exchange -> slab
    cudaError_t step_sh(const void *in, void *out, int op)
    {
        if (op == COL_DIFFUSE && !p->is3d) return diff_step_sh(in, out);
        cudaError_t e = to_columns(in);
        if (e == cudaSuccess) e = colpass_sh(shC(0), shC(0), op);
        if (e == cudaSuccess) e = from_columns(out);
        return e;
    }
    cudaError_t forward_sh(const void *in, void *out)
    {
        cudaError_t e = to_columns(in);
        if (e == cudaSuccess) e = colpass_sh(shC(0), out, COL_FWD);     // out of place (two-level pass)
        return e;
    }
    cudaError_t inverse_sh(const void *in, void *out)
    {
        cudaError_t e = colpass_sh(in, shC(0), COL_INV);
        if (e == cudaSuccess) e = from_columns(out);
        return e;
    }
    // ---- real plans (fftpde_plan_2d_r2c): half spectrum of pitch p->pitch -----------
    int64_t hstride() const { return p->ny * p->pitch; }
    void *hscr(int i) const { return p->ws + p->o_scr + (size_t)i * (size_t)(batch * hstride()) * elem_cplx(p); }
    cudaError_t rc(const void *in, void *out, void *out2, int op)
    {
        return launch(p, FFTPDE_KERNEL_ROW, [&] {
            return launch_rc_rows<T>(p->nx, in, out, out2, p->ny * batch, p->pitch, op, p->ws + p->o_twm,
                                     p->ws + p->o_twr, p->stream);
        });
    }
    cudaError_t colsr(const void *in, void *out, int op)
    {
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->pitch, hstride(), batch, op, ctw(), tables<T>(p), p->stream);
        });
    }
    cudaError_t wave_colsr(void *U, void *V)
    {
        return launch(p, FFTPDE_KERNEL_WAVE_COL, [&] {
            return launch_wave_cols<T>(p->ny, U, V, p->pitch, hstride(), batch, ctw(), tables<T>(p), p->stream);
        });
    }
    cudaError_t copy_half(const void *src, size_t spitch, void *dst, size_t dpitch)
    {
        const size_t ec = elem_cplx(p);
        return cudaMemcpy2DAsync(dst, dpitch * ec, src, spitch * ec, (size_t)(p->nx / 2 + 1) * ec,
                                 (size_t)(p->ny * batch), cudaMemcpyDeviceToDevice, p->stream);
    }
    // real -> compact half spectrum [batch][ny][nx/2 + 1]
    cudaError_t forward_real(const void *in, void *out)
    {
        void *S = hscr(0), *Tm = p->colP ? hscr(1) : hscr(0);      // two-level FWD is out of place
        cudaError_t e = rc(in, S, nullptr, RC_FWD);
        if (e == cudaSuccess) e = colsr(S, Tm, COL_FWD);
        if (e == cudaSuccess) e = copy_half(Tm, p->pitch, out, p->nx / 2 + 1);
        return e;
    }
    cudaError_t inverse_real(const void *in, void *out)
    {
        void *S = hscr(0), *Tm = p->colP ? hscr(1) : hscr(0);
        cudaError_t e = copy_half(in, p->nx / 2 + 1, S, p->pitch);
        if (e == cudaSuccess) e = colsr(S, Tm, COL_INV);
        if (e == cudaSuccess) e = rc(Tm, out, nullptr, RC_INV);
        return e;
    }
    cudaError_t poisson_real(const void *in, void *out)
    {
        void *S = hscr(0);
        cudaError_t e = rc(in, S, nullptr, RC_FWD);
        if (e == cudaSuccess) e = colsr(S, S, COL_POISSON);
        if (e == cudaSuccess) e = rc(S, out, nullptr, RC_INV);
        return e;
    }
    // separable diffusion of real fields (R26): per step the x diffusion of every
    // real row (half-spectrum round trip inside the row pass, RC_DIFF) and the y
    // diffusion of every column, done on the real field viewed as nx/2 complex
    // columns (pairs of real columns: the y operator is real, so it acts on the
    // pair's real and imaginary parts independently); in place, u materialised
    cudaError_t diffuse_real(const void *u0, void *u, int64_t nsteps)
    {
        OpTables<T> ty = tables<T>(p);
        ty.ex = (const T *)(p->ws + p->o_one);
        cudaError_t e = cudaSuccess;
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            const void *src = k == 0 ? u0 : u;
            e = launch(p, FFTPDE_KERNEL_ROW, [&] {
                return launch_rc_rows<T>(p->nx, src, u, nullptr, p->ny * batch, p->pitch, RC_DIFF, p->ws + p->o_twm,
                                         p->ws + p->o_twr, p->stream, p->ws + p->o_ex);
            });
            if (e == cudaSuccess)
                e = launch(p, FFTPDE_KERNEL_COL, [&] {
                    return launch_cols<T>(p->ny, u, u, p->nx / 2, p->ny * (p->nx / 2), batch, COL_DIFFUSE, ctw(), ty,
                                          p->stream);
                });
        }
        return e;
    }
    cudaError_t wave_real(void *U, void *V, int64_t nsteps)
    {
        void *SU = hscr(0), *SV = hscr(1);
        cudaError_t e = rc(U, SU, nullptr, RC_FWD);
        if (e == cudaSuccess) e = rc(V, SV, nullptr, RC_FWD);
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            e = wave_colsr(SU, SV);
            if (e != cudaSuccess) break;
            if (k + 1 < nsteps) {
                e = rc(SU, SU, U, RC_MID);
                if (e == cudaSuccess) e = rc(SV, SV, V, RC_MID);
            } else {
                e = rc(SU, U, nullptr, RC_INV);
                if (e == cudaSuccess) e = rc(SV, V, nullptr, RC_INV);
            }
        }
        return e;
    }
    // ---- 3D (fftpde_plan_3d): this Passes runs with batch = nz, stride = nx ny ----
    template <bool ZOP> OpTables<T> tables3(T scale) const
    {
        OpTables<T> t = tables<T>(p);
        if (ZOP) {            // z-pass: line index = x + nx y, element index = z
            t.kx2 = (const T *)(p->ws + p->o_kxy2);
            t.ky2 = (const T *)(p->ws + p->o_kz2);
            t.ex = (const T *)(p->ws + p->o_exy);
            t.ey = (const T *)(p->ws + p->o_ez);
        }
        t.scale = scale;
        return t;
    }
    T scale3() const { return (T)(1.0 / ((double)p->nx * (double)p->ny * (double)p->nz)); }
    cudaError_t ypass(const void *in, void *out, int op)
    {
        // forward, or the inverse left unscaled (1/(nx ny nz) is applied in the z-pass)
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, p->nx, stride, batch, op, ctw(), tables3<false>((T)1), p->stream);
        });
    }
    cudaError_t zpass(const void *in, void *out, int op)
    {
        const ColTw ztw = this->ztw();
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->nz, in, out, p->nx * p->ny, p->nx * p->ny * p->nz, 1, op, ztw,
                                  tables3<true>(scale3()), p->stream);
        });
    }
    // The two-level y-pass's plain forward / inverse are out of place (col2.cuh),
    // so with p->colP they go through the scratch; the operator passes are in place.
    cudaError_t forward3(const void *in, void *out)
    {
        if (p->zP) {                        // the two-level z-pass transforms out of place
            cudaError_t e = rows(in, scratch(0), 0);
            if (e == cudaSuccess) e = ypass(scratch(0), scratch(1), COL_FWD);
            if (e == cudaSuccess) e = zpass(scratch(1), out, COL_FWD);
            return e;
        }
        void *A = p->colP ? scratch(0) : out;
        cudaError_t e = rows(in, A, 0);
        if (e == cudaSuccess) e = ypass(A, out, COL_FWD);
        if (e == cudaSuccess) e = zpass(out, out, COL_FWD);
        return e;
    }
    cudaError_t inverse3(const void *in, void *out)
    {
        if (p->zP) {
            cudaError_t e = zpass(in, scratch(0), COL_INV);
            if (e == cudaSuccess) e = ypass(scratch(0), scratch(1), COL_INV);
            if (e == cudaSuccess) e = rows(scratch(1), out, 1);
            return e;
        }
        void *B = p->colP ? scratch(0) : out;
        cudaError_t e = zpass(in, out, COL_INV);
        if (e == cudaSuccess) e = ypass(out, B, COL_INV);
        if (e == cudaSuccess) e = rows(B, out, 1);
        return e;
    }
    cudaError_t poisson3(const void *in, void *out)
    {
        void *Y = p->colP ? scratch(0) : out;
        cudaError_t e = rows(in, Y, 0);
        if (e == cudaSuccess) e = ypass(Y, out, COL_FWD);
        if (e == cudaSuccess) e = zpass(out, out, COL_POISSON);
        if (e == cudaSuccess) e = ypass(out, Y, COL_INV);
        if (e == cudaSuccess) e = rows(Y, out, 1);
        return e;
    }
    // nsteps exact diffusion steps in the separable form (R26): per step the 1D
    // diffusion along x (rows), y (y-pass) and z (z-pass), in place on u, one read
    // and one write each; u is materialised after every step
    cudaError_t diffuse3(const void *u0, void *u, int64_t nsteps)
    {
        OpTables<T> ty = tables3<false>((T)1);
        ty.ex = (const T *)(p->ws + p->o_one);
        ty.ey = (const T *)(p->ws + p->o_ey);
        OpTables<T> tz = tables3<true>((T)1);
        tz.ex = (const T *)(p->ws + p->o_zscale);
        tz.ey = (const T *)(p->ws + p->o_ez);
        const ColTw ztw = this->ztw();
        cudaError_t e = cudaSuccess;
        for (int64_t k = 0; k < nsteps && e == cudaSuccess; ++k) {
            e = rows_diff(k == 0 ? u0 : u, u);
            if (e == cudaSuccess)
                e = launch(p, FFTPDE_KERNEL_COL, [&] {
                    return launch_cols<T>(p->ny, u, u, p->nx, stride, batch, COL_DIFFUSE, ctw(), ty, p->stream);
                });
            if (e == cudaSuccess)
                e = launch(p, FFTPDE_KERNEL_COL, [&] {
                    return launch_cols<T>(p->nz, u, u, p->nx * p->ny, p->nx * p->ny * p->nz, 1, COL_DIFFUSE, ztw, tz,
                                          p->stream);
                });
        }
        return e;
    }
    cudaError_t kop(void *X, const void *S, int op, double D, double dt)
    {
        return launch(p, FFTPDE_KERNEL_POINTWISE, [&] {
            return launch_kop<T>(X, S, p->nx, p->ny, batch, stride, op, p->ws + p->o_kx, p->ws + p->o_ky,
                                 p->ws + p->o_kx2, p->ws + p->o_ky2, D, dt, p->stream);
        });
    }
    // out = iDFT2(m .* DFT2(in)), m a diagonal operator (kspace.cu)
    cudaError_t apply(const void *in, void *out, int op)
    {
        cudaError_t e = forward(in, out);
        if (e == cudaSuccess) e = kop(out, nullptr, op, 0.0, 0.0);
        if (e == cudaSuccess) e = inverse(out, out);
        return e;
    }
    // exact steps of u_t = D nabla^2 u + s (static s): s^ once, then per step
    // forward u, u^ <- E u^ + Phi s^, inverse (materialising u)
    cudaError_t diffuse_source(const void *u0, const void *src, void *u, double D, double dt, int64_t nsteps,
                               void *scratch)
    {
        const size_t fb = (size_t)(batch * stride) * elem_cplx(p);
        void *Sh = scratch, *Uh = (unsigned char *)scratch + fb;
        cudaError_t e = forward(src, Sh);
        for (int64_t n = 0; n < nsteps && e == cudaSuccess; ++n) {
            e = forward(n == 0 ? u0 : u, Uh);
            if (e == cudaSuccess) e = kop(Uh, Sh, KOP_DIFFSRC, D, dt);
            if (e == cudaSuccess) e = inverse(Uh, u);
        }
        return e;
    }
    // RK4 with the orbiting source (rk4.cu): state (u^, v^) and three source
    // spectra in the caller's scratch; the source transform reuses forward().
    cudaError_t wave_rk4(void *u, void *ut, double c, const SrcParams &base, double A, double Omega, double gamma,
                         double rs, double t0, double dt, int64_t nsteps, void *means, void *scratch)
    {
        const size_t fb = (size_t)(p->nx * p->ny) * elem_cplx(p);
        unsigned char *sc = (unsigned char *)scratch;
        void *Uh = sc, *Vh = sc + fb, *S[3] = {sc + 2 * fb, sc + 3 * fb, sc + 4 * fb};
        auto source_spectrum = [&](double t, void *dst) {
            SrcParams q = base;
            q.x0 = rs * std::cos(Omega * t);
            q.y0 = rs * std::sin(Omega * t);
            q.amp = A * std::cos(gamma * t);
            cudaError_t e = launch(p, FFTPDE_KERNEL_POINTWISE,
                                   [&] { return launch_source<T>(dst, p->nx, p->ny, q, p->stream); });
            return e == cudaSuccess ? forward(dst, dst) : e;
        };
        cudaError_t e = forward(u, Uh);
        if (e == cudaSuccess) e = forward(ut, Vh);
        if (e == cudaSuccess && means) { ++p->launches; e = launch_mean<T>(Uh, means, p->nx, p->ny, p->stream); }
        if (e == cudaSuccess) e = source_spectrum(t0, S[0]);
        int i0 = 0, ih = 1, i1 = 2;
        for (int64_t n = 0; n < nsteps && e == cudaSuccess; ++n) {
            const double t = t0 + (double)n * dt;
            e = source_spectrum(t + 0.5 * dt, S[ih]);
            if (e == cudaSuccess) e = source_spectrum(t + dt, S[i1]);
            if (e != cudaSuccess) break;
            void *mo = means ? (unsigned char *)means + (size_t)(n + 1) * elem_cplx(p) : nullptr;
            e = launch(p, FFTPDE_KERNEL_POINTWISE, [&] {
                return launch_rk4<T>(Uh, Vh, S[i0], S[ih], S[i1], p->nx, p->ny, p->ws + p->o_kx2, p->ws + p->o_ky2,
                                     c, dt, mo, p->stream);
            });
            std::swap(i0, i1);                      // s^(t + dt) is the next step's s^(t)
        }
        if (e == cudaSuccess) e = inverse(Uh, u);
        if (e == cudaSuccess) e = inverse(Vh, ut);
        return e;
    }
};

template <typename F> fftpde_status dispatch(fftpde_plan p, int64_t batch, int64_t stride, F &&f)
{
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    cudaError_t e;
    p->nccl_failed = false;
    if (p->dtype == FFTPDE_C128) {
        Passes<double> ps{p, batch, stride};
        e = f(ps);
    } else {
        Passes<float> ps{p, batch, stride};
        e = f(ps);
    }
    if (p->nccl_failed) return FFTPDE_ERR_NCCL;
    return cuda_status(e);
}

// Run a multi-launch sequence through a cached CUDA graph.  The sequence is
// captured once per (kind, buffers, batch, stride, nsteps) on a private stream
// (the caller's stream may be the legacy default stream, which cannot be
// captured) and replayed on the plan's stream; the kernels read their operator
// tables by pointer, so new (D, dt) / (c, dt) need no re-capture.
// Accumulate the kernel times of one replay of a profiling graph.
fftpde_status collect_graph_profile(fftpde_plan p, const fftpde_plan_s::Graph &gr)
{
    if (gr.prof.empty()) return FFTPDE_OK;
    if (cudaStreamSynchronize(p->stream) != cudaSuccess) return FFTPDE_ERR_CUDA;
    for (auto &ev : gr.prof) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev.second.first, ev.second.second) != cudaSuccess) return FFTPDE_ERR_CUDA;
        p->prof_ms[ev.first] += ms;
        p->prof_n[ev.first] += 1;
    }
    return FFTPDE_OK;
}

// Run a multi-launch sequence through a cached CUDA graph.  The sequence is
// captured once per (kind, buffers, batch, stride, nsteps) on a private stream
// (the caller's stream may be the legacy default stream, which cannot be
// captured) and replayed on the plan's stream; the kernels read their operator
// tables by pointer, so new (D, dt) / (c, dt) need no re-capture.  With
// profiling on, a separate graph is captured whose kernel nodes are bracketed
// by event-record nodes, so per-kernel times are those of graph execution
// (a stream launch costs ~4 us on B200, a graph kernel node ~0.6 us).
template <typename F>
fftpde_status run_graphed(fftpde_plan p, std::array<uint64_t, 6> key, F &&enqueue)
{
    if (!p->use_graphs) return enqueue();
    if (p->profiling) key[0] |= 0x100;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    for (auto &gr : p->graphs) {
        if (gr.key == key) {
            p->launches += gr.launches;
            if (cudaGraphLaunch(gr.exec, p->stream) != cudaSuccess) return FFTPDE_ERR_CUDA;
            return collect_graph_profile(p, gr);
        }
    }
    if (!p->cap_stream && cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
        return FFTPDE_ERR_CUDA;
    cudaStream_t user = p->stream;
    const int64_t l0 = p->launches;
    if (cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeRelaxed) != cudaSuccess)
        return FFTPDE_ERR_CUDA;
    p->stream = p->cap_stream;
    p->capturing = true;
    p->cap_prof.clear();
    fftpde_status st = enqueue();
    p->capturing = false;
    p->stream = user;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(p->cap_stream, &graph);
    const int64_t n = p->launches - l0;
    p->launches = l0;
    if (st != FFTPDE_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return st != FFTPDE_OK ? st : FFTPDE_ERR_CUDA;
    }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return FFTPDE_ERR_CUDA;
    if (p->graphs.size() >= 8) {
        for (auto &ev : p->graphs.front().prof) { p->event_pool.push_back(ev.second.first); p->event_pool.push_back(ev.second.second); }
        cudaGraphExecDestroy(p->graphs.front().exec);
        p->graphs.erase(p->graphs.begin());
    }
    p->graphs.push_back({key, exec, n, std::move(p->cap_prof)});
    p->cap_prof.clear();
    p->launches += n;
    if (cudaGraphLaunch(exec, p->stream) != cudaSuccess) return FFTPDE_ERR_CUDA;
    return collect_graph_profile(p, p->graphs.back());
}

fftpde_status ensure_diffusion_tables(fftpde_plan p, double D, double dt)
{
    if (p->diff_valid && p->diff_D == D && p->diff_dt == dt) return FFTPDE_OK;
    const double scale = 1.0 / ((double)p->nx * (double)p->ny);
    std::vector<double> ex((size_t)p->nx), ey((size_t)p->ny);
    for (int64_t a = 0; a < p->nx; ++a) ex[(size_t)a] = std::exp(-D * p->kx2[(size_t)a] * dt) * scale;
    for (int64_t b = 0; b < p->ny; ++b) ey[(size_t)b] = std::exp(-D * p->ky2[(size_t)b] * dt);
    fftpde_status s = upload(p, p->o_ex, ex);
    if (s == FFTPDE_OK) s = upload(p, p->o_ey, ey);
    if (s == FFTPDE_OK && (p->fs || p->fsd)) {   // per-axis factors: e^{-D kx^2 dt}/nx, e^{-D ky^2 dt}/ny
        std::vector<double> mx((size_t)p->nx), my((size_t)p->ny);
        for (int64_t a = 0; a < p->nx; ++a) mx[(size_t)a] = std::exp(-D * p->kx2[(size_t)a] * dt) / (double)p->nx;
        for (int64_t b = 0; b < p->ny; ++b) my[(size_t)b] = std::exp(-D * p->ky2[(size_t)b] * dt) / (double)p->ny;
        s = upload(p, p->o_fs_mx, fourstep_mul_order(mx));
        if (s == FFTPDE_OK) s = upload(p, p->o_fs_my, fourstep_mul_order(my));
    }
    if (s != FFTPDE_OK) return s;
    p->diff_valid = true;
    p->diff_D = D;
    p->diff_dt = dt;
    return FFTPDE_OK;
}

fftpde_status ensure_wave_tables(fftpde_plan p, double c, double dt)
{
    if (p->wave_valid && p->wave_c == c && p->wave_dt == dt) return FFTPDE_OK;
    const double scale = 1.0 / ((double)p->nx * (double)p->ny);
    const size_t n = (size_t)(p->qx * p->qy);
    std::vector<double> C(n), S1(n), S2(n);
    for (int64_t qa = 0; qa < p->qx; ++qa) {
        for (int64_t qb = 0; qb < p->qy; ++qb) {
            const size_t i = (size_t)(qa * p->qy + qb);
            const double k2 = p->kx2[(size_t)qa] + p->ky2[(size_t)qb];
            const double kappa = c * std::sqrt(k2);
            if (kappa == 0.0) {            // eq:OmegaZero: u <- u + dt v, v unchanged
                C[i] = scale;
                S1[i] = dt * scale;
                S2[i] = 0.0;
            } else {                       // eq:OmegaNonZero and its time derivative
                const double sn = std::sin(kappa * dt);
                C[i] = std::cos(kappa * dt) * scale;
                S1[i] = (sn / kappa) * scale;
                S2[i] = (-kappa * sn) * scale;
            }
        }
    }
    fftpde_status s = upload(p, p->o_wc, C);
    if (s == FFTPDE_OK) s = upload(p, p->o_ws1, S1);
    if (s == FFTPDE_OK) s = upload(p, p->o_ws2, S2);
    if (s != FFTPDE_OK) return s;
    p->wave_valid = true;
    p->wave_c = c;
    p->wave_dt = dt;
    return FFTPDE_OK;
}

fftpde_status copy_grids(fftpde_plan p, const void *src, void *dst, int64_t batch, int64_t stride)
{
    if (src == dst) return FFTPDE_OK;
    DeviceGuard g(p->device);
    const size_t ec = elem_cplx(p);
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)stride * ec, src, (size_t)stride * ec,
                                      (size_t)(p->nx * p->ny) * ec, (size_t)batch,
                                      cudaMemcpyDeviceToDevice, p->stream);
    return cuda_status(e);
}

} // namespace

// Two-level column pass split ny = P Q (col2.cuh); 0 when the single-level
// pass is used (short columns, or fewer columns than one 128-byte block).
void fftpde::col2_split(int64_t ny, int64_t nx, int elem_bytes, int64_t &P, int64_t &Q)
{
    P = Q = 0;
    const int64_t W = 128 / elem_bytes;
    if (nx < W || nx % W) return;
    switch (ny) {
    case 2048: P = 32; Q = 64; break;
    case 4096: P = 64; Q = 64; break;
    case 8192: P = 64; Q = 128; break;
    case 16384: P = 128; Q = 128; break;
    case 32768: P = 128; Q = 256; break;
    default: break;
    }
}

void fftpde::row2_split(int64_t nx, int64_t &P, int64_t &Q)
{
    P = Q = 0;
    if (nx == 16384) { P = 128; Q = 128; }
    if (nx == 32768) { P = 128; Q = 256; }
}

// ============================================================================
extern "C" {

const char *fftpde_status_string(fftpde_status s)
{
    switch (s) {
    case FFTPDE_OK: return "ok";
    case FFTPDE_ERR_INVALID_ARG: return "invalid argument";
    case FFTPDE_ERR_EMPTY: return "empty input (zero-sized axis or batch)";
    case FFTPDE_ERR_NOT_POW2_X: return "nx is not a power of two (radix-2 restriction)";
    case FFTPDE_ERR_NOT_POW2_Y: return "ny is not a power of two (radix-2 restriction)";
    case FFTPDE_ERR_UNSUPPORTED: return "unsupported size for this build";
    case FFTPDE_ERR_WORKSPACE: return "workspace missing or too small";
    case FFTPDE_ERR_CUDA: return "CUDA error";
    case FFTPDE_ERR_NCCL: return "NCCL error";
    case FFTPDE_ERR_NOT_POW2_Z: return "nz is not a power of two (radix-2 restriction)";
    }
    return "unknown status";
}

fftpde_status fftpde_plan_2d(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t batch,
                             fftpde_dtype dtype, double Lx, double Ly, int device)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    *plan = nullptr;
    if (dtype != FFTPDE_C64 && dtype != FFTPDE_C128) return FFTPDE_ERR_INVALID_ARG;
    if (nx == 0 || ny == 0 || batch == 0) return FFTPDE_ERR_EMPTY;
    if (nx < 0 || ny < 0 || batch < 0) return FFTPDE_ERR_INVALID_ARG;
    if (!is_pow2(nx)) return FFTPDE_ERR_NOT_POW2_X;
    if (!is_pow2(ny)) return FFTPDE_ERR_NOT_POW2_Y;
    if (nx > kMaxLen2 || ny > kMaxLen2 || batch > 65535) return FFTPDE_ERR_UNSUPPORTED;
    if (ny > kMaxLen) {   // long columns need the two-level pass: whole 128-byte column blocks
        int64_t P, Q;
        fftpde::col2_split(ny, nx, dtype == FFTPDE_C128 ? 16 : 8, P, Q);
        if (!P) return FFTPDE_ERR_UNSUPPORTED;
    }
    if (!std::isfinite(Lx) || !std::isfinite(Ly) || !(Lx > 0) || !(Ly > 0)) return FFTPDE_ERR_INVALID_ARG;
    if (device < 0) return FFTPDE_ERR_INVALID_ARG;

    fftpde_plan p = new (std::nothrow) fftpde_plan_s;
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    p->nx = nx; p->ny = ny; p->batch = batch; p->dtype = dtype;
    p->Lx = Lx; p->Ly = Ly; p->device = device;
    p->qx = nx / 2 + 1;
    p->qy = ny / 2 + 1;
    p->use_graphs = std::getenv("FFTPDE_NO_GRAPHS") == nullptr;
    build_twiddles(nx, p->twx);
    build_twiddles(ny, p->twy);
    build_twiddles(nx, p->twx8, 8);
    build_twiddles(ny, p->twy8, 8);
    build_twiddles(nx, p->twx32, 32);
    build_twiddles(ny, p->twy32, 32);
    build_k2(nx, Lx, p->kx2);
    build_k2(ny, Ly, p->ky2);
    build_k(nx, Lx, p->kx);
    build_k(ny, Ly, p->ky);
    fftpde::col2_split(ny, nx, dtype == FFTPDE_C128 ? 16 : 8, p->colP, p->colQ);
    if (p->colP) {
        build_twiddles(p->colP, p->twP, FFTPDE_COL2_EMAX);
        build_twiddles(p->colQ, p->twQ, FFTPDE_COL2_EMAX);
        build_plain_twiddles(ny, p->twN);
    }
    p->fs = fftpde::fourstep_supported(nx, ny, batch, dtype == FFTPDE_C128 ? 16 : 8) &&
            std::getenv("FFTPDE_NO_FOURSTEP") == nullptr;
    if (p->fs) build_fourstep_tables(nx, p->fs_tw, p->fs_tw32, p->fs_tw16);
    fftpde::row2_split(nx, p->rowP, p->rowQ);
    if (p->rowP) {
        build_twiddles(p->rowP, p->rtwP, FFTPDE_R2D_E);
        build_twiddles(p->rowQ, p->rtwQ, FFTPDE_R2D_E);
        build_split_twiddles(nx, p->rowP, p->rowQ, p->rtwN);
    }

    const size_t er = elem_real(p), ec = elem_cplx(p);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
    p->o_twx = take(p->twx.size() / 2 * ec);
    p->o_twy = take(p->twy.size() / 2 * ec);
    p->o_twx8 = take(p->twx8.size() / 2 * ec);
    p->o_twy8 = take(p->twy8.size() / 2 * ec);
    p->o_twx32 = take(p->twx32.size() / 2 * ec);
    p->o_twy32 = take(p->twy32.size() / 2 * ec);
    p->o_one = take((size_t)std::max(nx, ny) * er);
    p->o_kx2 = take((size_t)nx * er);
    p->o_ky2 = take((size_t)ny * er);
    p->o_kx = take((size_t)nx * er);
    p->o_ky = take((size_t)ny * er);
    p->o_ex = take((size_t)nx * er);
    p->o_ey = take((size_t)ny * er);
    const size_t q = (size_t)(p->qx * p->qy) * er;
    p->o_wc = take(q);
    p->o_ws1 = take(q);
    p->o_ws2 = take(q);
    if (p->rowP) {
        p->o_rtwP = take(p->rtwP.size() / 2 * ec);
        p->o_rtwQ = take(p->rtwQ.size() / 2 * ec);
        p->o_rtwN = take(p->rtwN.size() / 2 * ec);
    }
    if (p->colP) {
        p->o_twP = take(p->twP.size() / 2 * ec);
        p->o_twQ = take(p->twQ.size() / 2 * ec);
        p->o_twN = take(p->twN.size() / 2 * ec);
    }
    if (p->fs) {
        p->o_fs_tw = take(p->fs_tw.size() / 2 * ec);
        p->o_fs_tw32 = take(p->fs_tw32.size() / 2 * ec);
        p->o_fs_tw16 = take(p->fs_tw16.size() / 2 * ec);
        p->o_fs_mx = take((size_t)nx * er);
        p->o_fs_my = take((size_t)ny * er);
        p->o_fs_sync = take(1024);                     // team barrier counters of the fused B pass
    }
    p->o_scr = take(2 * (size_t)(batch * nx * ny) * ec);    // last: sharded plans replace it by slabs
    p->need = off;
    *plan = p;
    return FFTPDE_OK;
}

size_t fftpde_workspace_size(fftpde_plan plan) { return plan ? plan->need : 0; }

fftpde_status fftpde_set_stream(fftpde_plan plan, void *cuda_stream)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    plan->stream = (cudaStream_t)cuda_stream;
    return FFTPDE_OK;
}

fftpde_status fftpde_set_workspace(fftpde_plan plan, void *dev_ptr, size_t bytes)
{
    if (!plan || !dev_ptr) return FFTPDE_ERR_INVALID_ARG;
    if (((uintptr_t)dev_ptr & 255u) != 0) return FFTPDE_ERR_INVALID_ARG;
    if (bytes < plan->need) return FFTPDE_ERR_WORKSPACE;
    DeviceGuard g(plan->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    plan->ws = (unsigned char *)dev_ptr;
    plan->ws_bytes = bytes;
    plan->diff_valid = plan->wave_valid = false;
    fftpde_status s;
    cudaError_t e;
    if (plan->dtype == FFTPDE_C128) {
        e = cudaMemcpyAsync(plan->ws + plan->o_twx, plan->twx.data(), plan->twx.size() * 8,
                            cudaMemcpyHostToDevice, plan->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(plan->ws + plan->o_twy, plan->twy.data(), plan->twy.size() * 8,
                                cudaMemcpyHostToDevice, plan->stream);
        s = cuda_status(e);
    } else {
        s = upload(plan, plan->o_twx, plan->twx);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_twy, plan->twy);
    }
    if (s == FFTPDE_OK) s = upload(plan, plan->o_twx8, plan->twx8);
    if (s == FFTPDE_OK) s = upload(plan, plan->o_twy8, plan->twy8);
    if (s == FFTPDE_OK) s = upload(plan, plan->o_twx32, plan->twx32);
    if (s == FFTPDE_OK) s = upload(plan, plan->o_twy32, plan->twy32);
    if (s == FFTPDE_OK && plan->rowP) {
        s = upload(plan, plan->o_rtwP, plan->rtwP);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_rtwQ, plan->rtwQ);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_rtwN, plan->rtwN);
    }
    if (s == FFTPDE_OK && (plan->fs || plan->fsd)) {
        s = upload(plan, plan->o_fs_tw, plan->fs_tw);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_fs_tw32, plan->fs_tw32);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_fs_tw16, plan->fs_tw16);
    }
    if (s == FFTPDE_OK && plan->colP) {
        s = upload(plan, plan->o_twP, plan->twP);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_twQ, plan->twQ);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_twN, plan->twN);
    }
    if (s == FFTPDE_OK) s = upload(plan, plan->o_one, std::vector<double>((size_t)std::max(plan->nx, plan->ny), 1.0));
    if (s == FFTPDE_OK) s = upload(plan, plan->o_kx2, plan->kx2);
    if (s == FFTPDE_OK) s = upload(plan, plan->o_ky2, plan->ky2);
    if (s == FFTPDE_OK) s = upload(plan, plan->o_kx, plan->kx);
    if (s == FFTPDE_OK) s = upload(plan, plan->o_ky, plan->ky);
    if (s == FFTPDE_OK && plan->is_real) {
        s = upload(plan, plan->o_twm, plan->twm);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_twr, plan->twr);
    }
    if (s == FFTPDE_OK && plan->is3d) {
        plan->diff3_valid = false;
        s = upload(plan, plan->o_twz, plan->twz);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_twz8, plan->twz8);
        if (s == FFTPDE_OK && plan->zP) {
            s = upload(plan, plan->o_twPz, plan->twPz);
            if (s == FFTPDE_OK) s = upload(plan, plan->o_twQz, plan->twQz);
            if (s == FFTPDE_OK) s = upload(plan, plan->o_twNz, plan->twNz);
        }
        if (s == FFTPDE_OK) s = upload(plan, plan->o_kz2, plan->kz2);
        if (s == FFTPDE_OK) s = upload(plan, plan->o_kxy2, plan->kxy2);
    }
    if (s != FFTPDE_OK) plan->ws = nullptr;
    return s;
}

fftpde_status fftpde_destroy(fftpde_plan plan)
{
    if (!plan) return FFTPDE_OK;
    for (auto &v : plan->pending)
        for (auto &pr : v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (cudaEvent_t e : plan->event_pool) cudaEventDestroy(e);
    for (auto &gr : plan->graphs) {
        cudaGraphExecDestroy(gr.exec);
        for (auto &ev : gr.prof) { cudaEventDestroy(ev.second.first); cudaEventDestroy(ev.second.second); }
    }
    if (plan->cap_stream) cudaStreamDestroy(plan->cap_stream);
    if (plan->comm && nccl().ok) nccl().commDestroy(plan->comm);
    delete plan;
    return FFTPDE_OK;
}

fftpde_status fftpde_set_profiling(fftpde_plan plan, int enable)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    plan->profiling = enable != 0;
    return FFTPDE_OK;
}

fftpde_status fftpde_read_profile(fftpde_plan plan, int kernel_class, double *total_ms, int64_t *launches)
{
    if (!plan || kernel_class < 0 || kernel_class >= FFTPDE_KERNEL_CLASSES || !total_ms || !launches)
        return FFTPDE_ERR_INVALID_ARG;
    DeviceGuard g(plan->device);
    auto &v = plan->pending[kernel_class];
    for (auto &pr : v) {
        if (cudaEventSynchronize(pr.second) != cudaSuccess) return FFTPDE_ERR_CUDA;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) != cudaSuccess) return FFTPDE_ERR_CUDA;
        plan->prof_ms[kernel_class] += ms;
        plan->prof_n[kernel_class] += 1;
        plan->event_pool.push_back(pr.first);
        plan->event_pool.push_back(pr.second);
    }
    v.clear();
    *total_ms = plan->prof_ms[kernel_class];
    *launches = plan->prof_n[kernel_class];
    plan->prof_ms[kernel_class] = 0;
    plan->prof_n[kernel_class] = 0;
    return FFTPDE_OK;
}

int64_t fftpde_launch_count(fftpde_plan plan) { return plan ? plan->launches : 0; }

// ---- batched entry points ----------------------------------------------------
fftpde_status fftpde_forward_batched(fftpde_plan p, const void *in, void *out, int64_t batch,
                                     int64_t stride)
{
    fftpde_status s = check_call(p, batch, stride);
    if (s == FFTPDE_OK && p->colP && stride != p->nx * p->ny) s = FFTPDE_ERR_UNSUPPORTED;
    if (s == FFTPDE_OK) s = check_ptr(p, in);
    if (s == FFTPDE_OK) s = check_ptr(p, out);
    if (s != FFTPDE_OK) return s;
    return dispatch(p, batch, stride, [&](auto &ps) { return ps.forward(in, out); });
}

fftpde_status fftpde_inverse_batched(fftpde_plan p, const void *in, void *out, int64_t batch,
                                     int64_t stride)
{
    fftpde_status s = check_call(p, batch, stride);
    if (s == FFTPDE_OK && p->colP && stride != p->nx * p->ny) s = FFTPDE_ERR_UNSUPPORTED;
    if (s == FFTPDE_OK) s = check_ptr(p, in);
    if (s == FFTPDE_OK) s = check_ptr(p, out);
    if (s != FFTPDE_OK) return s;
    return dispatch(p, batch, stride, [&](auto &ps) { return ps.inverse(in, out); });
}

fftpde_status fftpde_poisson_batched(fftpde_plan p, const void *rho, void *u, int64_t batch,
                                     int64_t stride)
{
    fftpde_status s = check_call(p, batch, stride);
    if (s == FFTPDE_OK) s = check_ptr(p, rho);
    if (s == FFTPDE_OK) s = check_ptr(p, u);
    if (s != FFTPDE_OK) return s;
    return dispatch(p, batch, stride, [&](auto &ps) { return ps.solve_step(rho, u, COL_POISSON); });
}

fftpde_status fftpde_diffuse_batched(fftpde_plan p, const void *u0, void *u, int64_t batch,
                                     int64_t stride, double D, double dt, int64_t nsteps)
{
    fftpde_status s = check_call(p, batch, stride);
    if (s == FFTPDE_OK) s = check_ptr(p, u0);
    if (s == FFTPDE_OK) s = check_ptr(p, u);
    if (s != FFTPDE_OK) return s;
    if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0 || nsteps < 0)
        return FFTPDE_ERR_INVALID_ARG;
    if (nsteps == 0) return copy_grids(p, u0, u, batch, stride);
    {
        DeviceGuard g(p->device);
        s = ensure_diffusion_tables(p, D, dt);
    }
    if (s != FFTPDE_OK) return s;
    const std::array<uint64_t, 6> key{1, (uint64_t)(uintptr_t)u0, (uint64_t)(uintptr_t)u, (uint64_t)batch,
                                      (uint64_t)stride, (uint64_t)nsteps};
    return run_graphed(p, key, [&] {
        return dispatch(p, batch, stride, [&](auto &ps) { return ps.diffuse(u0, u, nsteps); });
    });
}

fftpde_status fftpde_wave_step_batched(fftpde_plan p, void *u, void *ut, int64_t batch,
                                       int64_t stride, double c, double dt, int64_t nsteps)
{
    fftpde_status s = check_call(p, batch, stride);
    if (s == FFTPDE_OK) s = check_ptr(p, u);
    if (s == FFTPDE_OK) s = check_ptr(p, ut);
    if (s != FFTPDE_OK) return s;
    if (u == ut) return FFTPDE_ERR_INVALID_ARG;
    if (!std::isfinite(c) || !std::isfinite(dt) || c < 0 || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
    if (nsteps == 0) return FFTPDE_OK;
    {
        DeviceGuard g(p->device);
        s = ensure_wave_tables(p, c, dt);
    }
    if (s != FFTPDE_OK) return s;
    const std::array<uint64_t, 6> key{2, (uint64_t)(uintptr_t)u, (uint64_t)(uintptr_t)ut, (uint64_t)batch,
                                      (uint64_t)stride, (uint64_t)nsteps};
    return run_graphed(p, key, [&] {
        return dispatch(p, batch, stride, [&](auto &ps) { return ps.wave(u, ut, nsteps); });
    });
}

// ---- slab building blocks --------------------------------------------------------
fftpde_status fftpde_rows(fftpde_plan p, const void *in, void *out, int64_t nrows, int inverse)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->is3d || p->is_real || p->sharded) return FFTPDE_ERR_UNSUPPORTED;
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    if (nrows == 0) return FFTPDE_ERR_EMPTY;
    if (nrows < 0) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = check_ptr(p, in);
    if (s == FFTPDE_OK) s = check_ptr(p, out);
    if (s != FFTPDE_OK) return s;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    cudaError_t e;
    if (p->dtype == FFTPDE_C128) {
        Passes<double> ps{p, 1, nrows * p->nx};
        const int64_t ny0 = p->ny;
        p->ny = nrows;                     // the row pass only uses ny as the row count
        e = ps.rows(in, out, inverse);
        p->ny = ny0;
    } else {
        Passes<float> ps{p, 1, nrows * p->nx};
        const int64_t ny0 = p->ny;
        p->ny = nrows;
        e = ps.rows(in, out, inverse);
        p->ny = ny0;
    }
    return cuda_status(e);
}

} // extern "C"
namespace {
fftpde_status cols_slab_impl(fftpde_plan p, const void *in, void *out, int64_t col0, int64_t ncols, int op, double D,
                             double dt, const PeerOut &po)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->is3d || p->is_real || p->sharded) return FFTPDE_ERR_UNSUPPORTED;
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    if (ncols == 0) return FFTPDE_ERR_EMPTY;
    if (ncols < 0 || !is_pow2(ncols) || p->nx % ncols || col0 < 0 || col0 % ncols || col0 + ncols > p->nx)
        return FFTPDE_ERR_INVALID_ARG;
    if (op != COL_POISSON && op != COL_DIFFUSE && op != FFTPDE_OP_DIFFUSE_Y) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = check_ptr(p, in);
    if (s == FFTPDE_OK) s = check_ptr(p, out);
    if (s != FFTPDE_OK) return s;
    const bool yonly = op == FFTPDE_OP_DIFFUSE_Y;     // the y factor alone (separable diffusion, R26)
    if (yonly) op = COL_DIFFUSE;
    if (op == COL_DIFFUSE) {
        if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0) return FFTPDE_ERR_INVALID_ARG;
        DeviceGuard g(p->device);
        s = ensure_diffusion_tables(p, D, dt);
        if (s != FFTPDE_OK) return s;
    }
    int64_t P2, Q2;
    fftpde::col2_split(p->ny, ncols, (int)elem_cplx(p), P2, Q2);
    if (p->ny > kMaxLen && !P2) return FFTPDE_ERR_UNSUPPORTED;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    cudaError_t e;
    const ColTw ctw{p->ws + p->o_twy, p->ws + p->o_twP, p->ws + p->o_twQ, p->ws + p->o_twN, p->ws + p->o_twy8,
                    p->ws + p->o_twy32};
    auto run = [&](auto tag) {
        using T = decltype(tag);
        OpTables<T> t = tables<T>(p);
        t.kx2 += col0;             // global column col0 + c
        t.ex = yonly ? (const T *)(p->ws + p->o_one) : t.ex + col0;
        return launch(p, FFTPDE_KERNEL_COL, [&] {
            return launch_cols<T>(p->ny, in, out, ncols, ncols * p->ny, 1, op, ctw, t, p->stream, po);
        });
    };
    if (p->colP == 0 && P2) return FFTPDE_ERR_UNSUPPORTED;   // two-level tables not built for this plan
    e = p->dtype == FFTPDE_C128 ? run(0.0) : run(0.0f);
    return cuda_status(e);
}
} // namespace
extern "C" {
fftpde_status fftpde_cols_slab(fftpde_plan p, const void *in, void *out, int64_t col0, int64_t ncols,
                               int op, double D, double dt)
{
    return cols_slab_impl(p, in, out, col0, ncols, op, D, dt, PeerOut{});
}

fftpde_status fftpde_cols_to_peers(fftpde_plan p, void *colslab, void *const *peers, int npeers, int rank, int64_t R,
                                   int op, double D, double dt)
{
    if (!p || !colslab || !peers || npeers < 1 || npeers > kMaxPeers || rank < 0 || rank >= npeers || R <= 0)
        return FFTPDE_ERR_INVALID_ARG;
    if (R * npeers != p->ny || p->nx % npeers || !is_pow2(p->nx / npeers)) return FFTPDE_ERR_INVALID_ARG;
    PeerOut po;
    for (int q = 0; q < npeers; ++q) {
        if (!peers[q] || ((uintptr_t)peers[q] & 15u)) return FFTPDE_ERR_INVALID_ARG;
        po.p[q] = peers[q];
    }
    const int64_t bw = p->nx / npeers;
    po.rank = rank;
    po.R = R;
    po.nx = p->nx;
    while (((int64_t)1 << po.bwlog) < bw) ++po.bwlog;
    // the column pass works in place on the slab (its scratch); the result goes to the peers
    return cols_slab_impl(p, colslab, colslab, rank * bw, bw, op, D, dt, po);
}

fftpde_status fftpde_pack_blocks(fftpde_plan p, const void *in, void *out, int64_t nrows, int64_t nblocks,
                                 int64_t bw, int direction)
{
    if (!p || !in || !out || in == out || nrows < 0 || nblocks < 0 || bw <= 0 || (direction != 0 && direction != 1))
        return FFTPDE_ERR_INVALID_ARG;
    const int64_t bytes = bw * (int64_t)elem_cplx(p);
    if (bytes % 16 || ((uintptr_t)in & 15u) || ((uintptr_t)out & 15u)) return FFTPDE_ERR_INVALID_ARG;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    ++p->launches;
    return cuda_status(launch_pack(in, out, nrows, nblocks, bytes, direction, p->stream));
}

// ---- diagonal k-space operators ----------------------------------------------------
fftpde_status fftpde_apply(fftpde_plan p, const void *in, void *out, int op)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = check_call(p, p->batch, p->nx * p->ny);
    if (s == FFTPDE_OK) s = check_ptr(p, in);
    if (s == FFTPDE_OK) s = check_ptr(p, out);
    if (s != FFTPDE_OK) return s;
    if (op != FFTPDE_KOP_LAPLACIAN && op != FFTPDE_KOP_DX && op != FFTPDE_KOP_DY) return FFTPDE_ERR_INVALID_ARG;
    return dispatch(p, p->batch, p->nx * p->ny, [&](auto &ps) { return ps.apply(in, out, op); });
}

size_t fftpde_diffuse_source_scratch_size(fftpde_plan p)
{
    return p ? 2 * (size_t)(p->batch * p->nx * p->ny) * elem_cplx(p) : 0;
}

fftpde_status fftpde_diffuse_source(fftpde_plan p, const void *u0, const void *src, void *u, double D, double dt,
                                    int64_t nsteps, void *scratch, size_t scratch_bytes)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = check_call(p, p->batch, p->nx * p->ny);
    if (s == FFTPDE_OK) s = check_ptr(p, u0);
    if (s == FFTPDE_OK) s = check_ptr(p, src);
    if (s == FFTPDE_OK) s = check_ptr(p, u);
    if (s != FFTPDE_OK) return s;
    if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0 || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
    if (src == u && u != u0) return FFTPDE_ERR_INVALID_ARG;
    if (nsteps == 0) return copy_grids(p, u0, u, p->batch, p->nx * p->ny);
    if (!scratch || scratch_bytes < fftpde_diffuse_source_scratch_size(p) || ((uintptr_t)scratch & 255u))
        return FFTPDE_ERR_WORKSPACE;
    uint64_t hsh = 1469598103934665603ull;
    const double prm[2] = {D, dt};
    const void *ptrs[2] = {src, scratch};
    for (const unsigned char *b : {(const unsigned char *)prm, (const unsigned char *)ptrs})
        for (size_t i = 0; i < 16; ++i) { hsh ^= b[i]; hsh *= 1099511628211ull; }
    const std::array<uint64_t, 6> key{4, (uint64_t)(uintptr_t)u0, (uint64_t)(uintptr_t)u, (uint64_t)p->batch,
                                      (uint64_t)nsteps, hsh};
    return run_graphed(p, key, [&] {
        return dispatch(p, p->batch, p->nx * p->ny,
                        [&](auto &ps) { return ps.diffuse_source(u0, src, u, D, dt, nsteps, scratch); });
    });
}

// ---- time-dependent source: RK4 ----------------------------------------------
size_t fftpde_wave_rk4_scratch_size(fftpde_plan p)
{
    return p ? 5 * (size_t)(p->nx * p->ny) * elem_cplx(p) : 0;
}

fftpde_status fftpde_wave_rk4(fftpde_plan p, void *u, void *ut, double c, double xmin, double ymin, double A,
                              double sigma, double Omega, double gamma, double rs, double t0, double dt,
                              int64_t nsteps, void *means, void *scratch, size_t scratch_bytes)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    if (p->batch != 1 || p->is3d || p->is_real || p->sharded) return FFTPDE_ERR_UNSUPPORTED;
    fftpde_status s = check_ptr(p, u);
    if (s == FFTPDE_OK) s = check_ptr(p, ut);
    if (s != FFTPDE_OK) return s;
    if (u == ut) return FFTPDE_ERR_INVALID_ARG;
    const double prm[] = {c, xmin, ymin, A, sigma, Omega, gamma, rs, t0, dt};
    for (double v : prm)
        if (!std::isfinite(v)) return FFTPDE_ERR_INVALID_ARG;
    if (c < 0 || !(sigma > 0) || !(dt > 0) || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
    if (means && ((uintptr_t)means % elem_cplx(p))) return FFTPDE_ERR_INVALID_ARG;
    if (!scratch || scratch_bytes < fftpde_wave_rk4_scratch_size(p) || ((uintptr_t)scratch & 255u))
        return FFTPDE_ERR_WORKSPACE;
    SrcParams base{xmin, ymin, p->Lx, p->Ly, 0.0, 0.0, 0.0, sigma};
    // the stage times and source positions are kernel arguments baked into the
    // captured graph: every parameter is part of the graph key
    uint64_t hsh = 1469598103934665603ull;
    auto mix = [&](const void *d, size_t n) {
        const unsigned char *b = (const unsigned char *)d;
        for (size_t i = 0; i < n; ++i) { hsh ^= b[i]; hsh *= 1099511628211ull; }
    };
    mix(prm, sizeof prm);
    mix(&scratch, sizeof scratch);
    const std::array<uint64_t, 6> key{3, (uint64_t)(uintptr_t)u, (uint64_t)(uintptr_t)ut, (uint64_t)(uintptr_t)means,
                                      (uint64_t)nsteps, hsh};
    return run_graphed(p, key, [&] {
        return dispatch(p, 1, p->nx * p->ny, [&](auto &ps) {
            return ps.wave_rk4(u, ut, c, base, A, Omega, gamma, rs, t0, dt, nsteps, means, scratch);
        });
    });
}

fftpde_status fftpde_peer_transpose(fftpde_plan p, const void *src, void *const *peers, int npeers, int rank,
                                    int64_t R, int64_t bw, int direction)
{
    if (!p || !src || !peers || npeers < 1 || npeers > kMaxPeers || rank < 0 || rank >= npeers || R < 0 || bw <= 0 ||
        (direction != 0 && direction != 1))
        return FFTPDE_ERR_INVALID_ARG;
    const int64_t bytes = bw * (int64_t)elem_cplx(p);
    if (bytes % 16 || ((uintptr_t)src & 15u)) return FFTPDE_ERR_INVALID_ARG;
    PeerPtrs pp{};
    for (int q = 0; q < npeers; ++q) {
        if (!peers[q] || ((uintptr_t)peers[q] & 15u)) return FFTPDE_ERR_INVALID_ARG;
        pp.p[q] = peers[q];
    }
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    ++p->launches;
    return cuda_status(launch_peer_transpose(src, pp, npeers, rank, R, bytes, direction, p->stream));
}

// ---- the distributed four-step pieces (R28) on a plain 32768^2 complex128 plan -------
namespace {
fftpde_status fs_part_args(fftpde_plan p, int nranks, int rank)
{
    if (!p || nranks < 1 || rank < 0 || rank >= nranks) return FFTPDE_ERR_INVALID_ARG;
    if (p->is3d || p->is_real || p->sharded || !p->fs || !fftpde::fs_dist_supported(nranks)) return FFTPDE_ERR_UNSUPPORTED;
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    return FFTPDE_OK;
}
bool aligned16(const void *q) { return q && ((uintptr_t)q & 15u) == 0; }
} // namespace

fftpde_status fftpde_fs_part_aa(fftpde_plan p, int op, int nranks, int rank, int xmode, const void *in, void *out,
                                void *phys)
{
    fftpde_status s = fs_part_args(p, nranks, rank);
    if (s != FFTPDE_OK) return s;
    if (op < 0 || op > 2 || (xmode != 0 && xmode != 1) || !aligned16(in) || !aligned16(out) ||
        (op == 2) != (phys != nullptr) || (phys && !aligned16(phys)))
        return FFTPDE_ERR_INVALID_ARG;
    return dispatch(p, 1, p->nx * p->ny, [&](auto &) {
        return launch(p, FFTPDE_KERNEL_AA, [&] {
            return launch_aa_part(op, nranks, rank, xmode, in, out, phys, p->ws + p->o_fs_tw, p->stream);
        });
    });
}

fftpde_status fftpde_fs_part_b(fftpde_plan p, int xmode, int nranks, int rank, void *f, double D, double dt,
                               void *const *peers, int npeers)
{
    fftpde_status s = fs_part_args(p, nranks, rank);
    if (s != FFTPDE_OK) return s;
    if ((xmode != 0 && xmode != 1) || !aligned16(f) || !std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0)
        return FFTPDE_ERR_INVALID_ARG;
    PeerPtrs pp{};
    if (peers) {
        if (npeers != nranks) return FFTPDE_ERR_INVALID_ARG;
        if (xmode == 1 && nranks > fftpde::kFsMaxPeerMaps) return FFTPDE_ERR_UNSUPPORTED;
        for (int q = 0; q < npeers; ++q) {
            if (!aligned16(peers[q])) return FFTPDE_ERR_INVALID_ARG;
            pp.p[q] = peers[q];
        }
    }
    {
        DeviceGuard g(p->device);
        if (!g.ok) return FFTPDE_ERR_CUDA;
        s = ensure_diffusion_tables(p, D, dt);
    }
    if (s != FFTPDE_OK) return s;
    return dispatch(p, 1, p->nx * p->ny, [&](auto &) {
        return launch(p, xmode ? FFTPDE_KERNEL_COL : FFTPDE_KERNEL_ROW, [&] {
            return launch_fs_b_part(xmode != 0, nranks, rank, f, p->ws + p->o_fs_tw32,
                                    (const double *)(p->ws + (xmode ? p->o_fs_my : p->o_fs_mx)), p->stream,
                                    peers ? &pp : nullptr);
        });
    });
}

fftpde_status fftpde_fs_part_perm(fftpde_plan p, int nranks, const void *in, void *out, int direction)
{
    fftpde_status s = fs_part_args(p, nranks, 0);
    if (s != FFTPDE_OK) return s;
    if (!aligned16(in) || !aligned16(out) || in == out || (direction != 0 && direction != 1))
        return FFTPDE_ERR_INVALID_ARG;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    ++p->launches;
    return cuda_status(launch_fs_perm(in, out, nranks, direction, p->stream));
}

fftpde_status fftpde_rows_to_peers(fftpde_plan p, const void *in, void *const *peers, int npeers, int rank,
                                   int64_t R, int op, double D, double dt)
{
    if (!p || !in || !peers || npeers < 1 || npeers > kMaxPeers || rank < 0 || rank >= npeers || R <= 0)
        return FFTPDE_ERR_INVALID_ARG;
    if (p->is3d || p->is_real || p->sharded) return FFTPDE_ERR_UNSUPPORTED;
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    if (op != FFTPDE_ROWS_FWD && op != FFTPDE_ROWS_DIFFUSE) return FFTPDE_ERR_INVALID_ARG;
    if (R * npeers != p->ny || p->nx % npeers || !is_pow2(p->nx / npeers)) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = check_ptr(p, in);
    if (s != FFTPDE_OK) return s;
    PeerOut po;
    for (int q = 0; q < npeers; ++q) {
        if (!peers[q] || ((uintptr_t)peers[q] & 15u)) return FFTPDE_ERR_INVALID_ARG;
        po.p[q] = peers[q];
    }
    po.rank = rank;
    po.R = R;
    while (((int64_t)1 << po.bwlog) < p->nx / npeers) ++po.bwlog;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    if (op == FFTPDE_ROWS_DIFFUSE) {
        if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0) return FFTPDE_ERR_INVALID_ARG;
        s = ensure_diffusion_tables(p, D, dt);
        if (s != FFTPDE_OK) return s;
    }
    const int dir = op == FFTPDE_ROWS_DIFFUSE ? ROW_DIFF : ROW_FWD;
    return dispatch(p, 1, R * p->nx, [&](auto &ps) {
        using T = typename std::remove_reference_t<decltype(ps)>::Real;
        (void)sizeof(T);
        return launch(p, FFTPDE_KERNEL_ROW, [&] {
            if (p->rowP)
                return launch_rows2<T>(p->nx, in, nullptr, nullptr, R, R * p->nx, 1, dir, ps.rtw(), p->stream,
                                       ps.rowmul(), po);
            return launch_rows<T>(p->nx, in, nullptr, nullptr, R, R * p->nx, 1, dir, ps.rtw(), p->stream,
                                  ps.rowmul(), po);
        });
    });
}

// ---- sharded plans ---------------------------------------------------------------
fftpde_status fftpde_nccl_unique_id(void *out)
{
    if (!out) return FFTPDE_ERR_INVALID_ARG;
    if (!nccl().ok) return FFTPDE_ERR_NCCL;
    ncclUniqueId id;
    if (nccl().getUniqueId(&id) != ncclSuccess) return FFTPDE_ERR_NCCL;
    std::memcpy(out, &id, sizeof id);
    return FFTPDE_OK;
}

} // extern "C"
namespace {
// the slab buffers (in place of the full-grid scratch, which sharded plans never use) + the communicator
fftpde_status finish_sharded(fftpde_plan p, int nranks, int rank, const void *uid, int64_t slab_elems)
{
    p->sharded = true;
    // 2D 32768^2 complex128 with a power-of-two P <= 32: the distributed four-step
    // (R28) on the plan's four-step tables; otherwise the slab path's own passes
    p->fsd = p->fs && !p->is3d && !p->pencil && fftpde::fs_dist_supported(nranks);
    p->fs = false;
    p->P = nranks;
    p->loopback = uid == nullptr;
    p->rank = p->loopback ? 0 : rank;
    p->slab_elems = slab_elems;
    const size_t slab = (size_t)slab_elems * elem_cplx(p) * (size_t)(p->loopback ? nranks : 1);
    size_t off = p->o_scr;
    auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
    p->o_shA = take(slab);
    p->o_shB = take(slab);
    p->o_shC = take(slab);
    p->need = off;
    if (p->loopback) return FFTPDE_OK;
    if (!nccl().ok) return FFTPDE_ERR_NCCL;
    DeviceGuard g(p->device);
    if (!g.ok) return FFTPDE_ERR_CUDA;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    if (nccl().commInitRank(&p->comm, nranks, id, rank) != ncclSuccess) {
        p->comm = nullptr;
        return FFTPDE_ERR_NCCL;
    }
    return FFTPDE_OK;
}
bool sharded_args_ok(const void *uid, int rank, int nranks)
{
    if (nranks < 1) return false;
    if (!uid) return rank == FFTPDE_SHARDED_LOOPBACK;
    return rank >= 0 && rank < nranks;
}
} // namespace
extern "C" {

fftpde_status fftpde_plan_2d_sharded(fftpde_plan *plan, int64_t nx, int64_t ny, fftpde_dtype dtype, double Lx,
                                     double Ly, int device, const void *nccl_unique_id, int rank, int nranks)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    *plan = nullptr;
    if (!sharded_args_ok(nccl_unique_id, rank, nranks)) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = fftpde_plan_2d(plan, nx, ny, 1, dtype, Lx, Ly, device);
    if (s != FFTPDE_OK) return s;
    fftpde_plan p = *plan;
    auto fail = [&](fftpde_status st) { fftpde_destroy(p); *plan = nullptr; return st; };
    const int64_t ec = (int64_t)elem_cplx(p);
    if (nx % nranks || ny % nranks || ((nx / nranks) * ec) % 16) return fail(FFTPDE_ERR_UNSUPPORTED);
    int64_t P2, Q2;
    fftpde::col2_split(ny, nx / nranks, (int)ec, P2, Q2);
    if (ny > kMaxLen && !P2) return fail(FFTPDE_ERR_UNSUPPORTED);   // column slab too narrow for long columns
    p->R = ny / nranks;
    p->BW = nx / nranks;
    s = finish_sharded(p, nranks, rank, nccl_unique_id, p->R * nx);
    return s == FFTPDE_OK ? s : fail(s);
}

fftpde_status fftpde_plan_3d_sharded(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t nz, fftpde_dtype dtype,
                                     double Lx, double Ly, double Lz, int device, const void *nccl_unique_id,
                                     int rank, int nranks)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    *plan = nullptr;
    if (!sharded_args_ok(nccl_unique_id, rank, nranks)) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = fftpde_plan_3d(plan, nx, ny, nz, dtype, Lx, Ly, Lz, device);
    if (s != FFTPDE_OK) return s;
    fftpde_plan p = *plan;
    auto fail = [&](fftpde_status st) { fftpde_destroy(p); *plan = nullptr; return st; };
    const int64_t ec = (int64_t)elem_cplx(p);
    if (nz % nranks || ny % nranks || ((ny / nranks) * nx * ec) % 16) return fail(FFTPDE_ERR_UNSUPPORTED);
    if (p->zP && ((ny / nranks) * nx * ec) % 128) return fail(FFTPDE_ERR_UNSUPPORTED);   // col2 z-pass blocks
    p->R = ny / nranks;
    p->nzl = nz / nranks;
    s = finish_sharded(p, nranks, rank, nccl_unique_id, p->nzl * ny * nx);
    return s == FFTPDE_OK ? s : fail(s);
}

fftpde_status fftpde_plan_3d_pencil(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t nz, fftpde_dtype dtype,
                                    double Lx, double Ly, double Lz, int device, const void *nccl_unique_id,
                                    int rank, int pz, int py)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    *plan = nullptr;
    if (pz < 1 || py < 1 || pz > 4096 || py > 4096) return FFTPDE_ERR_INVALID_ARG;
    const int nranks = pz * py;
    if (!sharded_args_ok(nccl_unique_id, rank, nranks)) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = fftpde_plan_3d(plan, nx, ny, nz, dtype, Lx, Ly, Lz, device);
    if (s != FFTPDE_OK) return s;
    fftpde_plan p = *plan;
    auto fail = [&](fftpde_status st) { fftpde_destroy(p); *plan = nullptr; return st; };
    const int64_t ec = (int64_t)elem_cplx(p);
    // every block the packs move is a whole number of 16-byte vectors
    if (nz % pz || ny % py || nx % py || ny % pz || ((nx / py) * ec) % 16) return fail(FFTPDE_ERR_UNSUPPORTED);
    if (p->zP && ((ny / pz) * (nx / py) * ec) % 128) return fail(FFTPDE_ERR_UNSUPPORTED);   // col2 z-pass blocks
    p->pencil = true;
    p->Pz = pz;
    p->Py = py;
    p->nzl = nz / pz;
    p->nyl = ny / py;
    p->nxl = nx / py;
    p->nyl2 = ny / pz;
    // the z-pass line tables in pencil order: rank r = i py + j, line yl2 nxl + xl is the
    // global line (x, y) = (j nxl + xl, i nyl2 + yl2); exy (diffusion) is derived from it
    std::vector<double> k((size_t)(nx * ny));
    for (int r = 0; r < nranks; ++r) {
        const int64_t i = r / py, j = r % py;
        for (int64_t yl = 0; yl < p->nyl2; ++yl)
            for (int64_t xl = 0; xl < p->nxl; ++xl)
                k[(size_t)((r * p->nyl2 + yl) * p->nxl + xl)] = p->kxy2[(size_t)((i * p->nyl2 + yl) * nx + j * p->nxl + xl)];
    }
    p->kxy2.swap(k);
    s = finish_sharded(p, nranks, rank, nccl_unique_id, p->nzl * p->nyl * nx);
    return s == FFTPDE_OK ? s : fail(s);
}

// ---- real plans -------------------------------------------------------------------
fftpde_status fftpde_plan_2d_r2c(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t batch, fftpde_dtype dtype,
                                 double Lx, double Ly, int device)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    *plan = nullptr;
    fftpde_status s = fftpde_plan_2d(plan, nx, ny, batch, dtype, Lx, Ly, device);
    if (s != FFTPDE_OK) return s;
    fftpde_plan p = *plan;
    const int64_t lpp = 128 / (int64_t)elem_cplx(p);                 // columns per 128-byte segment
    if (nx < 2 * lpp || nx / 2 > kMaxLen) {                           // row pass: nx/2 <= 8192 points
        fftpde_destroy(p);
        *plan = nullptr;
        return FFTPDE_ERR_UNSUPPORTED;
    }
    p->is_real = true;
    p->pitch = nx / 2 + lpp;            // multiple of the 128-byte column block, <= nx
    build_twiddles(nx / 2, p->twm);
    p->twr.clear();
    for (int64_t a = 0; a <= nx / 2; ++a) {
        double re, im;
        unit_root(nx, a, re, im);
        p->twr.push_back(re);
        p->twr.push_back(im);
    }
    const size_t ec = elem_cplx(p);
    size_t off = p->need;
    auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
    p->o_twm = take(p->twm.size() / 2 * ec);
    p->o_twr = take(p->twr.size() / 2 * ec);
    p->need = off;
    return FFTPDE_OK;
}

// ---- 3D plans ---------------------------------------------------------------------
fftpde_status fftpde_plan_3d(fftpde_plan *plan, int64_t nx, int64_t ny, int64_t nz, fftpde_dtype dtype, double Lx,
                             double Ly, double Lz, int device)
{
    if (!plan) return FFTPDE_ERR_INVALID_ARG;
    *plan = nullptr;
    if (nz == 0) return FFTPDE_ERR_EMPTY;
    if (nz < 0) return FFTPDE_ERR_INVALID_ARG;
    if (!std::isfinite(Lz) || !(Lz > 0)) return FFTPDE_ERR_INVALID_ARG;
    fftpde_status s = fftpde_plan_2d(plan, nx, ny, nz, dtype, Lx, Ly, device);   // batch = nz slabs
    if (s != FFTPDE_OK) return s;
    fftpde_plan p = *plan;
    auto fail = [&](fftpde_status st) { fftpde_destroy(p); *plan = nullptr; return st; };
    if (!is_pow2(nz)) return fail(FFTPDE_ERR_NOT_POW2_Z);
    // the z-pass: single-level for nz <= 1024, the two-level col2 pass (nz = zP zQ,
    // 128-byte blocks of lines) up to 32768; its per-line tables cover nx*ny lines
    if (nz > 32768 || nx * ny > ((int64_t)1 << 26)) return fail(FFTPDE_ERR_UNSUPPORTED);
    if (nz > 1024) {
        fftpde::col2_split(nz, nx * ny, (int)elem_cplx(p), p->zP, p->zQ);
        if (!p->zP) return fail(FFTPDE_ERR_UNSUPPORTED);
        build_twiddles(p->zP, p->twPz, FFTPDE_COL2_EMAX);
        build_twiddles(p->zQ, p->twQz, FFTPDE_COL2_EMAX);
        build_plain_twiddles(nz, p->twNz);
    }
    p->is3d = true;
    p->nz = nz;
    p->Lz = Lz;
    build_twiddles(nz, p->twz);
    build_twiddles(nz, p->twz8, 8);
    build_k2(nz, Lz, p->kz2);
    p->kxy2.resize((size_t)(nx * ny));
    for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) p->kxy2[(size_t)(y * nx + x)] = p->kx2[(size_t)x] + p->ky2[(size_t)y];
    const size_t er = elem_real(p), ec = elem_cplx(p);
    size_t off = p->o_scr;                     // the 3D tables go before the scratch, which stays last
    auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
    p->o_twz = take(p->twz.size() / 2 * ec);
    p->o_twz8 = take(p->twz8.size() / 2 * ec);
    if (p->zP) {
        p->o_twPz = take(p->twPz.size() / 2 * ec);
        p->o_twQz = take(p->twQz.size() / 2 * ec);
        p->o_twNz = take(p->twNz.size() / 2 * ec);
    }
    p->o_kz2 = take((size_t)nz * er);
    p->o_ez = take((size_t)nz * er);
    p->o_kxy2 = take((size_t)(nx * ny) * er);
    p->o_exy = take((size_t)(nx * ny) * er);
    p->o_zscale = take((size_t)(nx * ny) * er);
    p->o_scr = take(2 * (size_t)(nz * nx * ny) * ec);
    p->need = off;
    return FFTPDE_OK;
}

} // extern "C"
namespace {
fftpde_status ensure_diffusion_tables3(fftpde_plan p, double D, double dt)
{
    if (p->diff3_valid && p->diff3_D == D && p->diff3_dt == dt) return FFTPDE_OK;
    const double scale = 1.0 / ((double)p->nx * (double)p->ny * (double)p->nz);
    std::vector<double> exy(p->kxy2.size()), ez((size_t)p->nz);
    for (size_t i = 0; i < exy.size(); ++i) exy[i] = std::exp(-D * p->kxy2[i] * dt) * scale;
    for (int64_t z = 0; z < p->nz; ++z) ez[(size_t)z] = std::exp(-D * p->kz2[(size_t)z] * dt);
    fftpde_status s = upload(p, p->o_exy, exy);
    if (s == FFTPDE_OK) s = upload(p, p->o_ez, ez);
    // separable form (R26): x factor / (nx ny) in the rows (2D tables), y factor in
    // the y-pass, z factor / nz in the z-pass (the z-pass operator slot is
    // (line, element) = (1/nz, ez[c]))
    if (s == FFTPDE_OK) s = ensure_diffusion_tables(p, D, dt);
    if (s == FFTPDE_OK) s = upload(p, p->o_zscale, std::vector<double>(p->kxy2.size(), 1.0 / (double)p->nz));
    if (s != FFTPDE_OK) return s;
    p->diff3_valid = true;
    p->diff3_D = D;
    p->diff3_dt = dt;
    return FFTPDE_OK;
}

fftpde_status check3(fftpde_plan p, const void *a, const void *b)
{
    if (!p->ws) return FFTPDE_ERR_WORKSPACE;
    fftpde_status s = check_ptr(p, a);
    return s == FFTPDE_OK ? check_ptr(p, b) : s;
}

template <typename F> fftpde_status dispatch3(fftpde_plan p, F &&f)
{
    return dispatch(p, p->nz, p->nx * p->ny, std::forward<F>(f));
}
} // namespace
extern "C" {

// ---- whole-plan entry points --------------------------------------------------
} // extern "C"
namespace {
template <typename F> fftpde_status dispatch_real(fftpde_plan p, F &&f)
{
    return dispatch(p, p->batch, p->nx * p->ny, std::forward<F>(f));
}
} // namespace
extern "C" {
fftpde_status fftpde_forward(fftpde_plan p, const void *in, void *out)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->sharded) {
        fftpde_status s = check3(p, in, out);
        if (s == FFTPDE_OK && in == out) s = FFTPDE_ERR_INVALID_ARG;
        return s != FFTPDE_OK ? s : dispatch_real(p, [&](auto &ps) { return ps.forward_sh(in, out); });
    }
    if (p->is_real) {
        fftpde_status s = check3(p, in, out);
        return s != FFTPDE_OK ? s : dispatch_real(p, [&](auto &ps) { return ps.forward_real(in, out); });
    }
    if (p->is3d) {
        fftpde_status s = check3(p, in, out);
        return s != FFTPDE_OK ? s : dispatch3(p, [&](auto &ps) { return ps.forward3(in, out); });
    }
    return fftpde_forward_batched(p, in, out, p->batch, p->nx * p->ny);
}
fftpde_status fftpde_inverse(fftpde_plan p, const void *in, void *out)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->sharded) {
        fftpde_status s = check3(p, in, out);
        return s != FFTPDE_OK ? s : dispatch_real(p, [&](auto &ps) { return ps.inverse_sh(in, out); });
    }
    if (p->is_real) {
        fftpde_status s = check3(p, in, out);
        return s != FFTPDE_OK ? s : dispatch_real(p, [&](auto &ps) { return ps.inverse_real(in, out); });
    }
    if (p->is3d) {
        fftpde_status s = check3(p, in, out);
        return s != FFTPDE_OK ? s : dispatch3(p, [&](auto &ps) { return ps.inverse3(in, out); });
    }
    return fftpde_inverse_batched(p, in, out, p->batch, p->nx * p->ny);
}
fftpde_status fftpde_poisson(fftpde_plan p, const void *rho, void *u)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->sharded) {
        fftpde_status s = check3(p, rho, u);
        return s != FFTPDE_OK ? s : dispatch_real(p, [&](auto &ps) { return ps.step_sh(rho, u, COL_POISSON); });
    }
    if (p->is_real) {
        fftpde_status s = check3(p, rho, u);
        return s != FFTPDE_OK ? s : dispatch_real(p, [&](auto &ps) { return ps.poisson_real(rho, u); });
    }
    if (p->is3d) {
        fftpde_status s = check3(p, rho, u);
        return s != FFTPDE_OK ? s : dispatch3(p, [&](auto &ps) { return ps.poisson3(rho, u); });
    }
    return fftpde_poisson_batched(p, rho, u, p->batch, p->nx * p->ny);
}
fftpde_status fftpde_diffuse(fftpde_plan p, const void *u0, void *u, double D, double dt, int64_t nsteps)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->sharded) {
        fftpde_status s = check3(p, u0, u);
        if (s != FFTPDE_OK) return s;
        if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0 || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
        DeviceGuard g(p->device);
        if (nsteps == 0)
            return u0 == u ? FFTPDE_OK
                           : cuda_status(cudaMemcpyAsync(u, u0, (size_t)p->slab_elems * elem_cplx(p) *
                                                                         (size_t)(p->loopback ? p->P : 1),
                                                         cudaMemcpyDeviceToDevice, p->stream));
        s = p->is3d ? ensure_diffusion_tables3(p, D, dt) : ensure_diffusion_tables(p, D, dt);
        if (s != FFTPDE_OK) return s;
        if (p->fsd)
            return dispatch_real(p, [&](auto &ps) {
                if constexpr (std::is_same_v<std::decay_t<decltype(ps)>, Passes<double>>) return ps.diffuse_fsd(u0, u, nsteps);
                return cudaErrorNotSupported;
            });
        for (int64_t k = 0; k < nsteps && s == FFTPDE_OK; ++k)
            s = dispatch_real(p, [&](auto &ps) { return ps.step_sh(k == 0 ? u0 : u, u, COL_DIFFUSE); });
        return s;
    }
    if (p->is_real) {
        fftpde_status s = check3(p, u0, u);
        if (s != FFTPDE_OK) return s;
        if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0 || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
        if (nsteps == 0) {
            if (u0 == u) return FFTPDE_OK;
            DeviceGuard g(p->device);
            return cuda_status(cudaMemcpyAsync(u, u0, (size_t)(p->batch * p->nx * p->ny) * elem_real(p),
                                               cudaMemcpyDeviceToDevice, p->stream));
        }
        {
            DeviceGuard g(p->device);
            s = ensure_diffusion_tables(p, D, dt);
        }
        if (s != FFTPDE_OK) return s;
        const std::array<uint64_t, 6> key{6, (uint64_t)(uintptr_t)u0, (uint64_t)(uintptr_t)u, (uint64_t)p->batch,
                                          (uint64_t)p->nx, (uint64_t)nsteps};
        return run_graphed(p, key, [&] { return dispatch_real(p, [&](auto &ps) { return ps.diffuse_real(u0, u, nsteps); }); });
    }
    if (p->is3d) {
        fftpde_status s = check3(p, u0, u);
        if (s != FFTPDE_OK) return s;
        if (!std::isfinite(D) || !std::isfinite(dt) || D < 0 || dt < 0 || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
        if (nsteps == 0) return copy_grids(p, u0, u, p->nz, p->nx * p->ny);
        {
            DeviceGuard g(p->device);
            s = ensure_diffusion_tables3(p, D, dt);
        }
        if (s != FFTPDE_OK) return s;
        const std::array<uint64_t, 6> key{5, (uint64_t)(uintptr_t)u0, (uint64_t)(uintptr_t)u, (uint64_t)p->nz,
                                          (uint64_t)p->nx, (uint64_t)nsteps};
        return run_graphed(p, key, [&] { return dispatch3(p, [&](auto &ps) { return ps.diffuse3(u0, u, nsteps); }); });
    }
    return fftpde_diffuse_batched(p, u0, u, p->batch, p->nx * p->ny, D, dt, nsteps);
}
fftpde_status fftpde_wave_step(fftpde_plan p, void *u, void *ut, double c, double dt, int64_t nsteps)
{
    if (!p) return FFTPDE_ERR_INVALID_ARG;
    if (p->is3d || p->sharded) return FFTPDE_ERR_UNSUPPORTED;
    if (p->is_real) {
        fftpde_status s = check3(p, u, ut);
        if (s != FFTPDE_OK) return s;
        if (u == ut || !std::isfinite(c) || !std::isfinite(dt) || c < 0 || nsteps < 0) return FFTPDE_ERR_INVALID_ARG;
        if (nsteps == 0) return FFTPDE_OK;
        {
            DeviceGuard g(p->device);
            s = ensure_wave_tables(p, c, dt);
        }
        if (s != FFTPDE_OK) return s;
        const std::array<uint64_t, 6> key{7, (uint64_t)(uintptr_t)u, (uint64_t)(uintptr_t)ut, (uint64_t)p->batch,
                                          (uint64_t)p->nx, (uint64_t)nsteps};
        return run_graphed(p, key, [&] { return dispatch_real(p, [&](auto &ps) { return ps.wave_real(u, ut, nsteps); }); });
    }
    return fftpde_wave_step_batched(p, u, ut, p->batch, p->nx * p->ny, c, dt, nsteps);
}

} // extern "C"
