// dispatch.cuh -- launch configurations and length dispatch of the pass kernels.
// Included by the per-dtype instantiation units (passes_c128.cu, passes_c64.cu).
#pragma once
#include <atomic>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <utility>
#include "kernels.cuh"
#include "pipe.cuh"
#include "col2.cuh"
#include "row2d.cuh"
#include "line.cuh"
#include "tmacols.cuh"
#include <cudaTypedefs.h>
#ifndef FFTPDE_COL2_MINB
#define FFTPDE_COL2_MINB 2
#endif


namespace fftpde {

#define FFTPDE_LEN_CASES(X) \
    X(1) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

// Opt a kernel into > 48 KiB dynamic shared memory once per device.
template <typename K> struct SmemOptIn {
    std::atomic<uint64_t> done{0};
    cudaError_t operator()(K kernel, size_t bytes)
    {
        if (bytes <= 48 * 1024) return cudaSuccess;
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        const uint64_t bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e == cudaSuccess) done.fetch_or(bit);
        return e;
    }
};

// ---- launch shapes ---------------------------------------------------------

// Persistent pipelined line pass: grid = resident CTAs (occupancy x SMs).
template <typename T, int N, bool COLS> struct PipeCfg {
    using C = typename cplx_t<T>::type;
    static constexpr int TPT = Shape<N>::TPT;
    static constexpr int TARGET = (COLS && sizeof(T) == 4) ? 512 : 256;   // threads per CTA
    static constexpr int W = TPT >= TARGET ? 1 : TARGET / TPT;
    static constexpr int NBUF = PipeSmem<C, N, W, COLS, 2>::BYTES <= 200 * 1024 ? 2 : 1;
    // a persistent thread's twiddles stay in registers when the budget allows
    static constexpr bool TWREG = W * TPT <= 256 && Shape<N>::STAGES <= 2;
    // rows of >= 2048 points arrive as one bulk copy per row (tools/exp_line.cu:
    // 4096-point rows FWD 118 -> 99 us, MID 194 -> 185 us; 2048 MID 175 -> 157 us)
    static constexpr bool BULK = !COLS && N >= 2048;
    using L = PipeSmem<C, N, W, COLS, NBUF>;
    static constexpr size_t SMEM = L::BYTES + (BULK ? 8 * NBUF * W : 0);
};

inline int sm_count()
{
    static std::atomic<int> cached{0};
    int v = cached.load();
    if (v) return v;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cached.store(v);
    return v;
}

// Launch with programmatic dependent launch (PDL) allowed: the grid may be
// scheduled while its predecessor on the stream drains; the kernel's pdl_wait()
// orders its field accesses after the predecessor's completion.  Only kernels
// that call pdl_wait() before touching field memory go through here.
// FFTPDE_PDL = bit mask of the launch families that use it (A/B measurements):
// 1 line passes (pipe / line / small solve), 2 col2, 4 row2d.  Default 5: on
// B200 PDL gains 3% on C2 (line passes) and 2% on C5 (row2d), while an early
// launched col2 grid slows C3 by 18% (its clusters are placed while the row
// pass drains; profiles/r01/pdl_ab.txt), so col2 is launched normally.
// PDL_FOURSTEP: the four-step C5 passes (fourstep.cu); off by default: early-launched
// successors hold SM slots while the predecessor's last tiles drain (C5 solve
// 660 vs 594 ms per 20 steps with it on).
enum PdlFamily { PDL_LINE = 1, PDL_COL2 = 2, PDL_ROW2D = 4, PDL_FOURSTEP = 8 };
inline bool pdl_enabled(int family = PDL_LINE)
{
    static const int mask = [] {
        const char *e = std::getenv("FFTPDE_PDL");
        return e ? std::atoi(e) : PDL_LINE | PDL_ROW2D;
    }();
    return (mask & family) != 0;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_fam(int family, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled(family) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <typename T, int N, bool COLS, int OP>
cudaError_t pipe_n(const void *in, void *out, PipeArgs args, const void *tw, const OpTables<T> &tab,
                   cudaStream_t st, const PeerOut &po = PeerOut{})
{
    using C = typename cplx_t<T>::type;
    using Cfg = PipeCfg<T, N, COLS>;
    constexpr int W = Cfg::W;
    constexpr int THREADS = W * Shape<N>::TPT;
    const size_t smem = Cfg::SMEM;
    auto k = pipe_kernel<T, N, W, COLS, OP, Cfg::NBUF, 1, Cfg::TWREG, Cfg::BULK>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, smem);
    if (e != cudaSuccess) return e;
    static std::atomic<int> per_sm{0};
    int occ = per_sm.load();
    if (!occ) {
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, THREADS, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        per_sm.store(occ);
    }
    args.groups = (args.nlines + W - 1) / W;
    const int64_t batch = args.ntiles;                  // caller passes the batch here
    args.ntiles = batch * args.groups;
    const int64_t grid = std::min<int64_t>(args.ntiles, (int64_t)occ * sm_count());
    return launch_pdl(k, dim3((unsigned)grid), dim3(THREADS), smem, st, (const C *)in, (C *)out, args, (const C *)tw,
                      tab, po);
}

// ---- occupancy-oriented line pass (line.cuh) ----------------------------------
// Shapes measured faster than the persistent pipe_kernel on B200
// (tools/exp_line.cu, profiles/r01/exp_line.txt); E = 0: use pipe_kernel.
template <typename T, int N, bool COLS> struct LinePolicy {
    static constexpr bool C64 = sizeof(T) == 4;
    // complex64 512-point lines (C4); complex128 1024-point lines (C2): radix 32,
    // one warp per row, 4 adjacent columns per CTA (tools/exp_e32.cu)
    static constexpr int E = (C64 && N == 512) ? (COLS ? 8 : 16) : (!C64 && N == 1024) ? 32 : 0;
    static constexpr int W = C64 ? (COLS ? 8 : 4) : (COLS ? 4 : 1);
    static constexpr int MINB = C64 ? (COLS ? 3 : 2) : (COLS ? 2 : 4);
};
template <int E> inline const void *tw_for(const ColTw &c) { return E == 8 ? c.tw8 : E == 32 ? c.tw32 : c.tw; }

template <typename T, int N, int E, int W, bool COLS, int OP, int MINB>
cudaError_t line_n(const void *in, void *out, void *out2, int64_t nlines, int64_t line_stride, int64_t elem_stride,
                   int64_t stride, int64_t batch, const void *tw, const OpTables<T> &tab, cudaStream_t st,
                   const PeerOut &po = PeerOut{}, int family = PDL_LINE)
{
    using C = typename cplx_t<T>::type;
    using L = LineSmem<C, N, E, W, COLS>;
    auto k = line_kernel<T, N, E, W, COLS, OP, MINB>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, L::BYTES);
    if (e != cudaSuccess) return e;
    LineArgs a{nlines, line_stride, elem_stride, stride, (nlines + W - 1) / W, out2};
    const int64_t grid = batch * a.groups;
    return launch_fam(family, k, dim3((unsigned)grid), dim3(W * (N / E)), L::BYTES, st, (const C *)in, (C *)out, a,
                      (const C *)tw, tab, po);
}

template <typename T, int N>
cudaError_t rows_n(const void *in, void *out, void *out2, int64_t ny, int64_t stride, int64_t batch,
                   int dir, const ColTw &ctw, cudaStream_t st, RowMul rm, const PeerOut &po)
{
    OpTables<T> tab{};
    tab.scale = (T)1;
    if (dir == ROW_DIFF) {                    // operator slot (line, element) = (ones[b], mul[a])
        if (!rm.mul || !rm.ones) return cudaErrorInvalidValue;
        tab.ex = (const T *)rm.ones;
        tab.ey = (const T *)rm.mul;
        tab.ey2d = (const T *)rm.mul2d;
        tab.ey2d_mod = rm.mod;
    }
    using LP = LinePolicy<T, N, false>;
    if constexpr (LP::E > 0) {
        const void *tw = tw_for<LP::E>(ctw);
        if (tw) {   // (a plan without this radix's table takes the pipe pass)
        if (dir == ROW_DIFF)
            return line_n<T, N, LP::E, LP::W, false, LN_DIFFUSE, LP::MINB>(in, out, nullptr, ny, N, 1, stride, batch, tw, tab, st, po);
        if (dir == ROW_INV)
            return line_n<T, N, LP::E, LP::W, false, LN_INV, LP::MINB>(in, out, nullptr, ny, N, 1, stride, batch, tw, tab, st, po);
        if (dir == ROW_MID)
            return line_n<T, N, LP::E, LP::W, false, LN_MID, LP::MINB>(in, out, out2, ny, N, 1, stride, batch, tw, tab, st, po);
        return line_n<T, N, LP::E, LP::W, false, LN_FWD, LP::MINB>(in, out, nullptr, ny, N, 1, stride, batch, tw, tab, st, po);
        }
    }
    const void *tw = ctw.tw;
    PipeArgs a{ny, N, 1, stride, batch, 0, dir, out2};
    if (dir == ROW_DIFF) return pipe_n<T, N, false, PIPE_DIFFUSE>(in, out, a, tw, tab, st, po);
    if (dir == ROW_INV) return pipe_n<T, N, false, PIPE_INV>(in, out, a, tw, tab, st, po);
    if (dir == ROW_MID) return pipe_n<T, N, false, PIPE_MID>(in, out, a, tw, tab, st, po);
    return pipe_n<T, N, false, PIPE_FWD>(in, out, a, tw, tab, st, po);
}

// ---- TMA column pass (tmacols.cuh): complex128 columns of 256..1024 points ----
// cuTensorMapEncodeTiled comes from the driver through the runtime's entry-point
// query (no link-time libcuda dependency); null if unavailable.
inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *f = nullptr;
        const char *env = std::getenv("FFTPDE_TMA");      // FFTPDE_TMA=0: the non-TMA passes (tests)
        if (env && env[0] == '0') return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000)f;
    }();
    return fn;
}
// the field as a 3D tensor of reals {2 nx, ny, batch}; boxes of 2W reals x BOXR rows
template <typename T>
bool tma_map(CUtensorMap &m, const void *p, int64_t nx, int64_t ny, int64_t batch, int64_t stride, int W, int boxr,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B, CUtensorMapL2promotion prom = CU_TENSOR_MAP_L2_PROMOTION_L2_128B)
{
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t esz = 2 * sizeof(T);
    cuuint64_t dims[3] = {(cuuint64_t)(2 * nx), (cuuint64_t)ny, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)nx * esz, (cuuint64_t)stride * esz};
    cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)boxr, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(&m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
               const_cast<void *>(p), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, prom,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// complex128 columns of 256 / 512 points (radix 16, one CTA per SM); complex64
// columns of 512 points (radix 32, three CTAs per SM) (tools/exp_tma.cu, exp_e32.cu)
template <typename T, int N> struct TmaColPolicy {
    static constexpr bool C64 = sizeof(T) == 4;
    static constexpr bool ON = C64 ? N == 512 : (N >= 256 && N <= 512);
    static constexpr int W = 64 / (2 * (int)sizeof(T));
    static constexpr int E = C64 ? 32 : 16;
    static constexpr int MINB = C64 ? 3 : 1;
};
// returns cudaErrorNotSupported when the shape or the driver does not allow it (caller falls back)
template <typename T, int N, int OP>
cudaError_t tma_cols_n(const void *in, void *out, int64_t nx, int64_t stride, int64_t batch, const void *tw,
                       const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    using TP = TmaColPolicy<T, N>;
    constexpr int W = TP::W;
    using L = TmaColSmem<C, N, W, TP::E>;
    if (nx < W || nx % W || batch > (int64_t)1 << 31) return cudaErrorNotSupported;
    CUtensorMap mi, mo;
    if (!tma_map<T>(mi, in, nx, N, batch, stride, W, L::BOXR)) return cudaErrorNotSupported;
    if (in == out) mo = mi;
    else if (!tma_map<T>(mo, out, nx, N, batch, stride, W, L::BOXR)) return cudaErrorNotSupported;
    auto k = tma_cols_kernel<T, N, W, OP, TP::MINB, TP::E>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, L::BYTES);
    if (e != cudaSuccess) return e;
    constexpr int THREADS = W * Shape<N, TP::E>::TPT;
    static std::atomic<int> per_sm{0};
    int occ = per_sm.load();
    if (!occ) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, THREADS, L::BYTES);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        per_sm.store(occ);
    }
    TmaColArgs a{nx, nx / W, 0};
    a.ntiles = batch * a.groups;
    const int64_t grid = std::min<int64_t>(a.ntiles, (int64_t)occ * sm_count());
    return launch_pdl(k, dim3((unsigned)grid), dim3(THREADS), L::BYTES, st, mi, mo, a, (const C *)tw, tab);
}

inline bool fs_tma_by()
{
    // measured slower than the line pass (C5 col pass 11.3 vs 11.0 ms per step): opt-in
    static const bool on = [] { const char *e = std::getenv("FFTPDE_FS_TMA_BY"); return e && e[0] == '1'; }();
    return on;
}
template <typename T, int N>
cudaError_t cols_n(const void *in, void *out, int64_t nx, int64_t stride, int64_t batch, int op,
                   const ColTw &ctw, const OpTables<T> &tab, cudaStream_t st, const PeerOut &po = PeerOut{})
{
    using LP = LinePolicy<T, N, true>;
    // complex128 1024-point columns take the TMA pass only as the four-step By pass of
    // an HBM-resident field (C5); the L2-resident C2 columns are faster in the line pass
    constexpr bool TMA_FS = sizeof(T) == 8 && N == 1024;
    if constexpr (TmaColPolicy<T, N>::ON || TMA_FS) if (!po.p[0] && (TmaColPolicy<T, N>::ON || (tab.ey2d && fs_tma_by()))) {
        using TP = TmaColPolicy<T, N>;
        const void *tw = tw_for<TP::E>(ctw);
        cudaError_t e = cudaErrorNotSupported;
        if (tw) switch (op) {
        case COL_FWD: e = tma_cols_n<T, N, PIPE_FWD>(in, out, nx, stride, batch, tw, tab, st); break;
        case COL_INV: e = tma_cols_n<T, N, PIPE_INV_SCALED>(in, out, nx, stride, batch, tw, tab, st); break;
        case COL_POISSON: e = tma_cols_n<T, N, PIPE_POISSON>(in, out, nx, stride, batch, tw, tab, st); break;
        case COL_DIFFUSE: e = tma_cols_n<T, N, PIPE_DIFFUSE>(in, out, nx, stride, batch, tw, tab, st); break;
        default: return cudaErrorInvalidValue;
        }
        if (e != cudaErrorNotSupported) return e;
    }
    if constexpr (LP::E > 0) {
        const void *tw = tw_for<LP::E>(ctw);
        if (tw) switch (op) {
        case COL_FWD: return line_n<T, N, LP::E, LP::W, true, LN_FWD, LP::MINB>(in, out, nullptr, nx, 1, nx, stride, batch, tw, tab, st, po);
        case COL_INV: return line_n<T, N, LP::E, LP::W, true, LN_INV_SCALED, LP::MINB>(in, out, nullptr, nx, 1, nx, stride, batch, tw, tab, st, po);
        case COL_POISSON: return line_n<T, N, LP::E, LP::W, true, LN_POISSON, LP::MINB>(in, out, nullptr, nx, 1, nx, stride, batch, tw, tab, st, po);
        case COL_DIFFUSE: return line_n<T, N, LP::E, LP::W, true, LN_DIFFUSE, LP::MINB>(in, out, nullptr, nx, 1, nx, stride, batch, tw, tab, st, po);
        default: return cudaErrorInvalidValue;
        }
    }
    const void *tw = ctw.tw;
    PipeArgs a{nx, 1, nx, stride, batch, 0, op, nullptr};
    switch (op) {
    case COL_FWD: return pipe_n<T, N, true, PIPE_FWD>(in, out, a, tw, tab, st, po);
    case COL_INV: return pipe_n<T, N, true, PIPE_INV_SCALED>(in, out, a, tw, tab, st, po);
    case COL_POISSON: return pipe_n<T, N, true, PIPE_POISSON>(in, out, a, tw, tab, st, po);
    case COL_DIFFUSE: return pipe_n<T, N, true, PIPE_DIFFUSE>(in, out, a, tw, tab, st, po);
    default: return cudaErrorInvalidValue;
    }
}

template <typename T, int N>
cudaError_t wave_cols_n(void *U, void *V, int64_t nx, int64_t stride, int64_t batch,
                        const void *tw, const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    constexpr int W = Shape<N>::TPT >= 256 ? 1 : 256 / Shape<N>::TPT;
    constexpr int THREADS = W * Shape<N>::TPT;
    const size_t smem = WaveSmem<C, N, W>::BYTES;
    auto k = col_wave_kernel<T, N, W>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((nx + W - 1) / W), (unsigned)batch);
    k<<<grid, THREADS, smem, st>>>((C *)U, (C *)V, nx, stride, (const C *)tw, tab);
    return cudaGetLastError();
}

template <typename T, int N, int OP>
cudaError_t small_op_n(const void *in, void *out, int64_t stride, int64_t batch, const void *twx,
                       const void *twy, const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    using L = SmallLayout<C, N, N>;
    auto k = small_solve_kernel<T, N, N, OP>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, L::BYTES);
    if (e != cudaSuccess) return e;
    return launch_pdl(k, dim3((unsigned)batch), dim3(L::THREADS), L::BYTES, st, (const C *)in, (C *)out, stride,
                      (const C *)twx, (const C *)twy, tab);
}

template <typename T, int N>
cudaError_t small_n(const void *in, void *out, int64_t stride, int64_t batch, int op,
                    const void *twx, const void *twy, const OpTables<T> &tab, cudaStream_t st)
{
    switch (op) {
    case COL_FWD: return small_op_n<T, N, COL_FWD>(in, out, stride, batch, twx, twy, tab, st);
    case COL_INV: return small_op_n<T, N, COL_INV>(in, out, stride, batch, twx, twy, tab, st);
    case COL_POISSON: return small_op_n<T, N, COL_POISSON>(in, out, stride, batch, twx, twy, tab, st);
    case COL_DIFFUSE: return small_op_n<T, N, COL_DIFFUSE>(in, out, stride, batch, twx, twy, tab, st);
    default: return cudaErrorInvalidValue;
    }
}

// ---- two-level cluster column pass ------------------------------------------
template <typename T, int P, int Q> struct Col2Cfg {
    using C = typename cplx_t<T>::type;
    static constexpr int EMAX = FFTPDE_COL2_EMAX;
    static constexpr int TIMAX = Col2Geom<C>::W * (Shape<P, EMAX>::TPT > Shape<Q, EMAX>::TPT
                                                   ? Shape<P, EMAX>::TPT : Shape<Q, EMAX>::TPT);
    static constexpr int NT = TIMAX > 128 ? TIMAX : 128;      // a CTA holds at least one item
    using IA = Col2Items<C, Q, NT, EMAX>;
    using IB = Col2Items<C, P, NT, EMAX>;
    static constexpr int CLA = P / IA::SLOTS, CLB = Q / IB::SLOTS;
    static constexpr int CL0 = CLA > CLB ? CLA : CLB;
    static constexpr int CL = CL0 < 1 ? 1 : CL0 > 8 ? 8 : CL0;
    static constexpr size_t SA = (size_t)IA::SLOTS * IA::SLOT_ELEMS * sizeof(C);
    static constexpr size_t SB = (size_t)IB::SLOTS * IB::SLOT_ELEMS * sizeof(C);
    static constexpr size_t SMEM = SA > SB ? SA : SB;
    static constexpr int MINB = NT > 256 ? 1 : NT > 128 ? FFTPDE_COL2_MINB : 4;
};

template <typename T, int P, int Q, int OP>
cudaError_t col2_n(Col2Args<T> g, int64_t batch, const OpTables<T> &tab, cudaStream_t st, const PeerOut &po = PeerOut{})
{
    using Cfg = Col2Cfg<T, P, Q>;
    auto k = col2_kernel<T, P, Q, OP, Cfg::CL, Cfg::NT, Cfg::MINB, Cfg::EMAX>;
    constexpr size_t smem = Cfg::SMEM;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(Cfg::CL * g.nblocks * batch), 1, 1);
    cfg.blockDim = dim3(Cfg::NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Cfg::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled(PDL_COL2) ? 2 : 1;
    e = cudaLaunchKernelEx(&cfg, k, g, tab, po);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int P, int Q>
cudaError_t col2_op(int op, Col2Args<T> g, int64_t batch, const OpTables<T> &tab, cudaStream_t st,
                    const PeerOut &po = PeerOut{})
{
    switch (op) {
    case COL_FWD: return col2_n<T, P, Q, C2_FWD>(g, batch, tab, st);
    case COL_INV: return col2_n<T, P, Q, C2_INV_SCALED>(g, batch, tab, st);
    case COL_POISSON: return col2_n<T, P, Q, C2_POISSON>(g, batch, tab, st, po);
    case COL_DIFFUSE: return col2_n<T, P, Q, C2_DIFFUSE>(g, batch, tab, st, po);
    case 4: return col2_n<T, P, Q, C2_WAVE>(g, batch, tab, st);
    default: return cudaErrorInvalidValue;
    }
}

template <typename T>
cudaError_t launch_col2(int64_t ny, int64_t P, int op, Col2Args<T> g, int64_t batch,
                        const OpTables<T> &tab, cudaStream_t st,
                        const PeerOut &po = PeerOut{})
{
    switch (ny) {
    case 2048: return col2_op<T, 32, 64>(op, g, batch, tab, st, po);
    case 4096: return col2_op<T, 64, 64>(op, g, batch, tab, st, po);
    case 8192: return col2_op<T, 64, 128>(op, g, batch, tab, st, po);
    case 16384: return col2_op<T, 128, 128>(op, g, batch, tab, st, po);
    case 32768: return col2_op<T, 128, 256>(op, g, batch, tab, st, po);
    default: (void)P; return cudaErrorInvalidValue;
    }
}

// ---- long rows: DSMEM four-step on a cluster (row2d.cuh) ------------------------
template <typename T, int P, int Q, int OP>
cudaError_t row2d_n(const void *in, void *out, void *out2, int64_t ny, int64_t stride, int64_t batch,
                    const ColTw &tw, cudaStream_t st, const void *mul = nullptr, const PeerOut &po = PeerOut{})
{
    using C = typename cplx_t<T>::type;
    // 32768-point rows: 16-CTA (non-portable) clusters, half a row's slice per CTA:
    // 12-13% faster than 8-CTA clusters on B200 (tools/exp_row2d.cu); 16384: 8
    constexpr int CL = P * Q >= 32768 ? 16 : 8;
    using G = Row2dGeom<C, P, Q, CL>;
    auto k = row2d_kernel<T, P, Q, CL, OP>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, G::BYTES);
    if (e != cudaSuccess) return e;
    if constexpr (CL > 8) {
        static const cudaError_t np = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (np != cudaSuccess) return np;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(G::NT, 1, 1);
    cfg.dynamicSmemBytes = G::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static std::atomic<int> max_clusters{0};
    int ncl = max_clusters.load();
    if (!ncl) {
        cfg.gridDim = dim3(CL, 1, 1);
        e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
        if (e != cudaSuccess) return e;
        if (ncl < 1) ncl = 1;
        max_clusters.store(ncl);
    }
    cfg.numAttrs = pdl_enabled(PDL_ROW2D) ? 2 : 1;
    const int64_t nrows = ny * batch;
    const int64_t g = std::min<int64_t>(nrows, ncl);          // persistent clusters
    cfg.gridDim = dim3((unsigned)(CL * g), 1, 1);
    e = cudaLaunchKernelEx(&cfg, k, (const C *)in, (C *)out, (C *)out2, nrows, ny, stride, (const C *)tw.twP,
                           (const C *)tw.twQ, (const C *)tw.twN, (const T *)mul, po);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int P, int Q>
cudaError_t row2d_dir(const void *in, void *out, void *out2, int64_t ny, int64_t stride, int64_t batch, int dir,
                      const ColTw &tw, cudaStream_t st, RowMul rm, const PeerOut &po)
{
    if (dir == ROW_DIFF) {
        if (!rm.mul) return cudaErrorInvalidValue;
        return row2d_n<T, P, Q, R2D_DIFF>(in, out, nullptr, ny, stride, batch, tw, st, rm.mul, po);
    }
    if (po.p[0] && dir != ROW_FWD) return cudaErrorInvalidValue;   // peer output: FWD and DIFF only
    if (dir == ROW_INV) return row2d_n<T, P, Q, R2D_INV>(in, out, nullptr, ny, stride, batch, tw, st);
    if (dir == ROW_MID) return row2d_n<T, P, Q, R2D_MID>(in, out, out2, ny, stride, batch, tw, st);
    return row2d_n<T, P, Q, R2D_FWD>(in, out, nullptr, ny, stride, batch, tw, st, nullptr, po);
}

template <typename T>
cudaError_t launch_rows2(int64_t nx, const void *in, void *out, void *out2, int64_t ny, int64_t stride,
                         int64_t batch, int dir, const ColTw &tw, cudaStream_t st, RowMul rm, PeerOut po)
{
    switch (nx) {
    case 16384: return row2d_dir<T, 128, 128>(in, out, out2, ny, stride, batch, dir, tw, st, rm, po);
    case 32768: return row2d_dir<T, 128, 256>(in, out, out2, ny, stride, batch, dir, tw, st, rm, po);
    default: return cudaErrorInvalidValue;
    }
}

// ---- length dispatch -------------------------------------------------------
template <typename T>
cudaError_t launch_rows(int64_t n, const void *in, void *out, void *out2, int64_t ny, int64_t stride,
                        int64_t batch, int dir, const ColTw &tw, cudaStream_t st, RowMul rm, PeerOut po)
{
    switch (n) {
#define X(L) case L: return rows_n<T, L>(in, out, out2, ny, stride, batch, dir, tw, st, rm, po);
        FFTPDE_LEN_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

template <typename T>
cudaError_t launch_cols(int64_t ny, const void *in, void *out, int64_t nx, int64_t stride,
                        int64_t batch, int op, const ColTw &ctw, const OpTables<T> &tab,
                        cudaStream_t st, PeerOut po)
{
    using C = typename cplx_t<T>::type;
    int64_t P = 0, Q = 0;
    col2_split(ny, nx, (int)sizeof(C), P, Q);
    if (P) {
        Col2Args<T> g{(C *)out, nullptr, (const C *)in, nx, stride, nx / Col2Geom<C>::W,
                      (const C *)ctw.twP, (const C *)ctw.twQ, (const C *)ctw.twN};
        return launch_col2<T>(ny, P, op, g, batch, tab, st, po);
    }
    switch (ny) {
#define X(L) case L: return cols_n<T, L>(in, out, nx, stride, batch, op, ctw, tab, st, po);
        FFTPDE_LEN_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

// Wave column pass on cluster pairs with TMA (tmacols.cuh, tools/exp_wave.cu):
// complex128 columns of 2048 / 4096 points, radix 32; cudaErrorNotSupported
// when the driver's tensor-map encoder is unavailable (the caller falls back).
template <typename T, int N>
cudaError_t tma_wave2_n(void *U, void *V, int64_t nx, int64_t stride, int64_t batch, const void *tw,
                        const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    // build parameters for A/B runs (tools/ab_lib.sh): radix 16 with two CTAs per SM
    // measured equal (C3 wave pass 300 vs 298 us), radix 32 with three CTAs per SM
    // (register cap, spills) and radix 16 with one CTA per SM slower (357, 416 us)
#ifndef FFTPDE_WAVE2_EX
#define FFTPDE_WAVE2_EX 32
#endif
#ifndef FFTPDE_WAVE2_MINB
#define FFTPDE_WAVE2_MINB 1
#endif
    constexpr int EX = FFTPDE_WAVE2_EX;
    using L = TmaWave2Smem<C, N, EX>;
    if (batch > (int64_t)1 << 31 || nx * batch > (int64_t)1 << 30) return cudaErrorNotSupported;
    CUtensorMap mu, mv;
    if (!tma_map<T>(mu, U, nx, N, batch, stride, 1, L::BOXR, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B) ||
        !tma_map<T>(mv, V, nx, N, batch, stride, 1, L::BOXR, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
        return cudaErrorNotSupported;
    auto k = tma_wave2_cols_kernel<T, N, EX, FFTPDE_WAVE2_MINB>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, L::BYTES);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * nx * batch), 1, 1);
    cfg.blockDim = dim3(Shape<N, EX>::TPT, 1, 1);
    cfg.dynamicSmemBytes = L::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    int na = 1;
    // A/B knob: FFTPDE_WAVE2_SCHED=1 / 2 asks for the spread / load-balancing cluster scheduling policy
    static const int sched = [] { const char *s = std::getenv("FFTPDE_WAVE2_SCHED"); return s ? std::atoi(s) : 0; }();
    if (sched == 1 || sched == 2) {
        attr[na].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
        attr[na].val.clusterSchedulingPolicyPreference =
            sched == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
        ++na;
    }
    if (pdl_enabled(PDL_COL2)) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    e = cudaLaunchKernelEx(&cfg, k, mu, mv, nx, (const C *)tw, tab, (C *)U, (C *)V, stride);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T>
cudaError_t launch_wave_cols(int64_t ny, void *U, void *V, int64_t nx, int64_t stride,
                             int64_t batch, const ColTw &ctw, const OpTables<T> &tab,
                             cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    if (sizeof(T) == 8 && (ny == 2048 || ny == 4096) && ctw.tw32) {
        const void *tw = tw_for<FFTPDE_WAVE2_EX>(ctw);
        const cudaError_t e = ny == 2048 ? tma_wave2_n<T, 2048>(U, V, nx, stride, batch, tw, tab, st)
                                         : tma_wave2_n<T, 4096>(U, V, nx, stride, batch, tw, tab, st);
        if (e != cudaErrorNotSupported) return e;
    }
    int64_t P = 0, Q = 0;
    col2_split(ny, nx, (int)sizeof(C), P, Q);
    if (P) {
        Col2Args<T> g{(C *)U, (C *)V, (const C *)U, nx, stride, nx / Col2Geom<C>::W,
                      (const C *)ctw.twP, (const C *)ctw.twQ, (const C *)ctw.twN};
        return launch_col2<T>(ny, P, 4, g, batch, tab, st);
    }
    const void *tw = ctw.tw;
    switch (ny) {
#define X(L) case L: return wave_cols_n<T, L>(U, V, nx, stride, batch, tw, tab, st);
        FFTPDE_LEN_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

template <typename T> bool small_supported(int64_t nx, int64_t ny)
{
    return nx == ny && (nx == 16 || nx == 32 || nx == 64);
}

template <typename T>
cudaError_t launch_small(int64_t nx, int64_t ny, const void *in, void *out, int64_t stride,
                         int64_t batch, int op, const void *twx, const void *twy,
                         const OpTables<T> &tab, cudaStream_t st)
{
    if (nx != ny) return cudaErrorInvalidValue;
    switch (nx) {
    case 16: return small_n<T, 16>(in, out, stride, batch, op, twx, twy, tab, st);
    case 32: return small_n<T, 32>(in, out, stride, batch, op, twx, twy, tab, st);
    case 64: return small_n<T, 64>(in, out, stride, batch, op, twx, twy, tab, st);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace fftpde
