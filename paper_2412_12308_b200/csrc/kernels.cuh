// kernels.cuh -- wave column pass and single-CTA small-grid solve (sm_100a).
//
// The row passes and the Poisson/diffusion column pass are pipe_kernel
// (pipe.cuh).  Here:
//   col_wave_kernel   : both wave fields of W columns: forward along y, the exact
//                       oscillator update (eq:OmegaZero/NonZero, PAPER.md:459-471,
//                       1/(nx ny) folded into its tables), inverse along y
//   small_solve_kernel: a whole small grid resident in one CTA's shared memory,
//                       rows -> columns -> operator -> inverse columns -> inverse
//                       rows: one HBM round trip (C1).
#pragma once
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

// Smem pitch (in complex elements) of one column buffer so that W columns
// accessed by the lanes of one shared-memory phase hit distinct banks:
// a phase is 128 B = LPP elements; column c starts at c*S with S = LPP/W mod LPP.
template <typename C, int N, int W> struct ColSmem {
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int RAW = Shape<N>::PADDED;
    static constexpr int S = W == 1 ? RAW : ((RAW + LPP - 1) / LPP) * LPP + (W >= LPP ? 1 : LPP / W);
    static constexpr size_t BYTES = (size_t)W * S * sizeof(C);
};

// Column pass for the wave step: both fields (U, V) of W columns, forward along
// y, the exact oscillator update, inverse along y.  In place.  One field is in
// registers at a time; the other's spectrum waits in a shared-memory stash
// (thread-private slots), so a thread holds 16 complex values, not 32.
template <typename C, int N, int W> struct WaveSmem {
    using CS = ColSmem<C, N, W>;
    static constexpr size_t XBYTES = CS::BYTES;                 // exchange buffers
    static constexpr size_t BYTES = XBYTES + (size_t)W * N * sizeof(C);   // + stash
};

template <typename T, int N, int W>
__global__ void __launch_bounds__(W * Shape<N>::TPT)
col_wave_kernel(typename cplx_t<T>::type *U, typename cplx_t<T>::type *V,
                int64_t nx, int64_t stride,
                const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N>;
    using CS = ColSmem<C, N, W>;
    constexpr int E = S::E, TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);
    C *stash = reinterpret_cast<C *>(smem_raw + WaveSmem<C, N, W>::XBYTES);

    const int c = threadIdx.x % W;
    const int t = threadIdx.x / W;
    const int64_t a = (int64_t)blockIdx.x * W + c;
    const bool active = a < nx;
    const int64_t base = (int64_t)blockIdx.y * stride + (active ? a : 0) + (int64_t)t * nx;
    const int64_t estep = (int64_t)TPT * nx;
    SmemView<C, S::LOGE, 1> sm{smem + c * CS::S};
    // stash slot of element e of this thread: column-interleaved, unit stride across threads
    auto slot = [&](int e) -> C & { return stash[(t + TPT * e) * W + c]; };

    C v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? U[base + e * estep] : C{0, 0};
    fft<N, false>(v, sm, t, tw, SyncCTA{});
#pragma unroll
    for (int e = 0; e < E; ++e) slot(e) = v[e];                        // U^ -> stash
    asm volatile("" ::: "memory");
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? V[base + e * estep] : C{0, 0};
    fft<N, false>(v, sm, t, tw, SyncCTA{});
    asm volatile("" ::: "memory");   // keep the table loads below the transform (register pressure)
    // quadrant index: qa = |fold(a)|, qb = |fold(b)|
    const int64_t qa = active ? (a <= tab.nfold - a ? a : tab.nfold - a) : 0;
    const T *pC = tab.wC + qa * tab.qpitch;
    const T *pS1 = tab.wS1 + qa * tab.qpitch;
    const T *pS2 = tab.wS2 + qa * tab.qpitch;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int b = t + TPT * e;
        const int qb = b <= N - b ? b : N - b;
        const T cc = __ldg(pC + qb), s1 = __ldg(pS1 + qb), s2 = __ldg(pS2 + qb);
        const C uh = slot(e), vh = v[e];
        const C un = {cc * uh.x + s1 * vh.x, cc * uh.y + s1 * vh.y};   // C U + S1 V
        const C vn = {s2 * uh.x + cc * vh.x, s2 * uh.y + cc * vh.y};   // S2 U + C V
        slot(e) = un;
        v[e] = vn;
    }
    fft<N, true>(v, sm, t, tw, SyncCTA{});                               // inverse of V
    if (active) {
        C *dst = opaque_ptr(V + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = slot(e);
    fft<N, true>(v, sm, t, tw, SyncCTA{});                               // inverse of U
    if (active) {
        C *dst = opaque_ptr(U + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
    }
}

// ---------------------------------------------------------------------------
// Single-CTA solve of one small NX x NY grid per CTA (blockIdx.x = batch member),
// the whole grid resident in shared memory: rows -> columns -> operator ->
// inverse columns -> inverse rows, one HBM read and one HBM write.
template <typename C, int NX, int NY> struct SmallLayout {
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int ROWLEN = Shape<NX>::PADDED;
    // row pitch: padded row, then offset so rows sharing a smem phase differ in bank
    static constexpr int PITCH = ((ROWLEN + LPP - 1) / LPP) * LPP + LPP / 2;
    static constexpr int THREADS_R = NY * Shape<NX>::TPT;
    static constexpr int THREADS_C = NX * Shape<NY>::TPT;
    static constexpr int THREADS = THREADS_R > THREADS_C ? THREADS_R : THREADS_C;
    static constexpr int TWX = Shape<NX>::TW_SIZE > 0 ? Shape<NX>::TW_SIZE : 1;
    static constexpr int TWY = Shape<NY>::TW_SIZE > 0 ? Shape<NY>::TW_SIZE : 1;
    static constexpr size_t GRID = (size_t)NY * PITCH * sizeof(C);
    // grid + twiddle tables of both axes + the two k^2 / diffusion factor tables
    static constexpr size_t BYTES = GRID + (size_t)(TWX + TWY) * sizeof(C) + 2 * (size_t)(NX + NY) * sizeof(C) / 2;
};

template <typename T, int NX, int NY, int OP>
__global__ void __launch_bounds__(SmallLayout<typename cplx_t<T>::type, NX, NY>::THREADS)
small_solve_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out,
                   int64_t stride, const typename cplx_t<T>::type *__restrict__ twx,
                   const typename cplx_t<T>::type *__restrict__ twy, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using L = SmallLayout<C, NX, NY>;
    using SX = Shape<NX>;
    using SY = Shape<NY>;
    static_assert(SX::E == SY::E, "small_solve needs one thread layout for rows and columns");
    constexpr bool INV = OP == COL_INV;                 // plain inverse transform
    constexpr bool SOLVE = OP == COL_POISSON || OP == COL_DIFFUSE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *g = reinterpret_cast<C *>(smem_raw);
    // tables staged in shared memory once: no L2 round trip on the per-stage critical path
    C *stx = reinterpret_cast<C *>(smem_raw + L::GRID);
    C *sty = stx + L::TWX;
    T *sa = reinterpret_cast<T *>(sty + L::TWY);        // kx2 or ex  [NX]
    T *sb = sa + NX;                                     // ky2 or ey  [NY]
    const int64_t off = (int64_t)blockIdx.x * stride;
    const int tid = threadIdx.x;
    for (int i = tid; i < SX::TW_SIZE; i += L::THREADS) stx[i] = twx[i];
    for (int i = tid; i < SY::TW_SIZE; i += L::THREADS) sty[i] = twy[i];
    if constexpr (SOLVE) {
        const T *ta = OP == COL_POISSON ? tab.kx2 : tab.ex;
        const T *tb = OP == COL_POISSON ? tab.ky2 : tab.ey;
        for (int i = tid; i < NX; i += L::THREADS) sa[i] = ta[i];
        for (int i = tid; i < NY; i += L::THREADS) sb[i] = tb[i];
    }
    pdl_wait();
    pdl_trigger();

    // ---- phase 1: row transforms (forward, or inverse for COL_INV)
    {
        const int row = tid / SX::TPT, t = tid % SX::TPT;
        C v[SX::E];
#pragma unroll
        for (int e = 0; e < SX::E; ++e) v[e] = in[off + (int64_t)row * NX + t + SX::TPT * e];
        __syncthreads();                                 // tables staged
        SmemView<C, SX::LOGE, 1> sm{g + row * L::PITCH};
        fft_tw<NX, INV>(v, sm, t, TwSmem<NX, C>{stx, t}, SyncCTA{});
#pragma unroll
        for (int e = 0; e < SX::E; ++e) sm.at(t + SX::TPT * e) = v[e];
        __syncthreads();
    }
    // ---- phase 2: column transforms (+ operator + inverse columns)
    {
        const int col = tid % NX, t = tid / NX;
        SmemView<C, 30, L::PITCH> sm{g + padidx(col, SX::LOGE)};
        C v[SY::E];
#pragma unroll
        for (int e = 0; e < SY::E; ++e) v[e] = sm.at(t + SY::TPT * e);
        __syncthreads();
        if constexpr (INV) {
#pragma unroll
            for (int e = 0; e < SY::E; ++e) v[e] = cscale(v[e], tab.scale);
        }
        const TwSmem<NY, C> twc{sty, t};
        fft_tw<NY, INV>(v, sm, t, twc, SyncCTA{});
        if constexpr (SOLVE) {
#pragma unroll
            for (int e = 0; e < SY::E; ++e) {
                const int b = t + SY::TPT * e;
                T m;
                if constexpr (OP == COL_POISSON) {
                    const T k2 = sa[col] + sb[b];
                    m = poisson_mul(k2, tab.scale);    // -1/|k|^2, k = 0 zeroed
                } else {
                    m = sa[col] * sb[b];                          // exp(-D|k|^2 dt)/(nx ny)
                }
                v[e] = cscale(v[e], m);
            }
            fft_tw<NY, true>(v, sm, t, twc, SyncCTA{});
        }
#pragma unroll
        for (int e = 0; e < SY::E; ++e) sm.at(t + SY::TPT * e) = v[e];
        __syncthreads();
    }
    if constexpr (!SOLVE) {   // plain transform: write the grid
        for (int i = tid; i < NX * NY; i += L::THREADS) {
            const int row = i / NX, j = i % NX;
            out[off + i] = g[row * L::PITCH + padidx(j, SX::LOGE)];
        }
        return;
    } else {
        // ---- phase 3: inverse row transforms
        const int row = tid / SX::TPT, t = tid % SX::TPT;
        SmemView<C, SX::LOGE, 1> sm{g + row * L::PITCH};
        C v[SX::E];
#pragma unroll
        for (int e = 0; e < SX::E; ++e) v[e] = sm.at(t + SX::TPT * e);
        __syncthreads();
        fft_tw<NX, true>(v, sm, t, TwSmem<NX, C>{stx, t}, SyncCTA{});
#pragma unroll
        for (int e = 0; e < SX::E; ++e) out[off + (int64_t)row * NX + t + SX::TPT * e] = v[e];
    }
}

} // namespace fftpde
