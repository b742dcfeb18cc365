// line.cuh -- occupancy-oriented line pass (rows or short columns), sm_100a.
//
// One CTA transforms W lines (rows along x, or W adjacent columns along y)
// and exits; the block scheduler keeps several CTAs resident per SM, so the
// loads of one CTA overlap the butterflies of the others (no staging buffers:
// each thread loads its E elements straight into registers, 128-bit loads,
// coalesced along the row, or W*sizeof(C)-byte row segments for columns).
// Shared memory holds only the exchange buffer of each line, so a 1024-point
// complex128 line costs 18 KiB and 3-4 CTAs fit per SM.
//
// Per line: a transform along the line (eq:DFT sign +,
// or the conjugate kernel of PAPER.md:151-153), optionally the k-space
// operator of the column pass and the inverse transform; for rows, MID is the
// inverse transform of step s (stored: the materialised physical field) and
// the forward transform of step s+1, one HBM read for both.
#pragma once
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

enum LineOp { LN_FWD = 0, LN_INV_SCALED = 1, LN_POISSON = 2, LN_DIFFUSE = 3, LN_INV = 4, LN_MID = 5, LN_WAVE = 6 };

struct LineArgs {
    int64_t nlines;       // lines per grid (rows: ny, columns: nx)
    int64_t line_stride;  // elements between consecutive lines (rows: nx, columns: 1)
    int64_t elem_stride;  // elements between consecutive points of a line (rows: 1, columns: nx)
    int64_t batch_stride; // elements between grids
    int64_t groups;       // ceil(nlines / W)
    void *out2;           // LN_MID: physical-field output; LN_WAVE: second field (in place)
};

// Exchange-buffer pitch (elements) of one line.  Columns interleave W lines
// across the lanes of a warp (lane -> column tid % W): the pitch is offset so
// the W lines of one shared-memory phase start in distinct banks.
template <typename C, int N, int E, int W, bool COLS> struct LineSmem {
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int RAW = Shape<N, E>::PADDED;
    static constexpr int S = (!COLS || W == 1) ? RAW : ((RAW + LPP - 1) / LPP) * LPP + (W >= LPP ? 1 : LPP / W);
    static constexpr int NF = 1;
    static constexpr size_t BYTES = (size_t)W * S * sizeof(C);
};

template <int TPT, bool COLS> struct LnSync {
    int id;
    __device__ __forceinline__ void operator()() const
    {
        if constexpr (COLS) __syncthreads();
        else if constexpr (TPT <= 32) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(TPT) : "memory");
    }
};

template <typename T, int N, int E, int W, bool COLS, int OP, int MINB>
__global__ void __launch_bounds__(W * (N / E), MINB)
line_kernel(const typename cplx_t<T>::type *__restrict__ in, typename cplx_t<T>::type *out, LineArgs a,
            const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab, PeerOut po)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N, E>;
    using L = LineSmem<C, N, E, W, COLS>;
    constexpr int TPT = S::TPT;
    static_assert(S::E == E, "E must not exceed N");
    static_assert(COLS || TPT <= 32 || W <= 15, "one named barrier per row");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);

    const int tid = threadIdx.x;
    const int c = COLS ? tid % W : tid / TPT;
    const int t = COLS ? tid / W : tid % TPT;
    const int64_t tile = blockIdx.x;
    const int64_t b = tile / a.groups;
    const int64_t line = (tile - b * a.groups) * W + c;
    const bool active = line < a.nlines;
    const int64_t base = b * a.batch_stride + (active ? line : 0) * a.line_stride + (int64_t)t * a.elem_stride;
    const int64_t estep = (int64_t)TPT * a.elem_stride;
    constexpr bool INV1 = OP == LN_INV || OP == LN_INV_SCALED || OP == LN_MID;
    const LnSync<TPT, COLS> sync{1 + c};
    SmemView<C, S::LOGE, 1> sm{smem + c * L::S};
#ifndef FFTPDE_LINE_SPLIT
#define FFTPDE_LINE_SPLIT 1     // complex128 radix-32 lines: split twiddles (C2 4.244 -> 4.214 ms per solve)
#endif
    using TwP = std::conditional_t<FFTPDE_LINE_SPLIT != 0 && sizeof(T) == 8, TwL1Split<N, C, E>, TwL1<N, C, E>>;
    TwP twp;
    twp.tw = tw;
    twp.t = t;
    pdl_wait();
    pdl_trigger();

    C v[E];
    if (active) {
        const C *src = in + base;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = src[e * estep];
    } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = C{0, 0};
    }
    if constexpr (OP == LN_INV_SCALED) {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = cscale(v[e], tab.scale);
    }
    fft_tw<N, INV1, E>(v, sm, t, twp, sync);
    if constexpr (OP == LN_POISSON || OP == LN_DIFFUSE) {
        // k-space operator at (a, b): the line is column a, element e is row b
        if constexpr (OP == LN_POISSON) {
            const T kxa = tab.kx2[active ? line : 0];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const T k2 = kxa + __ldg(&tab.ky2[t + TPT * e]);
                v[e] = cscale(v[e], poisson_mul(k2, tab.scale));   // -1/|k|^2, k = 0 zeroed
            }
        } else if (tab.ey2d) {                      // four-step B pass: factor of line class cls
            const int64_t cls = COLS ? b : (active ? line : 0) % tab.ey2d_mod;
            const T *m = tab.ey2d + cls * N;
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + t + TPT * e));
        } else {
            const T exa = tab.ex[active ? line : 0];
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], exa * __ldg(&tab.ey[t + TPT * e]));   // exp(-D|k|^2 dt)/(nx ny)
        }
        fft_tw<N, true, E>(v, sm, t, twp, sync);
    }
    if constexpr (OP == LN_MID) {
        if (active) {
            C *dst = opaque_ptr(reinterpret_cast<C *>(a.out2) + base);
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
        }
        fft_tw<N, false, E>(v, sm, t, twp, sync);
    }
    if (active) {
        if (po.p[0]) {                              // scattered into the peers' slabs
#pragma unroll
            for (int e = 0; e < E; ++e) {
                C *d = COLS ? peer_col_dst<C>(po, t + TPT * e, line) : peer_row_dst<C>(po, line, t + TPT * e);
                *opaque_ptr(d) = v[e];
            }
            return;
        }
        C *dst = opaque_ptr(out + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
    }
}

} // namespace fftpde
