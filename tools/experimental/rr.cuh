// rr.cuh -- register-resident, prefetching line pass for long lines (sm_100a).
//
// The tile being transformed (W lines of N points, E = 16 points per thread)
// lives in registers: a 4096-point complex128 line pair is 128 KiB, half of
// the SM's 256 KiB register file.  Shared memory then only needs
//   * a prefetch buffer P (W*N elements) that receives the NEXT tile
//     (cp.async, 16 B per element) while this one is transformed, and
//   * a HALF-size exchange buffer X (W*(N/2 + pad)): every Stockham exchange
//     runs in two rounds, one per half of the index range.  In round r the
//     threads t < TPT/2 (r = 0) or t >= TPT/2 (r = 1) write their whole
//     butterfly block, which lies in that half because 16*Ns <= N/2, and every
//     thread reads its elements m in [8r, 8r+8), i.e. indices t + TPT m of that
//     half.
// so one CTA per SM keeps one tile computing and one loading, which the
// smem-staged pipe_kernel (2 full buffers) cannot do for 64 KiB lines.
//
// Per line: forward transform along the line (eq:DFT sign
// +), optionally the k-space operator of the column pass and the inverse
// transform; MID (rows) = the inverse transform of step s
// stored as the physical field, then the forward transform of step s+1.
#pragma once
#include "../../paper_2412_12308_b200/csrc/fft_core.cuh"
#include "../../paper_2412_12308_b200/csrc/line.cuh"
#include "../../paper_2412_12308_b200/csrc/pipe.cuh"

namespace fftpde {

template <typename C, int N, int W, bool COLS> struct RRSmem {
    using S = Shape<N, 16>;
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int HALF = N / 2;
    static constexpr int XRAW = HALF + (HALF >> S::LOGE);
    static constexpr int SX = (!COLS || W == 1) ? XRAW : ((XRAW + LPP - 1) / LPP) * LPP + (W >= LPP ? 1 : LPP / W);
    static constexpr size_t P_ELEMS = (size_t)W * N;
    static constexpr size_t X_ELEMS = (size_t)W * SX;
    static constexpr size_t BYTES = (P_ELEMS + X_ELEMS) * sizeof(C);
};

// Transform of v[e] = x[t + TPT e] through the half-size exchange buffer.
template <int N, bool INV, typename C, typename View, typename Tw, typename Sync>
__device__ __forceinline__ void fft_half(C (&v)[16], const View &sm, int t, const Tw &tw, Sync sync)
{
    using S = Shape<N, 16>;
    constexpr int E = 16, TPT = S::TPT, HALF = N / 2;
    static_assert(S::E == 16, "E = 16");
    int Ns = 1;
#pragma unroll
    for (int s = 0; s < S::STAGES; ++s) {
        const int k = t & (Ns - 1);
        if (s > 0) {
#pragma unroll
            for (int m = 1; m < E; ++m) v[m] = cmulw<INV>(v[m], tw.mid(s, m));
        }
        dft_r<E, INV>(v);
        const bool lo = t < TPT / 2;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (lo == (r == 0)) {
                C *wp = sm.ptr((t - k) * E + k - r * HALF);
#pragma unroll
                for (int m = 0; m < E; ++m) wp[View::off(m * Ns)] = v[m];
            }
            sync();
            const C *rp = sm.ptr(t);
#pragma unroll
            for (int m = 0; m < E / 2; ++m) v[r * 8 + m] = rp[View::off(m * TPT)];
            sync();
        }
        Ns *= E;
    }
    constexpr int R = S::R_LAST, Q = E / R;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        C u[R];
#pragma unroll
        for (int m = 0; m < R; ++m) u[m] = v[q + m * Q];
        if (S::NS_LAST > 1) {
#pragma unroll
            for (int m = 1; m < R; ++m) u[m] = cmulw<INV>(u[m], tw.last(q, m));
        }
        dft_r<R, INV>(u);
#pragma unroll
        for (int m = 0; m < R; ++m) v[q + m * Q] = u[m];
    }
}

template <typename T, int N, int W, bool COLS, int OP, int MINB = 1>
__global__ void __launch_bounds__(W * (N / 16), MINB)
rr_kernel(const typename cplx_t<T>::type *__restrict__ in, typename cplx_t<T>::type *out, LineArgs a,
          int64_t ntiles, const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N, 16>;
    using L = RRSmem<C, N, W, COLS>;
    constexpr int E = 16, TPT = S::TPT;
    static_assert(16 * (S::NS_LAST) <= 16 * N, "shape");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *P = reinterpret_cast<C *>(smem_raw);
    C *X = P + L::P_ELEMS;

    const int tid = threadIdx.x;
    const int c = COLS ? tid % W : tid / TPT;
    const int t = COLS ? tid / W : tid % TPT;
    const int64_t estep = (int64_t)TPT * a.elem_stride;
    constexpr bool INV1 = OP == LN_INV || OP == LN_INV_SCALED || OP == LN_MID;
    const LnSync<TPT, COLS> sync{1 + c};
    SmemView<C, S::LOGE, 1> sm{X + c * L::SX};
    const TwL1<N, C, 16> twp{tw, t};
    // P slot of element e of this thread's line
    auto pidx = [&](int e) -> int { return COLS ? (t + TPT * e) * W + c : c * N + t + TPT * e; };
    auto line_of = [&](int64_t tile, int64_t &b) -> int64_t {
        b = tile / a.groups;
        return (tile - b * a.groups) * W + c;
    };
    auto issue = [&](int64_t tile) {
        int64_t b;
        const int64_t line = line_of(tile, b);
        if (line < a.nlines) {
            const C *src = in + b * a.batch_stride + line * a.line_stride + (int64_t)t * a.elem_stride;
#pragma unroll
            for (int e = 0; e < E; ++e) cp_async_n<sizeof(C)>(P + pidx(e), src + e * estep);
        }
        cp_async_commit();
    };

    int64_t tile = blockIdx.x;
    if (tile < ntiles) issue(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        cp_async_wait<0>();
        __syncthreads();                                   // tile `tile` is in P (all threads' copies)
        C v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = P[pidx(e)];
        __syncthreads();                                   // P is free: prefetch the next tile
        const int64_t nxt = tile + gridDim.x;
        if (nxt < ntiles) issue(nxt);
        int64_t b;
        const int64_t line = line_of(tile, b);
        const bool active = line < a.nlines;
        const int64_t base = b * a.batch_stride + (active ? line : 0) * a.line_stride + (int64_t)t * a.elem_stride;

        if constexpr (OP == LN_INV_SCALED) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], tab.scale);
        }
        fft_half<N, INV1>(v, sm, t, twp, sync);
        if constexpr (OP == LN_POISSON || OP == LN_DIFFUSE) {
            asm volatile("" ::: "memory");
            if constexpr (OP == LN_POISSON) {
                const T kxa = tab.kx2[active ? line : 0];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const T k2 = kxa + __ldg(&tab.ky2[t + TPT * e]);
                    v[e] = cscale(v[e], k2 == (T)0 ? (T)0 : -tab.scale / k2);   // -1/|k|^2, k = 0 zeroed
                }
            } else {
                const T exa = tab.ex[active ? line : 0];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cscale(v[e], exa * __ldg(&tab.ey[t + TPT * e]));   // exp(-D|k|^2 dt)/(nx ny)
            }
            fft_half<N, true>(v, sm, t, twp, sync);
        }
        if constexpr (OP == LN_MID) {
            if (active) {
                C *dst = opaque_ptr(reinterpret_cast<C *>(a.out2) + base);
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
            }
            fft_half<N, false>(v, sm, t, twp, sync);
        }
        if (active) {
            C *dst = opaque_ptr(out + base);
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
        }
    }
    cp_async_wait<0>();
}

} // namespace fftpde
