// wave_line.cuh -- experiment only (tools/exp_line.cu, exp_e32.cu): the wave column
// pass as a non-persistent line kernel; the library uses tma_wave2_cols_kernel.
#pragma once
#include "../../paper_2412_12308_b200/csrc/line.cuh"

namespace fftpde {

// Wave column pass for short columns: both fields of W columns, forward along
// y, the exact oscillator update (eq:OmegaZero/NonZero PAPER.md:459-471, the
// 1/(nx ny) folded into the tables), inverse along y; in place.  The first
// field's spectrum waits in a shared-memory stash while the second is
// transformed, so a thread holds E values, not 2E.
template <typename C, int N, int E, int W> struct WaveLineSmem {
    using X = LineSmem<C, N, E, W, true>;
    static constexpr size_t XBYTES = X::BYTES;
    static constexpr size_t BYTES = XBYTES + (size_t)W * N * sizeof(C);
};

template <typename T, int N, int E, int W, int MINB>
__global__ void __launch_bounds__(W * (N / E), MINB)
wave_line_kernel(typename cplx_t<T>::type *U, typename cplx_t<T>::type *V, LineArgs a,
                 const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N, E>;
    using L = LineSmem<C, N, E, W, true>;
    constexpr int TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);
    C *stash = reinterpret_cast<C *>(smem_raw + WaveLineSmem<C, N, E, W>::XBYTES);

    const int tid = threadIdx.x;
    const int c = tid % W, t = tid / W;
    const int64_t tile = blockIdx.x;
    const int64_t b = tile / a.groups;
    const int64_t col = (tile - b * a.groups) * W + c;
    const bool active = col < a.nlines;
    const int64_t base = b * a.batch_stride + (active ? col : 0) + (int64_t)t * a.elem_stride;
    const int64_t estep = (int64_t)TPT * a.elem_stride;
    const LnSync<TPT, true> sync{0};
    SmemView<C, S::LOGE, 1> sm{smem + c * L::S};
    const TwL1<N, C, E> twp{tw, t};
    auto slot = [&](int e) -> C & { return stash[(t + TPT * e) * W + c]; };
    pdl_wait();
    pdl_trigger();

    C v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? U[base + e * estep] : C{0, 0};
    fft_tw<N, false, E>(v, sm, t, twp, sync);
#pragma unroll
    for (int e = 0; e < E; ++e) slot(e) = v[e];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? V[base + e * estep] : C{0, 0};
    fft_tw<N, false, E>(v, sm, t, twp, sync);
    const int64_t qa = active ? (col <= tab.nfold - col ? col : tab.nfold - col) : 0;
    const T *pC = tab.wC + qa * tab.qpitch, *pS1 = tab.wS1 + qa * tab.qpitch, *pS2 = tab.wS2 + qa * tab.qpitch;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int bb = t + TPT * e;
        const int qb = bb <= N - bb ? bb : N - bb;
        const T cc = __ldg(pC + qb), s1 = __ldg(pS1 + qb), s2 = __ldg(pS2 + qb);
        const C uh = slot(e), vh = v[e];
        slot(e) = C{cc * uh.x + s1 * vh.x, cc * uh.y + s1 * vh.y};   // C U + S1 V
        v[e] = C{s2 * uh.x + cc * vh.x, s2 * uh.y + cc * vh.y};      // S2 U + C V
    }
    fft_tw<N, true, E>(v, sm, t, twp, sync);
    if (active) {
        C *dst = opaque_ptr(V + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = slot(e);
    fft_tw<N, true, E>(v, sm, t, twp, sync);
    if (active) {
        C *dst = opaque_ptr(U + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
    }
}

} // namespace fftpde
