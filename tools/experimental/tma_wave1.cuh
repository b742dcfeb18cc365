// tma_wave1.cuh -- experiment only (tools/exp_wave.cu): one CTA per column holding
// both wave fields; superseded by the cluster-pair tma_wave2_cols_kernel.
#pragma once
#include "../../paper_2412_12308_b200/csrc/tmacols.cuh"

namespace fftpde {

// ---------------------------------------------------------------------------
// Wave column pass with TMA (C3: 4096-point complex128 columns of two fields).
// One CTA per column a: U[:, a] and V[:, a] are brought in by the tensor
// memory accelerator as boxes of 256 rows x 16 bytes (one element per row; the
// neighbouring columns' CTAs use the other halves of the same sectors, which L2
// serves), transformed along y, advanced by the exact oscillator update
// (eq:OmegaZero/NonZero; 1/(nx ny) folded into the tables),
// inverse-transformed and stored back the same way.  Half of the threads own U,
// half V; the update pairs them through shared memory.  No four-step split, no
// L2-resident intermediate: one HBM read and one write of each field.
template <typename C, int N, int EX> struct TmaWaveSmem {
    static constexpr int RAW = Shape<N, EX>::PADDED;
    static constexpr size_t LINE = ((size_t)RAW * sizeof(C) + 127) / 128 * 128;
    static constexpr int BOXR = N < 256 ? N : 256;
    static constexpr int NBOX = N / BOXR;
    static constexpr size_t BYTES = 2 * LINE + 128 + 16;
};

template <typename T, int N, int EX>
__global__ void __launch_bounds__(2 * Shape<N, EX>::TPT, 1)
tma_wave_cols_kernel(const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mv, int64_t ncols,
                     const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N, EX>;
    using L = TmaWaveSmem<C, N, EX>;
    constexpr int E = S::E, TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((128u - (tma_smem(smem_raw) & 127u)) & 127u);
    const uint32_t mbar = tma_smem(base + 2 * L::LINE);
    const int tid = threadIdx.x;
    const int f = tid / TPT, t = tid % TPT;               // field (0: U, 1: V), thread of its line
    const LineSync<TPT> lsync{1 + f};
    const int64_t bz = blockIdx.x / ncols;
    const int64_t a = blockIdx.x - bz * ncols;            // column (x wavenumber index)
    C *line = reinterpret_cast<C *>(base + f * L::LINE);
    if (tid == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mu) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mv) : "memory");
    }
    __syncthreads();
    pdl_wait();
    if (tid == 0) {
        tma_mbar_expect(mbar, (uint32_t)(2 * N * sizeof(C)));
        const uint32_t du = tma_smem(base), dv = tma_smem(base + L::LINE);
#pragma unroll
        for (int k = 0; k < L::NBOX; ++k) {
            tma_load3(du + k * L::BOXR * (int)sizeof(C), &mu, (int)(2 * a), k * L::BOXR, (int)bz, mbar);
            tma_load3(dv + k * L::BOXR * (int)sizeof(C), &mv, (int)(2 * a), k * L::BOXR, (int)bz, mbar);
        }
    }
    pdl_trigger();
    tma_mbar_wait(mbar, 0);
    C v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = line[t + TPT * e];
    lsync();
    SmemView<C, S::LOGE, 1> sm{line};
    const TwL1<N, C, EX> twp{tw, t};
    fft_tw<N, false, EX>(v, sm, t, twp, lsync);
#pragma unroll
    for (int e = 0; e < E; ++e) line[t + TPT * e] = v[e];
    __syncthreads();                                     // both spectra in shared memory
    {
        const C *other = reinterpret_cast<const C *>(base + (1 - f) * L::LINE);
        const int64_t qa = a <= tab.nfold - a ? a : tab.nfold - a;   // |fold(a)|
        const T *pC = tab.wC + qa * tab.qpitch, *pS = (f ? tab.wS2 : tab.wS1) + qa * tab.qpitch;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int b = t + TPT * e;
            const int qb = b <= N - b ? b : N - b;
            const T cc = __ldg(pC + qb), ss = __ldg(pS + qb);
            const C o = other[b];
            // U: C U + S1 V;  V: S2 U + C V
            v[e] = C{cc * v[e].x + ss * o.x, cc * v[e].y + ss * o.y};
        }
    }
    __syncthreads();                                     // the partner's spectrum has been read
    fft_tw<N, true, EX>(v, sm, t, twp, lsync);
#pragma unroll
    for (int e = 0; e < E; ++e) line[t + TPT * e] = v[e];
    tma_fence_smem();
    __syncthreads();
    if (tid == 0) {
        const uint32_t su = tma_smem(base), sv = tma_smem(base + L::LINE);
#pragma unroll
        for (int k = 0; k < L::NBOX; ++k) {
            tma_store3(&mu, (int)(2 * a), k * L::BOXR, (int)bz, su + k * L::BOXR * (int)sizeof(C));
            tma_store3(&mv, (int)(2 * a), k * L::BOXR, (int)bz, sv + k * L::BOXR * (int)sizeof(C));
        }
        tma_commit();
        tma_wait_read0();                                // smem must outlive the bulk reads
    }
}

} // namespace fftpde
