// rowt16.cuh -- the transposing 32768-point row diffusion pass (rowt.cuh) with
// 16 points per thread: 512 threads per CTA, one CTA per SM, 8-CTA clusters.
//
// Same mathematics as rowt.cuh (R26, R27; solCalorFourier,
// PAPER.md:378-386; the row / column split of PAPER.md:262-273):
//   pass 1: t = (D_x u)^T,  pass 2: u = (D_y' t)^T,
// one row of N = P Q = 2048 x 16 points, n = n1 + P n2, k = k1 + Q k2:
//   X[k1 + Q k2] = sum_{n1} w_P^{n1 k2} w_N^{n1 k1} sum_{n2} x[n1 + P n2] w_Q^{n2 k1}.
// A cluster of 8 CTAs owns RP = 2 rows (1 MiB) at a time:
//   phase A  (thread = (rho, n1), 512 per CTA): 16-point DFT over n2 in
//            registers, times w_N^{n1 k1} (per-CTA shared-memory slice), pushed
//            by st.async to the owner of item (rho, k1) (4 items per CTA);
//   phase B  (128 threads = item (rho, k1)): the 2048-point Stockham transform
//            (fft_core.cuh, radix 16 x 16 x 8, exchanges in the item's own
//            receive region), times the row factor, the inverse, pushed back;
//   phase A' : times w_N^{-n1 k1}, inverse 16-point DFT, transposed store of
//            32-byte sectors (the pair's two rows are adjacent in the output).
// Sixteen warps per SM (against 4-8 with 32 points per thread) hide the FP64 and
// shared-memory latencies of the butterflies; 8-CTA clusters tile the 148 SMs
// evenly (18 clusters), where 16-CTA clusters left 76 SMs with two CTAs.
#pragma once
#include "fft_core.cuh"
#include "row2d.cuh"
#include "rowt.cuh"

namespace fftpde {

template <int NTH> struct NamedSync {
    int id;
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NTH) : "memory"); }
};

template <int CL_ = 8> struct RowT16Geom {
    static constexpr int N = 32768, P = 2048, Q = 16;
    static constexpr int CL = CL_;                // CTAs per cluster (8: 512 threads, one CTA per SM;
                                                  // 16: 256 threads, two CTAs per SM)
    static constexpr int MINB = CL >= 16 ? 2 : 1;
    static constexpr int RP = 2;                  // rows per cluster iteration
    static constexpr int NT = RP * P / CL;        // 512 threads = phase-A items per CTA
    static constexpr int JA = P / CL;             // 256 values of n1 per CTA
    static constexpr int IB = RP * Q / CL;        // 4 phase-B items per CTA
    static constexpr int TI = P / Q;              // 128 threads per phase-B item
    using SP = Shape<P, 16>;
    static constexpr int RITEM = SP::PADDED;      // 2176: one item's receive + exchange region
    static constexpr int R_ELEMS = IB * RITEM;    // 8704 >= NT * Q (phase A' receive layout [k1][tid])
    static constexpr int TW_ELEMS = Q * JA;       // the CTA's inter-phase twiddles [k1][j]
    static constexpr size_t BYTES = (size_t)(R_ELEMS + TW_ELEMS) * 16 + 16;   // + mbarrier
    static constexpr uint32_t RX_BYTES = (uint32_t)(NT * Q * 16);              // per exchange
    static constexpr int JB = JA / TI;            // phase-A owners' n1 blocks per phase-B thread stride
    static_assert(R_ELEMS >= NT * Q && IB * TI == NT && SP::TPT == TI && JA >= TI, "layout");
};

// Tables (host, per index, exact integer reduction; fftpde_api.cu build_rowt16_tables):
//   twA [rank][k1][j] = w_N^{(256 rank + j) k1}
//   twP               = the radix-16 stage table of 2048 (fft_core.cuh Shape<2048>)
//   mul [k1][e][t]    = m(k1 + 16 t + 2048 e)          (the row factor incl. 1/N)
template <int CL_>
__global__ void __launch_bounds__(RowT16Geom<CL_>::NT, RowT16Geom<CL_>::MINB)
rowt16_kernel(const double2 *__restrict__ in, double2 *__restrict__ out, int64_t nrows,
              const double2 *__restrict__ twA, const double2 *__restrict__ twP, const double *__restrict__ mul)
{
    using G = RowT16Geom<CL_>;
    constexpr int N = G::N, P = G::P, Q = G::Q;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *R = reinterpret_cast<double2 *>(smem_raw);
    double2 *TW = R + G::R_ELEMS;
    const uint32_t mbar = smem_addr(TW + G::TW_ELEMS);
    const uint32_t Rbase = smem_addr(R);
    const uint32_t rank = cl_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // phase A: tid = 32 w + 16 rho + jl, j = 16 w + jl, n1 = 256 rank + j
    const int rho = (lane >> 4) & 1;
    const int j = 16 * warp + (lane & 15);
    const int n1 = G::JA * (int)rank + j;
    // phase B: item ib = tid / 128, t = tid % 128; global item (rhoB, k1B)
    const int ib = tid / G::TI, t = tid % G::TI;
    const int itB = G::IB * (int)rank + ib;
    const int rhoB = itB / Q, k1B = itB % Q;
    const SmemView<double2, G::SP::LOGE, 1> sm{R + ib * G::RITEM};
    const NamedSync<G::TI> isync{1 + ib};

    for (int i = tid; i < G::TW_ELEMS; i += G::NT) TW[i] = twA[(size_t)rank * G::TW_ELEMS + i];
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) mbar_expect_tx(mbar, G::RX_BYTES);
    cl_arrive_relaxed();                                      // mbarriers initialised, buffers free
    uint32_t phase = 0;

    const int64_t npairs = nrows / G::RP;
    const int64_t ncl = gridDim.x / G::CL;
    int64_t pair = blockIdx.x / G::CL;
    pdl_wait();
    auto prefetch_pair = [&](int64_t pr) {      // this CTA's 2 x 16 runs of 256 points (4 KiB) -> L2
        if (pr < npairs && tid < G::RP * Q) {
            const int64_t yy = G::RP * pr + tid / Q;
            prefetch_l2_bulk(in + yy * N + G::JA * (int)rank + P * (tid % Q), G::JA * 16);
        }
    };
    prefetch_pair(pair);
    int it_ = 0;
    (void)it_;
    for (; pair < npairs; pair += ncl, ++it_) {
        RT_MARK(0);
        if (pair + ncl >= npairs) pdl_trigger();
        prefetch_pair(pair + ncl);
        const int64_t y = G::RP * pair + rho;
        double2 v[Q];
        {
            const double2 *src = in + y * N + n1;
#pragma unroll
            for (int e = 0; e < Q; ++e) v[e] = __ldcs(src + P * e);          // x[n1 + P n2], read once
        }
        // ---- phase A: 16-point DFT over n2 -> k1, times w_N^{n1 k1}
        dft_r<Q, false>(v);
        RT_MARK(1);
#pragma unroll
        for (int k = 1; k < Q; ++k) v[k] = cmulw<false>(v[k], TW[k * G::JA + j]);
        RT_MARK(2);
        cl_wait_acquire();                                    // every receive buffer is free
        RT_MARK(3);
#pragma unroll
        for (int k0 = 0; k0 < Q; k0 += G::IB) {               // items (rho, k0 .. k0+3) -> CTA (rho Q + k0) / IB
            const uint32_t to = (uint32_t)((rho * Q + k0) / G::IB);
            const uint32_t dst = mapa_rank(Rbase + (uint32_t)n1 * 16u, to), mb = mapa_rank(mbar, to);
#pragma unroll
            for (int i = 0; i < G::IB; ++i) st_async(dst + (uint32_t)(i * G::RITEM * 16), v[k0 + i], mb);
        }
        // phase B's tables -> L1 while the exchange is in flight (cluster waits invalidate L1):
        // the 2048-point stage table (36 KiB, 288 lines) and the items' factors (4 x 16 KiB)
        if (tid < (G::SP::TW_SIZE * 16 + 127) / 128) prefetch_l1(twP + 8 * tid);
        prefetch_l1(mul + (size_t)k1B * P + 16 * t);
        RT_MARK(4);
        mbar_wait(mbar, phase);
        phase ^= 1u;
        RT_MARK(5);
        // ---- phase B: item (rhoB, k1B), 2048 points n1 = t + 128 e
        double2 u[Q];
        {
            const double2 *Ri = R + ib * G::RITEM;
#pragma unroll
            for (int e = 0; e < Q; ++e) u[e] = Ri[t + G::TI * e];
        }
        isync();                                              // the item's region becomes its exchange buffer
        fft_tw<P, false, 16>(u, sm, t, TwL1<P, double2, 16>{twP, t}, isync);   // u[e] = X[k1B + 16 (t + 128 e)]
        {
            const double *mq = mul + (size_t)k1B * P + t;
#pragma unroll
            for (int e = 0; e < Q; ++e) u[e] = cscale(u[e], __ldg(mq + G::TI * e));
        }
        fft_tw<P, true, 16>(u, sm, t, TwL1<P, double2, 16>{twP, t}, isync);    // u[e] = Y'[n1 = t + 128 e]
        if (tid == 0) mbar_expect_tx(mbar, G::RX_BYTES);
        cl_arrive_after(u[0].x + u[1].x);                     // my reads of R are done (u[0], u[1] depend on all)
        RT_MARK(6);
        cl_wait_acquire();
        RT_MARK(7);
        {   // -> phase-A owner of n1 = t + 128 e: CTA e / JB, j = t + 128 (e % JB), R[k1B][tdst(j)]
            const int tdst0 = 32 * (t >> 4) + 16 * rhoB + (t & 15);
            const uint32_t a0 = Rbase + (uint32_t)(k1B * G::NT + tdst0) * 16u;
#pragma unroll
            for (int e = 0; e < Q; e += G::JB) {
                const uint32_t to = (uint32_t)(e / G::JB);
                const uint32_t dst = mapa_rank(a0, to), mb = mapa_rank(mbar, to);
#pragma unroll
                for (int h = 0; h < G::JB; ++h)               // j + 128 h: tdst + 256 h
                    st_async(dst + (uint32_t)(256 * 16 * h), u[e + h], mb);
            }
        }
        RT_MARK(8);
        mbar_wait(mbar, phase);
        phase ^= 1u;
        RT_MARK(9);
        // ---- phase A': times w_N^{-n1 k1}, inverse 16-point DFT over k1 -> n2, transposed store
#pragma unroll
        for (int k = 0; k < Q; ++k) v[k] = R[k * G::NT + tid];
#pragma unroll
        for (int k = 1; k < Q; ++k) v[k] = cmulw<true>(v[k], TW[k * G::JA + j]);
        dft_r<Q, true>(v);
        if (tid == 0) mbar_expect_tx(mbar, G::RX_BYTES);
        cl_arrive_after(v[0].x);                              // R is free for the next pair
        RT_MARK(10);
        {
            double2 *dst = out + (int64_t)n1 * nrows + y;
#pragma unroll
            for (int e = 0; e < Q; ++e) __stcs(dst + (int64_t)P * e * nrows, v[e]);
        }
    }
    cl_wait_acquire();   // balances the last arrive; no CTA leaves while others may write its smem
}

} // namespace fftpde
