// rowt.cuh -- 1D diffusion of 32768-point complex128 rows with a TRANSPOSED
// store, on a 16-CTA thread-block cluster (sm_100a).  Used for both axes of the
// separable C5 diffusion step (R26, R27):
//
//   pass 1:  t = ( D_x u )^T      rows of u are x-lines, t[x][y]
//   pass 2:  u = ( D_y' t )^T     rows of t are y-lines, back to u[y][x]
//
// where D_x = F_x^{-1} diag(e^{-D kx^2 dt}/nx) F_x is the 1D diffusion along a
// row (solCalorFourier, with the 2D transform split into its
// row and column halves as in PAPER.md:262-273).  Both passes read rows
// contiguously; the field is materialised in its natural layout after every
// step (R8), and no pass reads a column.
//
// One row of N = P Q = 1024 x 32 points, n = n1 + P n2, k = k1 + Q k2:
//   X[k1 + Q k2] = sum_{n1} w_P^{n1 k2} w_N^{n1 k1} sum_{n2} x[n1 + P n2] w_Q^{n2 k1}
// (eq:DFT, reorganised like the paper's own split of the 2D
// sum).  A cluster owns RP = 2 rows at a time:
//   phase A  (thread = (row rho, n1)):  the 32-point DFT over n2 entirely in
//            registers (no shared-memory exchange), times w_N^{n1 k1} from a
//            per-CTA shared-memory slice; each result is pushed with st.async
//            into the owner of item (rho, k1) (distributed shared memory,
//            completing on the owner's mbarrier);
//   phase B  (warp = item (rho, k1)):   the 1024-point DFT over n1 as 32 x 32
//            in registers with one warp-private transpose through shared
//            memory (__syncwarp only), times the row factor m(k), the inverse
//            1024-point DFT, pushed back to the phase-A owners;
//   phase A' : times w_N^{-n1 k1}, inverse 32-point DFT over k1, and the
//            transposed store out[x][y]: the two rows of the pair are adjacent
//            in the output, so lanes (rho = 0, 1) of the same x write one
//            32-byte sector.
// Two CTAs (128 threads, <= 255 registers) share an SM, so one CTA's loads and
// exchanges overlap the other's FP64 work.
#pragma once
#include "fft_core.cuh"
#include "row2d.cuh"

namespace fftpde {

// barrier.cluster.arrive.relaxed issued only after `dep` has been computed.  The
// receive buffer is released by this arrive: every shared-memory read of it that
// precedes the arrive has been consumed into `dep` (a DFT output depending on all
// of them), so each read has returned its value before the arrive can issue (in-
// order issue waits on the register), and no later remote write can change what
// it returned.  A .release arrive would order the same reads, but ptxas lowers it
// to MEMBAR.ALL.GPU, which also waits for this thread's outstanding global
// stores (r02 ncu: the exchange loop stalled behind it).
__device__ __forceinline__ void cl_arrive_after(double dep)
{
    asm volatile("barrier.cluster.arrive.relaxed.aligned; // %0" ::"d"(dep) : "memory");
}

__device__ __forceinline__ void prefetch_l2_bulk(const void *g, uint32_t bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l1(const void *g)
{
    asm volatile("prefetch.global.L1 [%0];" ::"l"(g));
}

struct RowTGeom {
    static constexpr int N = 32768, P = 1024, Q = 32;
    static constexpr int CL = 16;                 // CTAs per cluster (non-portable size)
    static constexpr int RP = 2;                  // rows per cluster iteration
    static constexpr int NT = RP * P / CL;        // 128 threads = phase-A items per CTA
    static constexpr int JA = P / CL;             // 64 values of n1 per CTA
    static constexpr int IB = RP * Q / CL;        // 4 phase-B items per CTA (one per warp)
    static constexpr int PITCH = Q + 1;           // 33: conflict-free column reads of a 32 x 32 block
    static constexpr int RITEM = Q * PITCH;       // 1056 >= P: one item's receive region
    static constexpr int R_ELEMS = IB * RITEM;    // 4224 >= NT * Q (phase A' receive layout [k1][tid])
    static constexpr int TW_ELEMS = Q * JA;       // the CTA's inter-phase twiddles [k1][j]
    static constexpr size_t BYTES = (size_t)(R_ELEMS + TW_ELEMS) * 16 + 16;   // + mbarrier
    static constexpr uint32_t RX_BYTES = (uint32_t)(NT * Q * 16);              // per exchange
    static_assert(R_ELEMS >= NT * Q && RITEM >= P && IB * 32 == NT, "layout");
};

// Tables (host, per index, exact integer reduction; fftpde_api.cu build_rowt_tables):
//   twA [rank][k1][j] = w_N^{(64 rank + j) k1}          (N entries)
//   tw32[a][b]        = w_1024^{a b}, a, b < 32          (symmetric)
//   mul [k1][s][q]    = m(k1 + 32 q + 1024 s)            (the row factor incl. 1/N)
#ifdef FFTPDE_ROWT_TRACE
__device__ long long rowt_trace[64][12];
#define RT_MARK(i) do { if (tid == 0 && blockIdx.x == 0 && it_ < 64) rowt_trace[it_][i] = clock64(); } while (0)
#else
#define RT_MARK(i) do { } while (0)
#endif
template <int UNUSED = 0>
__global__ void __launch_bounds__(RowTGeom::NT, 2)
rowt_kernel(const double2 *__restrict__ in, double2 *__restrict__ out, int64_t nrows,
            const double2 *__restrict__ twA, const double2 *__restrict__ tw32, const double *__restrict__ mul)
{
    using G = RowTGeom;
    constexpr int N = G::N, P = G::P, Q = G::Q, PITCH = G::PITCH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *R = reinterpret_cast<double2 *>(smem_raw);
    double2 *TW = R + G::R_ELEMS;
    const uint32_t mbar = smem_addr(TW + G::TW_ELEMS);
    const uint32_t Rbase = smem_addr(R);
    const uint32_t rank = cl_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // phase A: tid = 32 w + 16 rho + jl, j = 16 w + jl, n1 = 64 rank + j
    const int rho = (lane >> 4) & 1;
    const int j = 16 * warp + (lane & 15);
    const int n1 = G::JA * (int)rank + j;
    // phase B: warp -> item (rhoB, k1B)
    const int itB = G::IB * (int)rank + warp;
    const int rhoB = itB / Q, k1B = itB % Q;

    for (int i = tid; i < G::TW_ELEMS; i += G::NT) TW[i] = twA[(size_t)rank * G::TW_ELEMS + i];
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // every CTA's mbarrier is initialised (fence.mbarrier_init) and its receive buffer free
    if (tid == 0) mbar_expect_tx(mbar, G::RX_BYTES);
    cl_arrive_relaxed();
    uint32_t phase = 0;

    const int64_t npairs = nrows / G::RP;
    const int64_t ncl = gridDim.x / G::CL;
    int64_t pair = blockIdx.x / G::CL;
    pdl_wait();
    auto prefetch_pair = [&](int64_t pr) {      // this CTA's 2 x 32 runs of 64 points (1 KiB) -> L2
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
        // ---- phase A: 32-point DFT over n2 -> k1, times w_N^{n1 k1}
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
        // phase B's tables -> L1 while the exchange is in flight (each cluster wait
        // invalidates L1): tw32 (16 KiB, 128 lines) and this warp's factors (8 KiB, 64 lines)
        prefetch_l1(tw32 + 8 * tid);
        prefetch_l1(mul + (size_t)k1B * P + 16 * lane);
        prefetch_l1(mul + (size_t)k1B * P + 16 * lane + 512);
        RT_MARK(4);
        mbar_wait(mbar, phase);
        phase ^= 1u;
        RT_MARK(5);
        // ---- phase B: item (rhoB, k1B), 1024 points n1 = lane + 32 m
        double2 *Rw = R + warp * G::RITEM;
        double2 u[Q];
#pragma unroll
        for (int m = 0; m < Q; ++m) u[m] = Rw[lane + 32 * m];
        dft_r<Q, false>(u);                                   // over m -> q (lane = t)
#pragma unroll
        for (int q = 1; q < Q; ++q) u[q] = cmulw<false>(u[q], __ldg(tw32 + q * 32 + lane));   // w_1024^{t q}
        __syncwarp();
#pragma unroll
        for (int q = 0; q < Q; ++q) Rw[q * PITCH + lane] = u[q];
        __syncwarp();
#pragma unroll
        for (int t = 0; t < Q; ++t) u[t] = Rw[lane * PITCH + t];   // lane = q now
        dft_r<Q, false>(u);                                   // over t -> s: X[k1B + 32 (q + 32 s)]
        {
            const double *mq = mul + (size_t)k1B * P + lane;
#pragma unroll
            for (int s = 0; s < Q; ++s) u[s] = cscale(u[s], __ldg(mq + 32 * s));
        }
        dft_r<Q, true>(u);                                    // inverse over s -> t
#pragma unroll
        for (int t = 1; t < Q; ++t) u[t] = cmulw<true>(u[t], __ldg(tw32 + t * 32 + lane));   // w_1024^{-t q}
        __syncwarp();
#pragma unroll
        for (int t = 0; t < Q; ++t) Rw[lane * PITCH + t] = u[t];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < Q; ++q) u[q] = Rw[q * PITCH + lane];   // lane = t again
        dft_r<Q, true>(u);                                    // inverse over q -> m: Y'[n1 = lane + 32 m]
        if (tid == 0) mbar_expect_tx(mbar, G::RX_BYTES);
        cl_arrive_after(u[0].x);                              // my reads of R are done (u[0] depends on all)
        RT_MARK(6);
        cl_wait_acquire();
        RT_MARK(7);
        {   // -> phase-A owner of n1 = lane + 32 m: CTA m / 2, thread tdst, R[k1B][tdst] (lanes contiguous)
            const int tdst0 = 32 * (lane >> 4) + 16 * rhoB + (lane & 15);
            const uint32_t a0 = Rbase + (uint32_t)(k1B * G::NT + tdst0) * 16u;
#pragma unroll
            for (int m = 0; m < Q; m += 2) {
                const uint32_t to = (uint32_t)(m / 2);
                const uint32_t dst = mapa_rank(a0, to), mb = mapa_rank(mbar, to);
                st_async(dst, u[m], mb);                      // jj = lane
                st_async(dst + 64u * 16u, u[m + 1], mb);      // jj = lane + 32: tdst + 64
            }
        }
        RT_MARK(8);
        mbar_wait(mbar, phase);
        phase ^= 1u;
        RT_MARK(9);
        // ---- phase A': times w_N^{-n1 k1}, inverse 32-point DFT over k1 -> n2, transposed store
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
