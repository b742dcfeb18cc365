// row2d.cuh -- four-step row pass for long rows on a thread-block cluster
// whose distributed shared memory holds the whole row (sm_100a).
//
// A row of N = P*Q points (16384, 32768: 256-512 KiB of complex128) is split
// as n = n1 + P n2, k = k1 + Q k2 (the same DFT as eq:DFT, PAPER.md:119-124,
// reorganised like the paper's own row/column split of the 2D sum,
// PAPER.md:262-273):
//   X[k1 + Q k2] = sum_{n1} w_P^{n1 k2} w_N^{n1 k1} sum_{n2} x[n1 + P n2] w_Q^{n2 k1}.
// CTA r of the CL-CTA cluster owns
//   phase A items n1 in [r PA, (r+1) PA)      (PA = P/CL): Q-point transforms over n2
//   phase B items k1 in [r QB, (r+1) QB)      (QB = Q/CL): P-point transforms over n1
// and the A -> B exchange (7/8 of the row for CL = 8) goes CTA-to-CTA through
// distributed shared memory (st.shared::cluster into the owner's receive
// buffer), not through L2: HBM and L2 see one read and one write of the row.
// Every thread holds R2E points in both phases (N/CL = R2E x threads).
//
// The inverse runs the phases in reverse (B^-1 then A^-1, conjugate kernels),
// so its output is distributed exactly like the forward input: MID (inverse
// of step s -> physical field, forward of step s+1) needs no redistribution
// between the two transforms.
#pragma once
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

// R2D_DIFF: forward transform, times mul[a] (natural wavenumber index a), inverse
// transform, one store (the x factor of a separable operator, e.g. diffusion)
enum Row2dOp { R2D_FWD = 0, R2D_INV = 1, R2D_MID = 2, R2D_DIFF = 3 };

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(uint32_t a, double2 v)
{
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t a, float2 v)
{
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
// asynchronous remote store that completes on the receiver's mbarrier (tx bytes)
__device__ __forceinline__ void st_async(uint32_t a, double2 v, uint32_t mbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                 ::"r"(a), "d"(v.x), "d"(v.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void st_async(uint32_t a, float2 v, uint32_t mbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                 ::"r"(a), "f"(v.x), "f"(v.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"(mbar), "r"(parity) : "memory");
}
__device__ __forceinline__ void cl_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait_acquire() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cl_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// points per thread (the radix of the in-register stages) in both phases
// (FFTPDE_R2D_E, launch.h: the host builds the stage tables with the same radix)
constexpr int R2E = FFTPDE_R2D_E;

template <typename C, int P, int Q, int CL> struct Row2dGeom {
    static constexpr int N = P * Q;
    static constexpr int PA = P / CL, QB = Q / CL;           // items per CTA in phases A and B
    static constexpr int TA = Q / R2E, TB = P / R2E;         // threads per item
    static constexpr int NT = PA * TA;                       // == QB * TB == N / (R2E CL)
    static constexpr int LPP = 128 / (int)sizeof(C);
    // exchange buffer: item-interleaved lanes -> pitch = 1 mod LPP/ (16 B lanes per phase)
    static constexpr int SA = ((Shape<Q, R2E>::PADDED + LPP - 1) / LPP) * LPP + 1;
    static constexpr int SB = ((Shape<P, R2E>::PADDED + LPP - 1) / LPP) * LPP + 1;
    static constexpr int XE = PA * SA > QB * SB ? PA * SA : QB * SB;
    // receive buffer: phase-B input [jb][n1] (pitch P+1) or phase-A^-1 input [ia][k1] (pitch Q+1)
    static constexpr int RE = QB * (P + 1) > PA * (Q + 1) ? QB * (P + 1) : PA * (Q + 1);
    // per-CTA twiddle slices (inter-phase w_N^{n1 k1} = S1 S2 for the CTA's n1,
    // and = U1 U2 for the CTA's k1): PA*(16 + Q/16) + QB*(16 + P/16) entries
    // slice pitches padded by one element: lanes of a warp hold consecutive items
    // and read the same column, so an unpadded power-of-two pitch would put them
    // all on the same banks
    static constexpr int A1 = 17, A2 = Q / 16 + 1, B1 = 17, B2 = P / 16 + 1;
    static constexpr int TWE = PA * (A1 + A2) + QB * (B1 + B2);
    // input staging: the CTA's share of the next row, [e][thread]
    static constexpr int SE = N / CL;
    static constexpr size_t BYTES = (size_t)(XE + RE + TWE + SE) * sizeof(C) + 16;   // + mbarrier
    static_assert(NT == QB * TB, "thread counts of the phases must agree");
    static_assert(PA >= 1 && QB >= 1, "cluster too large for the split");
};

// per-thread asynchronous global -> shared copy of one element (no register
// destination, so no register scoreboard spans the row it is in flight for)
__device__ __forceinline__ void r2_cp_async(const void *smem, const double2 *g)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void r2_cp_async(const void *smem, const float2 *g)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(smem)), "l"(g) : "memory");
}

// Tables: twP, twQ = stage tables (radix R2E) of P and Q; twS = split inter-phase
// twiddles, each entry rounded once from its exact angle:
//   S1[n1][l] = w_N^{n1 l}      (l < 16)    at twS[n1*16 + l]
//   S2[n1][h] = w_N^{16 n1 h}   (h < Q/16)  at twS[P*16 + n1*(Q/16) + h]
//   U1[k1][l] = w_N^{k1 l}      (l < 16)    at twS[P*16 + P*(Q/16) + k1*16 + l]
//   U2[k1][h] = w_N^{16 k1 h}   (h < P/16)  at twS[P*16 + P*(Q/16) + Q*16 + k1*(P/16) + h]
// w_N^{n1 k1} = S1[n1][k1 & 15] S2[n1][k1 >> 4] = U1[k1][n1 & 15] U2[k1][n1 >> 4].
template <typename T, int P, int Q, int CL, int OP>
__global__ void __launch_bounds__(Row2dGeom<typename cplx_t<T>::type, P, Q, CL>::NT, (R2E <= 8 ? 2 : 1))
row2d_kernel(const typename cplx_t<T>::type *__restrict__ in, typename cplx_t<T>::type *out,
             typename cplx_t<T>::type *out2, int64_t nrows, int64_t ny, int64_t stride,
             const typename cplx_t<T>::type *__restrict__ twP, const typename cplx_t<T>::type *__restrict__ twQ,
             const typename cplx_t<T>::type *__restrict__ twS, const T *__restrict__ mul, PeerOut po)
{
    using C = typename cplx_t<T>::type;
    using G = Row2dGeom<C, P, Q, CL>;
    constexpr int N = G::N, PA = G::PA, QB = G::QB, TA = G::TA, TB = G::TB, NT = G::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *X = reinterpret_cast<C *>(smem_raw);
    C *R = X + G::XE;
    C *TWA1 = R + G::RE;                    // [PA][16]    (pitch A1)
    C *TWA2 = TWA1 + PA * G::A1;            // [PA][Q/16]  (pitch A2)
    C *TWB1 = TWA2 + PA * G::A2;            // [QB][16]    (pitch B1)
    C *TWB2 = TWB1 + QB * G::B1;            // [QB][P/16]  (pitch B2)
    C *S = TWB2 + QB * G::B2;               // [R2E][NT]   next row's input
    const uint32_t mbar = smem_addr(S + G::SE);
    const uint32_t rank = cl_rank();
    const int tid = threadIdx.x;
    // phase A layout: item ia (n1 = rank PA + ia) fastest across lanes
    const int ia = tid % PA, ta = tid / PA;
    const int n1 = (int)rank * PA + ia;
    // phase B layout: item jb (k1 = rank QB + jb) fastest across lanes
    const int jb = tid % QB, tb = tid / QB;
    const int k1 = (int)rank * QB + jb;
    SmemView<C, Shape<R2E>::LOGE, 1> smA{X + ia * G::SA};
    SmemView<C, Shape<R2E>::LOGE, 1> smB{X + jb * G::SB};
    const SyncCTA sync{};
    const uint32_t Rbase = smem_addr(R);
    constexpr uint32_t RX_BYTES = (uint32_t)(N / CL * sizeof(C));   // bytes received per exchange

    // twiddle slices of this CTA -> smem (once)
    {
        const C *S1 = twS, *S2 = twS + P * 16, *U1 = S2 + P * (Q / 16), *U2 = U1 + Q * 16;
        for (int i = tid; i < PA * 16; i += NT) TWA1[(i / 16) * G::A1 + i % 16] = S1[(int)rank * PA * 16 + i];
        for (int i = tid; i < PA * (Q / 16); i += NT)
            TWA2[(i / (Q / 16)) * G::A2 + i % (Q / 16)] = S2[(int)rank * PA * (Q / 16) + i];
        for (int i = tid; i < QB * 16; i += NT) TWB1[(i / 16) * G::B1 + i % 16] = U1[(int)rank * QB * 16 + i];
        for (int i = tid; i < QB * (P / 16); i += NT)
            TWB2[(i / (P / 16)) * G::B2 + i % (P / 16)] = U2[(int)rank * QB * (P / 16) + i];
    }
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cl_arrive_release();
    cl_wait_acquire();                       // every CTA's mbarrier is initialised
    uint32_t phase = 0;
    auto twA = [&](int k) -> C {             // w_N^{n1 k}, n1 = this thread's phase-A item
        const C a = TWA1[ia * G::A1 + (k & 15)], b = TWA2[ia * G::A2 + (k >> 4)];
        return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
    };
    auto twB = [&](int n) -> C {             // w_N^{n k1}, k1 = this thread's phase-B item
        const C a = TWB1[jb * G::B1 + (n & 15)], b = TWB2[jb * G::B2 + (n >> 4)];
        return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
    };
    auto row_ptr = [&](const C *base, int64_t row) -> const C * {
        const int64_t b = row / ny;
        return base + b * stride + (row - b * ny) * (int64_t)N;
    };
    // input of a row: phase-A layout x[n1 + P (ta + TA e)] (FWD, DIFF) or phase-B^-1
    // layout X[k1 + Q (tb + TB e)] (INV, MID).  The next row's input is copied
    // into the staging buffer (cp.async) while this row is transformed: held in
    // registers instead, its loads shared a scoreboard with this row's first
    // butterflies, which then waited out a DRAM latency every row
    // (ncu, profiles/r01/ncu_full_c5.txt: 9% of the samples on one DADD).
    // Each thread reads back only the slots it wrote (no barrier needed).
    auto prefetch = [&](int64_t row) {
        const C *src = row_ptr(in, row);
#pragma unroll
        for (int e = 0; e < R2E; ++e) {
            if constexpr (OP == R2D_FWD || OP == R2D_DIFF) r2_cp_async(S + e * NT + tid, src + n1 + P * (ta + TA * e));
            else r2_cp_async(S + e * NT + tid, src + k1 + Q * (tb + TB * e));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto take = [&](C (&u)[R2E]) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
        for (int e = 0; e < R2E; ++e) u[e] = S[e * NT + tid];
    };
    // receive-buffer protocol: the receiver arms its mbarrier with the bytes it
    // expects and releases its buffer with a relaxed cluster arrive once the
    // previous contents are consumed; senders wait on the cluster barrier
    // (every buffer free) and push with st.async (completes on the receiver's mbarrier)
    auto release_R = [&]() {
        if (tid == 0) mbar_expect_tx(mbar, RX_BYTES);
        cl_arrive_relaxed();
    };
    auto receive = [&]() {
        mbar_wait(mbar, phase);
        phase ^= 1u;
    };

    const int64_t ncl = gridDim.x / CL;
    release_R();
    int64_t row = blockIdx.x / CL;
    pdl_wait();
    if (row < nrows) prefetch(row);
    for (; row < nrows; row += ncl) {
        if (row + ncl >= nrows) pdl_trigger();   // this cluster's last row
        C v[R2E];
        take(v);
        // the staging slots are rewritten only after the first transform consumed them
        auto prefetch_next = [&]() {
            if (row + ncl < nrows) prefetch(row + ncl);
        };
        // inverse: v in the phase-B^-1 layout X[k1 + Q (tb + TB e)] -> x[n1 + P (ta + TA e)]
        auto inv_part = [&](C (&v)[R2E], bool first) {
            // ---- B^-1: inverse P-point transforms over k2 of items k1, times w_N^{-n1 k1}
            fft<P, true, R2E>(v, smB, tb, twP, sync);          // v[e] = Y[n1 = tb + TB e][k1]
            if (first) prefetch_next();
#pragma unroll
            for (int e = 0; e < R2E; ++e) v[e] = cmulw<true>(v[e], twB(tb + TB * e));
            cl_wait_acquire();                                // every receive buffer is free
#pragma unroll
            for (int e = 0; e < R2E; ++e) {                    // -> owner of n1, R[ia'][k1] (pitch Q+1)
                const int m1 = tb + TB * e;
                const uint32_t dst = (uint32_t)(m1 % PA) * (Q + 1) + k1;
                const uint32_t to = (uint32_t)(m1 / PA);
                st_async(mapa_rank(Rbase + dst * (uint32_t)sizeof(C), to), v[e], mapa_rank(mbar, to));
            }
            receive();
            // ---- A^-1: inverse Q-point transforms over k1 of items n1
#pragma unroll
            for (int e = 0; e < R2E; ++e) v[e] = R[ia * (Q + 1) + ta + TA * e];
            fft<Q, true, R2E>(v, smA, ta, twQ, sync);          // v[e] = x[n1 + P (ta + TA e)]
            release_R();                                      // (the transform consumed R)
        };
        // forward: v in the phase-A layout x[n1 + P (ta + TA e)] -> X[k1 + Q (tb + TB e)]
        // DIFF: the x factors of this thread's phase-B points (the same for every
        // row), loaded while the exchange is in flight
        T mrow[OP == R2D_DIFF ? R2E : 1];
        auto fwd_part = [&](C (&v)[R2E], bool first) {
            // ---- A: Q-point transforms over n2 of items n1, times w_N^{n1 k1}
            fft<Q, false, R2E>(v, smA, ta, twQ, sync);         // v[e] = Y[n1][k1 = ta + TA e]
            if (first) prefetch_next();
#pragma unroll
            for (int e = 0; e < R2E; ++e) v[e] = cmulw<false>(v[e], twA(ta + TA * e));
            cl_wait_acquire();
#pragma unroll
            for (int e = 0; e < R2E; ++e) {                    // -> owner of k1, R[jb'][n1] (pitch P+1)
                const int m1 = ta + TA * e;
                const uint32_t dst = (uint32_t)(m1 % QB) * (P + 1) + n1;
                const uint32_t to = (uint32_t)(m1 / QB);
                st_async(mapa_rank(Rbase + dst * (uint32_t)sizeof(C), to), v[e], mapa_rank(mbar, to));
            }
            if constexpr (OP == R2D_DIFF) {
#pragma unroll
                for (int e = 0; e < R2E; ++e) mrow[e] = __ldg(mul + k1 + Q * (tb + TB * e));
            }
            receive();
            // ---- B: P-point transforms over n1 of items k1 -> X[k1 + Q k2]
#pragma unroll
            for (int e = 0; e < R2E; ++e) v[e] = R[jb * (P + 1) + tb + TB * e];
            fft<P, false, R2E>(v, smB, tb, twP, sync);
            release_R();
        };
        if constexpr (OP == R2D_INV || OP == R2D_MID) {
            inv_part(v, true);
            C *dst = const_cast<C *>(row_ptr(OP == R2D_INV ? out : out2, row));
#pragma unroll
            for (int e = 0; e < R2E; ++e) dst[n1 + P * (ta + TA * e)] = v[e];
        }
        if constexpr (OP == R2D_FWD || OP == R2D_MID) {
            fwd_part(v, OP == R2D_FWD);
            if (OP == R2D_FWD && po.p[0]) {          // scattered into the peers' column slabs
#pragma unroll
                for (int e = 0; e < R2E; ++e) *peer_row_dst<C>(po, row, k1 + Q * (tb + TB * e)) = v[e];
            } else {
                C *dst = const_cast<C *>(row_ptr(out, row));
#pragma unroll
                for (int e = 0; e < R2E; ++e) dst[k1 + Q * (tb + TB * e)] = v[e];
            }
        }
        if constexpr (OP == R2D_DIFF) {
            fwd_part(v, true);
#pragma unroll
            for (int e = 0; e < R2E; ++e) v[e] = cscale(v[e], mrow[e]);
            inv_part(v, false);
            if (po.p[0]) {                           // scattered into the peers' column slabs
#pragma unroll
                for (int e = 0; e < R2E; ++e) *peer_row_dst<C>(po, row, n1 + P * (ta + TA * e)) = v[e];
            } else {
                C *dst = const_cast<C *>(row_ptr(out, row));
#pragma unroll
                for (int e = 0; e < R2E; ++e) dst[n1 + P * (ta + TA * e)] = v[e];
            }
        }
    }
    cl_wait_acquire();                       // no CTA leaves while others may still write its smem
}

} // namespace fftpde
