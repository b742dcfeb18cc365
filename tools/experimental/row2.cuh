// row2.cuh -- two-level (four-step) row pass for rows too long for one CTA
// (n = 16384, 32768: a complex128 row is 256-512 KiB).  One cluster of CL
// CTAs owns one row; the row is viewed as a Q x P matrix, x[n1 + P n2]:
//   forward: phase A  Q-point transforms over n2 for blocks of W consecutive n1
//                     (W * sizeof(C) = 128-byte segments), times w_N^{n1 k1},
//                     in place at n1 + P k1
//            phase B  P-point transforms over n1 of the contiguous lines
//                     n1 + P k1 (blocks of W consecutive k1); X[k1 + Q k2] is
//                     written in natural order through a shared-memory
//                     transpose (128-byte segments along k1) after a cluster
//                     barrier (every item has read its input first)
//   inverse: the same phases in reverse order with the conjugate kernels.
// The same factorisation as col2.cuh (eq:DFT); the row's
// intermediate stays in L2 between phases.
#pragma once
#include "../../paper_2412_12308_b200/csrc/col2.cuh"

namespace fftpde {

template <typename T, int P, int Q, int NT, int EMAX> struct Row2Smem {
    using C = typename cplx_t<T>::type;
    static constexpr int W = Col2Geom<C>::W;
    using IA = Col2Items<C, Q, NT, EMAX>;
    static constexpr int TB = W * Shape<P, EMAX>::TPT;
    static constexpr int SB = Shape<P, EMAX>::PADDED + 1;
    static constexpr int SLOT_B = W * SB > P * (W + 1) ? W * SB : P * (W + 1);
    static constexpr size_t A = (size_t)IA::SLOTS * IA::SLOT_ELEMS * sizeof(C);
    static constexpr size_t B = (size_t)(NT / TB) * SLOT_B * sizeof(C);
    static constexpr size_t BYTES = A > B ? A : B;
};

template <typename T, int P, int Q, bool INV, int CL, int NT, int EMAX>
__global__ void __launch_bounds__(NT)
row2_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out, int64_t nrows,
            int64_t ny, int64_t stride, const typename cplx_t<T>::type *twP,
            const typename cplx_t<T>::type *twQ, const typename cplx_t<T>::type *twN)
{
    using C = typename cplx_t<T>::type;
    constexpr int N = P * Q;
    constexpr int W = Col2Geom<C>::W;
    using SQ = Shape<Q, EMAX>;
    using SP = Shape<P, EMAX>;
    using IA = Col2Items<C, Q, NT, EMAX>;            // W lines of Q points, lanes across lines
    constexpr int TB = W * SP::TPT;                  // phase B item: W lines of P points
    constexpr int SLOTS_B = NT / TB;
    constexpr int SB = SP::PADDED + 1;               // per-line pitch (line-major lanes)
    constexpr int SLOT_B = W * SB > P * (W + 1) ? W * SB : P * (W + 1);   // exchange or transpose tile
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);

    const unsigned rank = cluster_rank();
    const int64_t row = blockIdx.x / CL;                 // grid = CL * nrows exactly
    const int64_t bidx = row / ny;
    const int64_t base = bidx * stride + (row - bidx * ny) * N;
    const int tid = threadIdx.x;

    // ---- phase A over blocks j of W consecutive n1 (lanes c), points n2/k1 = t + TPT e
    auto phaseA = [&](const C *src, bool inverse) {
        const int slot = tid / IA::TI, lt = tid % IA::TI;
        const int c = lt % W, t = lt / W;
        SmemView<C, SQ::LOGE, 1> sm{smem + slot * IA::SLOT_ELEMS + c * IA::S};
        const ItemSync<IA::TI> sync{1 + slot};
        constexpr int E = SQ::E, TPT = SQ::TPT;
        for (int j = (int)rank * IA::SLOTS + slot; j < P / W; j += CL * IA::SLOTS) {
            const int n1 = j * W + c;
            const int64_t r0 = base + n1 + (int64_t)P * t;
            C v[E];
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = ldcg(src + r0 + (int64_t)e * P * TPT);
            if (inverse) {
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmulw<true>(v[e], ldtw(twN + n1 * (t + TPT * e)));
                fft<Q, true, EMAX>(v, sm, t, twQ, sync);
            } else {
                fft<Q, false, EMAX>(v, sm, t, twQ, sync);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmulw<false>(v[e], ldtw(twN + n1 * (t + TPT * e)));
            }
            C *dst = opaque_ptr(out + r0);
#pragma unroll
            for (int e = 0; e < E; ++e) dst[(int64_t)e * P * TPT] = v[e];
        }
    };

    // ---- phase B items: blocks j of W consecutive k1; line l = k1 - W j, P points
    constexpr int EB = SP::E, TPB = SP::TPT;
    constexpr int ROUNDS = (Q / W + CL * SLOTS_B - 1) / (CL * SLOTS_B);
    static_assert(ROUNDS * EB <= 64, "phase B keeps a CTA's items in registers");
    const int bslot = tid / TB, blt = tid % TB;
    const int line = blt / TPB, bt = blt % TPB;        // transform layout (line-major)
    const int tc = blt % W, tr = blt / W;              // transpose layout (k1 fastest)
    C *tile = smem + bslot * SLOT_B;
    SmemView<C, SP::LOGE, 1> smb{tile + line * SB};
    const ItemSync<TB> bsync{1 + bslot};
    C vb[ROUNDS][EB];

    if constexpr (!INV) {
        phaseA(in, false);
        cluster_sync_acqrel();
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int j = (int)rank * SLOTS_B + bslot + r * CL * SLOTS_B;
            if (j < Q / W) {
                const int k1 = j * W + line;
                const C *src = out + base + (int64_t)P * k1 + bt;
#pragma unroll
                for (int e = 0; e < EB; ++e) vb[r][e] = ldcg(src + e * TPB);
                fft<P, false, EMAX>(vb[r], smb, bt, twP, bsync);   // X[k1 + Q k2], k2 = bt + TPB e
            }
        }
        cluster_sync_acqrel();                           // all inputs read: natural order may be written
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int j = (int)rank * SLOTS_B + bslot + r * CL * SLOTS_B;
            if (j < Q / W) {
#pragma unroll
                for (int e = 0; e < EB; ++e) tile[(bt + TPB * e) * (W + 1) + line] = vb[r][e];
                bsync();
                for (int k2 = tr; k2 < P; k2 += TB / W)
                    out[base + (int64_t)(j * W + tc) + (int64_t)Q * k2] = tile[k2 * (W + 1) + tc];
                bsync();
            }
        }
    } else {
        // phase B': natural-order input X[k1 + Q k2] -> inverse over k2 -> lines n1 + P k1
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int j = (int)rank * SLOTS_B + bslot + r * CL * SLOTS_B;
            if (j < Q / W) {
                for (int k2 = tr; k2 < P; k2 += TB / W)
                    tile[k2 * (W + 1) + tc] = ldcg(in + base + (int64_t)(j * W + tc) + (int64_t)Q * k2);
                bsync();
#pragma unroll
                for (int e = 0; e < EB; ++e) vb[r][e] = tile[(bt + TPB * e) * (W + 1) + line];
                bsync();
                fft<P, true, EMAX>(vb[r], smb, bt, twP, bsync);
            }
        }
        cluster_sync_acqrel();                           // all natural-order inputs read
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int j = (int)rank * SLOTS_B + bslot + r * CL * SLOTS_B;
            if (j < Q / W) {
                C *dst = out + base + (int64_t)P * (j * W + line) + bt;
#pragma unroll
                for (int e = 0; e < EB; ++e) dst[e * TPB] = vb[r][e];
            }
        }
        cluster_sync_acqrel();
        phaseA(out, true);
    }
}

} // namespace fftpde
