// col2_phase.cuh -- experiment only (tools/exp_col2.cu): the four-step column pass
// as three independent launches; measured slower than col2_kernel.
#pragma once
#include "../../paper_2412_12308_b200/csrc/col2.cuh"

namespace fftpde {

// ---------------------------------------------------------------------------
// Phase-split variant: the three phases as three independent launches (no
// cluster, no barriers), each CTA slot handling one item of one column block;
// the intermediate goes through global memory between launches.
enum Col2Phase { PH_A_FWD = 0, PH_B = 1, PH_A_INV = 2 };

template <typename T, int P, int Q, int PH, int OP, int NT, int MINB, int EMAX>
__global__ void __launch_bounds__(NT, MINB)
col2_phase_kernel(Col2Args<T> g, OpTables<T> tab, int64_t nitems)
{
    using C = typename cplx_t<T>::type;
    constexpr int N = P * Q;
    constexpr int W = Col2Geom<C>::W;
    constexpr int L = PH == PH_B ? P : Q;
    using I = Col2Items<C, L, NT, EMAX>;
    using SL = Shape<L, EMAX>;
    constexpr int E = SL::E, TPT = SL::TPT;
    constexpr int NF = OP == C2_WAVE ? 2 : 1;
    constexpr int PER_BLOCK = PH == PH_B ? Q : NF * P;    // items per column block
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);
    const int tid = threadIdx.x;
    const int slot = tid / I::TI, lt = tid % I::TI;
    const int c = lt % W, t = lt / W;
    SmemView<C, SL::LOGE, 1> sm{smem + slot * I::SLOT_ELEMS + c * I::S};
    const ItemSync<I::TI> sync{1 + slot};

    const uint64_t pol = l2_policy_last();
    for (int64_t item = (int64_t)blockIdx.x * I::SLOTS + slot; item < nitems;
         item += (int64_t)gridDim.x * I::SLOTS) {
        const int64_t blk = item / PER_BLOCK;
        const int j = (int)(item - blk * PER_BLOCK);
        const int64_t bidx = blk / g.nblocks;
        const int64_t col0 = (blk - bidx * g.nblocks) * W;
        const int64_t base = bidx * g.stride + col0;
        if constexpr (PH != PH_B) {
            const int f = j / P, n1 = j - f * P;
            C *F = f ? g.V : g.U;
            const C *src = (PH == PH_A_FWD && f == 0) ? g.in : F;
            const int64_t r0 = base + (int64_t)(n1 + P * t) * g.nx + c;
            const int64_t rstep = (int64_t)P * TPT * g.nx;
            C v[E];
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = src[r0 + e * rstep];
            if constexpr (PH == PH_A_INV) {
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmulw<true>(v[e], ldtw(g.twN + n1 * (t + TPT * e)));
                fft<Q, true, EMAX>(v, sm, t, g.twQ, sync);
            } else {
                fft<Q, false, EMAX>(v, sm, t, g.twQ, sync);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmulw<false>(v[e], ldtw(g.twN + n1 * (t + TPT * e)));
            }
            C *dst = opaque_ptr(F + r0);
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e * rstep] = v[e];
        } else {
            const int k1 = j;
            const int64_t r0 = base + (int64_t)(P * k1 + t) * g.nx + c;
            const int64_t rstep = (int64_t)TPT * g.nx;
            const int64_t a = col0 + c;
            C u[E];
#pragma unroll
            for (int e = 0; e < E; ++e) u[e] = g.U[r0 + e * rstep];
            fft<P, false, EMAX>(u, sm, t, g.twP, sync);
            if constexpr (OP == C2_WAVE) {
                C w[E];
#pragma unroll
                for (int e = 0; e < E; ++e) w[e] = g.V[r0 + e * rstep];
                fft<P, false, EMAX>(w, sm, t, g.twP, sync);
                const int64_t qa = a <= tab.nfold - a ? a : tab.nfold - a;
                const T *pC = tab.wC + qa * tab.qpitch, *pS1 = tab.wS1 + qa * tab.qpitch,
                        *pS2 = tab.wS2 + qa * tab.qpitch;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int b = k1 + Q * (t + TPT * e);
                    const int qb = b <= N - b ? b : N - b;
                    const T cc = __ldg(pC + qb), s1 = __ldg(pS1 + qb), s2 = __ldg(pS2 + qb);
                    const C uh = u[e], vh = w[e];
                    u[e] = {cc * uh.x + s1 * vh.x, cc * uh.y + s1 * vh.y};
                    w[e] = {s2 * uh.x + cc * vh.x, s2 * uh.y + cc * vh.y};
                }
                fft<P, true, EMAX>(w, sm, t, g.twP, sync);
                C *dv = opaque_ptr(g.V + r0);
#pragma unroll
                for (int e = 0; e < E; ++e) st_h(dv + e * rstep, w[e], pol);
            } else if constexpr (OP == C2_POISSON) {
                const T kxa = tab.kx2[a];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const T k2 = kxa + __ldg(&tab.ky2[k1 + Q * (t + TPT * e)]);
                    u[e] = cscale(u[e], k2 == (T)0 ? (T)0 : -tab.scale / k2);
                }
            } else if constexpr (OP == C2_DIFFUSE) {
                const T exa = tab.ex[a];
#pragma unroll
                for (int e = 0; e < E; ++e) u[e] = cscale(u[e], exa * __ldg(&tab.ey[k1 + Q * (t + TPT * e)]));
            }
            fft<P, true, EMAX>(u, sm, t, g.twP, sync);
            C *du = opaque_ptr(g.U + r0);
#pragma unroll
            for (int e = 0; e < E; ++e) du[e * rstep] = u[e];
        }
    }
}

} // namespace fftpde
