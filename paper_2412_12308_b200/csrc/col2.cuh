// col2.cuh -- two-level (four-step) column pass on a thread-block cluster.
//
// A column transform of length N = P*Q along y is split as
//   n = n1 + P n2,  k = k1 + Q k2:
//   X[k1 + Q k2] = sum_{n1} w_P^{n1 k2} w_N^{n1 k1} sum_{n2} x[n1 + P n2] w_Q^{n2 k1}
// (the same DFT as eq:DFT, reorganised like the paper's own
// row/column split of the 2D sum).  One cluster of CL CTAs owns a block of W
// adjacent columns (W * sizeof(C) = 128 B, full lines) over all N rows:
//   phase A : for each n1, a Q-point transform over n2 (rows n1 + P n2), times
//             w_N^{n1 k1}; stored in place at rows n1 + P k1
//   phase B : for each k1, a P-point transform over n1 (P consecutive rows), the
//             k-space operator at b = k1 + Q k2, the inverse P-point transform
//   phase A': for each n1, times w_N^{-n1 k1}, the inverse Q-point transform
// with a cluster barrier (release/acquire) between phases.  Every global access
// is a 128-byte row segment, the per-CTA footprint is a few small tiles, and
// the block's intermediate (W N sizeof(C) bytes) stays in L2 between phases, so
// HBM sees one read and one write of the field per column pass.
#pragma once
#include <cooperative_groups.h>
#include <type_traits>
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

enum Col2Op { C2_FWD = 0, C2_INV_SCALED = 1, C2_POISSON = 2, C2_DIFFUSE = 3, C2_WAVE = 4 };

__device__ __forceinline__ void cluster_sync_acqrel()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// L2-coherent 16 B / 8 B global load (the data was written by other SMs of the cluster)
__device__ __forceinline__ double2 ldcg(const double2 *p) { return __ldcg(p); }
__device__ __forceinline__ float2 ldcg(const float2 *p) { return __ldcg(p); }

// L2 eviction-priority policies: the four-step intermediate should stay in L2
// between phases (evict_last); the input read once and the final result are
// streamed (evict_first).
__device__ __forceinline__ uint64_t l2_policy_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ldcg_h(const double2 *p, uint64_t pol)
{
    double2 r;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float2 ldcg_h(const float2 *p, uint64_t pol)
{
    float2 r;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(r.x), "=f"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_h(double2 *p, double2 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_h(float2 *p, float2 v, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

template <typename C> struct Col2Geom {
    static constexpr int W = 128 / (int)sizeof(C);      // columns per block: one 128-byte line
};

// Items of one phase: transforms of length L over W columns, W * TPT threads each.
template <typename C, int L, int NT, int EMAX> struct Col2Items {
    static constexpr int W = Col2Geom<C>::W;
    static constexpr int TPT = Shape<L, EMAX>::TPT;
    static constexpr int TI = W * TPT;                  // threads per item
    static constexpr int SLOTS = NT / TI;               // concurrent items per CTA
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int RAW = Shape<L, EMAX>::PADDED;
    // per-column pitch: lanes of a smem phase are W columns -> offset columns by LPP/W
    static constexpr int S = ((RAW + LPP - 1) / LPP) * LPP + (W >= LPP ? 1 : LPP / W);
    static constexpr int SLOT_ELEMS = W * S;
    static_assert(NT % TI == 0, "item size must divide the CTA");
};

template <int TI> struct ItemSync {
    int id;
    __device__ __forceinline__ void operator()() const
    {
        if constexpr (TI <= 32) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(TI) : "memory");
    }
};

template <typename T> struct Col2Args {
    typename cplx_t<T>::type *U;   // field (in place)
    typename cplx_t<T>::type *V;   // second field (wave) or nullptr
    const typename cplx_t<T>::type *in;   // phase-A/B source of the first read (may equal U)
    int64_t nx, stride, nblocks;   // columns, batch stride, column blocks per grid
    const typename cplx_t<T>::type *twP, *twQ, *twN;   // stage tables of P and Q; w_N^m
};

template <typename T, int P, int Q, int OP, int CL, int NT, int MINB, int EMAX>
__global__ void __launch_bounds__(NT, MINB)
col2_kernel(Col2Args<T> g, OpTables<T> tab, PeerOut po)
{
    using C = typename cplx_t<T>::type;
    constexpr int N = P * Q;
    constexpr int W = Col2Geom<C>::W;
    using IA = Col2Items<C, Q, NT, EMAX>;     // phase A: Q-point transforms
    using IB = Col2Items<C, P, NT, EMAX>;     // phase B: P-point transforms
    using SQ = Shape<Q, EMAX>;
    using SP = Shape<P, EMAX>;
    constexpr int NF = OP == C2_WAVE ? 2 : 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);

    const unsigned rank = cluster_rank();
    const int64_t cid = blockIdx.x / CL;                 // cluster -> (batch, column block)
    const int64_t bidx = cid / g.nblocks;
    const int64_t col0 = (cid - bidx * g.nblocks) * W;
    const int64_t base = bidx * g.stride + col0;
    const int tid = threadIdx.x;
    pdl_wait();
    pdl_trigger();

    // ---------------------------------------------------------------- phase A
    // item = (field f, n1); CTA `rank` takes items rank*SLOTS + s + j*CL*SLOTS
    auto phaseA = [&](bool inverse, bool first_read) {
        const int slot = tid / IA::TI, lt = tid % IA::TI;
        const int c = lt % W, t = lt / W;
        C *sb = smem + slot * IA::SLOT_ELEMS + c * IA::S;
        SmemView<C, SQ::LOGE, 1> sm{sb};
        const ItemSync<IA::TI> sync{1 + slot};
        constexpr int E = SQ::E, TPT = SQ::TPT;
        constexpr int ITEMS = NF * P;
        constexpr int STEP = CL * IA::SLOTS;
        const int64_t rstep = (int64_t)P * TPT * g.nx;
        // element e of item `it`: row n1 + P (t + TPT e)  (n2 forward, k1 inverse)
        auto item_src = [&](int it) -> const C * {
            const int f = it / P, n1 = it - f * P;
            const C *F = f ? g.V : g.U;
            const C *src = (first_read && f == 0) ? g.in : F;
            return src + base + (int64_t)(n1 + P * t) * g.nx + c;
        };
        int it = (int)rank * IA::SLOTS + slot;
        // forward phase A: input streamed in, intermediate kept in L2;
        // inverse phase A': intermediate read for the last time, result streamed out
        const uint64_t pol_ld = l2_policy_first();
        const uint64_t pol_st = inverse ? l2_policy_first() : l2_policy_last();
        C v[E], nv[E];
        if (it < ITEMS) {
            const C *s0 = item_src(it);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = ldcg_h(s0 + e * rstep, pol_ld);
        }
        for (; it < ITEMS; it += STEP) {
            // prefetch the next item of this slot while this one is transformed
            const bool more = it + STEP < ITEMS;
            if (more) {
                const C *s1 = item_src(it + STEP);
#pragma unroll
                for (int e = 0; e < E; ++e) nv[e] = ldcg_h(s1 + e * rstep, pol_ld);
            }
            const int f = it / P, n1 = it - f * P;
            C *F = f ? g.V : g.U;
            // inter-phase twiddles w_N^{n1 (t + TPT e)} = w_N^{n1 t} (w_N^{n1 TPT})^e:
            // two table loads per item instead of E (at most E-1 extra roundings;
            // C5 column pass 481 -> 468 ms per 20 steps: the E scattered loads from
            // the N-entry table missed L1)
            auto interphase = [&](auto inv_tag) {
                constexpr bool IV = decltype(inv_tag)::value;
                const C w0 = ldtw(g.twN + n1 * t), ws = ldtw(g.twN + n1 * TPT);
                C w = w0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    v[e] = cmulw<IV>(v[e], w);
                    if (e + 1 < E) w = C{w.x * ws.x - w.y * ws.y, w.x * ws.y + w.y * ws.x};
                }
            };
            if (inverse) {
                interphase(std::true_type{});
                fft<Q, true, EMAX>(v, sm, t, g.twQ, sync);
            } else {
                fft<Q, false, EMAX>(v, sm, t, g.twQ, sync);
                interphase(std::false_type{});
            }
            if (inverse && po.p[0]) {               // final output -> the owners' row slabs
#pragma unroll
                for (int e = 0; e < E; ++e)
                    *opaque_ptr(peer_col_dst<C>(po, n1 + P * (t + TPT * e), col0 + c)) = v[e];
            } else {
                C *dst = opaque_ptr(F + base + (int64_t)(n1 + P * t) * g.nx + c);
#pragma unroll
                for (int e = 0; e < E; ++e) st_h(dst + e * rstep, v[e], pol_st);
            }
            if (more) {
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = nv[e];
            }
        }
    };

    // ---------------------------------------------------------------- phase B
    // item = k1 (both fields for the wave); P consecutive rows n1 + P k1
    auto phaseB = [&]() {
        const int slot = tid / IB::TI, lt = tid % IB::TI;
        const int c = lt % W, t = lt / W;
        C *sb = smem + slot * IB::SLOT_ELEMS + c * IB::S;
        SmemView<C, SP::LOGE, 1> sm{sb};
        const ItemSync<IB::TI> sync{1 + slot};
        constexpr int E = SP::E, TPT = SP::TPT;
        constexpr int STEP = CL * IB::SLOTS;
        const int64_t rstep = (int64_t)TPT * g.nx;
        const int64_t a = col0 + c;
        int k1 = (int)rank * IB::SLOTS + slot;
        const uint64_t pol = l2_policy_last();
        C u[E], nu[E];
        if (k1 < Q) {
            const C *s0 = g.U + base + (int64_t)(P * k1 + t) * g.nx + c;
#pragma unroll
            for (int e = 0; e < E; ++e) u[e] = ldcg_h(s0 + e * rstep, pol);
        }
        for (; k1 < Q; k1 += STEP) {
            const int64_t r0 = base + (int64_t)(P * k1 + t) * g.nx + c;
            const bool more = k1 + STEP < Q;
            if (more) {     // prefetch the next item of this slot (first field)
                const C *s1 = g.U + r0 + (int64_t)P * STEP * g.nx;
#pragma unroll
                for (int e = 0; e < E; ++e) nu[e] = ldcg_h(s1 + e * rstep, pol);
            }
            C w[OP == C2_WAVE ? E : 1];
            if constexpr (OP == C2_WAVE) {       // second field's loads in flight during the first's transform
#pragma unroll
                for (int e = 0; e < E; ++e) w[e] = ldcg_h(g.V + r0 + e * rstep, pol);
            }
            fft<P, false, EMAX>(u, sm, t, g.twP, sync);                // X[k1 + Q k2], k2 = t + TPT e
            if constexpr (OP == C2_WAVE) {
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
                    u[e] = {cc * uh.x + s1 * vh.x, cc * uh.y + s1 * vh.y};   // C U + S1 V
                    w[e] = {s2 * uh.x + cc * vh.x, s2 * uh.y + cc * vh.y};   // S2 U + C V
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
                    u[e] = cscale(u[e], poisson_mul(k2, tab.scale));   // -1/|k|^2, k=0 zeroed
                }
            } else if constexpr (OP == C2_DIFFUSE) {
                const T exa = tab.ex[a];
#pragma unroll
                for (int e = 0; e < E; ++e)
                    u[e] = cscale(u[e], exa * __ldg(&tab.ey[k1 + Q * (t + TPT * e)]));   // exp(-D|k|^2 dt)/(nx ny)
            }
            fft<P, true, EMAX>(u, sm, t, g.twP, sync);
            C *du = opaque_ptr(g.U + r0);
#pragma unroll
            for (int e = 0; e < E; ++e) st_h(du + e * rstep, u[e], pol);
            if (more) {
#pragma unroll
                for (int e = 0; e < E; ++e) u[e] = nu[e];
            }
        }
    };

    if constexpr (OP == C2_POISSON || OP == C2_DIFFUSE || OP == C2_WAVE) {
        phaseA(false, true);
        cluster_sync_acqrel();
        phaseB();
        cluster_sync_acqrel();
        phaseA(true, false);
    } else if constexpr (OP == C2_FWD) {
        // forward only, out of place: phase A in place on the source (a scratch
        // buffer), phase B reads it and writes the natural order b = k1 + Q k2
        // (rows k1 + Q k2) to the destination U
        C *srcw = const_cast<C *>(g.in);
        Col2Args<T> gs = g;
        gs.U = srcw;
        // phase A on the source
        {
            const int slot = tid / IA::TI, lt = tid % IA::TI;
            const int c = lt % W, t = lt / W;
            SmemView<C, SQ::LOGE, 1> sm{smem + slot * IA::SLOT_ELEMS + c * IA::S};
            const ItemSync<IA::TI> sync{1 + slot};
            constexpr int E = SQ::E, TPT = SQ::TPT;
            for (int n1 = (int)rank * IA::SLOTS + slot; n1 < P; n1 += CL * IA::SLOTS) {
                const int64_t r0 = base + (int64_t)(n1 + P * t) * g.nx + c;
                const int64_t rstep = (int64_t)P * TPT * g.nx;
                C v[E];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = ldcg(srcw + r0 + e * rstep);
                fft<Q, false, EMAX>(v, sm, t, g.twQ, sync);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cmulw<false>(v[e], ldtw(g.twN + n1 * (t + TPT * e)));
                C *dst = opaque_ptr(srcw + r0);
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e * rstep] = v[e];
            }
        }
        cluster_sync_acqrel();
        {
            const int slot = tid / IB::TI, lt = tid % IB::TI;
            const int c = lt % W, t = lt / W;
            SmemView<C, SP::LOGE, 1> sm{smem + slot * IB::SLOT_ELEMS + c * IB::S};
            const ItemSync<IB::TI> sync{1 + slot};
            constexpr int E = SP::E, TPT = SP::TPT;
            for (int k1 = (int)rank * IB::SLOTS + slot; k1 < Q; k1 += CL * IB::SLOTS) {
                C v[E];
                const int64_t r0 = base + (int64_t)(P * k1 + t) * g.nx + c;
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = ldcg(srcw + r0 + e * (int64_t)TPT * g.nx);
                fft<P, false, EMAX>(v, sm, t, g.twP, sync);
#pragma unroll
                for (int e = 0; e < E; ++e) g.U[base + (int64_t)(k1 + Q * (t + TPT * e)) * g.nx + c] = v[e];
            }
        }
        (void)gs;
    } else {  // C2_INV_SCALED, out of place: natural-order spectrum in g.in -> g.U, times 1/(nx ny)
        {
            const int slot = tid / IB::TI, lt = tid % IB::TI;
            const int c = lt % W, t = lt / W;
            SmemView<C, SP::LOGE, 1> sm{smem + slot * IB::SLOT_ELEMS + c * IB::S};
            const ItemSync<IB::TI> sync{1 + slot};
            constexpr int E = SP::E, TPT = SP::TPT;
            for (int k1 = (int)rank * IB::SLOTS + slot; k1 < Q; k1 += CL * IB::SLOTS) {
                C v[E];
#pragma unroll
                for (int e = 0; e < E; ++e)
                    v[e] = cscale(ldcg(g.in + base + (int64_t)(k1 + Q * (t + TPT * e)) * g.nx + c), tab.scale);
                fft<P, true, EMAX>(v, sm, t, g.twP, sync);
#pragma unroll
                for (int e = 0; e < E; ++e) g.U[base + (int64_t)(P * k1 + t + TPT * e) * g.nx + c] = v[e];
            }
        }
        cluster_sync_acqrel();
        phaseA(true, false);
    }
}

} // namespace fftpde
