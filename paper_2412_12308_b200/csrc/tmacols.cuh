// tmacols.cuh -- column pass with TMA tile movement (sm_100a).
//
// The y-pass of a field of rows [b][ny][nx]: W adjacent columns (W * sizeof(C)
// = 64 bytes) form a tile; a tile of N = ny rows is brought into shared memory
// by the tensor memory accelerator (cp.async.bulk.tensor, boxes of 256 rows x
// 64 bytes, 64-byte hardware swizzle, completion counted on an mbarrier) and
// written back the same way, so no thread issues a strided global access and the
// 64-byte row segments are gathered / scattered by the copy engine.  Per column
// (PAPER.md:266-273): forward transform along y (eq:DFT sign +), the k-space
// multiplier of the solve (eq:SolutionPoisson -1/|k|^2, or solCalorFourier
// exp(-D|k|^2 dt), with 1/(nx ny) folded in), inverse transform.
//
// Persistent CTAs, two tile slots: the TMA load of tile i+1 is in flight while
// tile i is transformed; a slot doubles as the transform's exchange buffer once
// its tile is in registers, and holds the results for the TMA store.
#pragma once
#include <cuda.h>
#include <type_traits>
#include "fft_core.cuh"
#include "launch.h"
#include "pipe.cuh"
#include "line.cuh"
#include "row2d.cuh"

namespace fftpde {

template <typename C, int N, int W, int E = 16> struct TmaColSmem {
    static_assert(W * sizeof(C) == 64, "tiles are 64-byte column segments (SWIZZLE_64B)");
    using PS = LineSmem<C, N, E, W, true>;                       // exchange pitch of a line
    static constexpr int BOXR = N < 256 ? N : 256;                  // rows per TMA box
    static constexpr int NBOX = N / BOXR;
    static constexpr size_t DENSE = (size_t)N * 64;
    static constexpr size_t XCH = (size_t)W * PS::S * sizeof(C);
    static constexpr size_t SLOT = (((DENSE > XCH ? DENSE : XCH) + 1023) / 1024) * 1024;
    static constexpr size_t BYTES = 2 * SLOT + 1024 + 64;          // + alignment slack + mbarriers
};

struct TmaColArgs {
    int64_t ncols;      // columns per grid (nx)
    int64_t groups;     // ceil(ncols / W)
    int64_t ntiles;     // batch * groups
};

__device__ __forceinline__ uint32_t tma_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_mbar_init(uint32_t mbar, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(n) : "memory");
}
__device__ __forceinline__ void tma_mbar_expect(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_mbar_wait(uint32_t mbar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n"
                 "W%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W%=;\n}" ::"r"(mbar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap *map, int x, int y, int z, uint32_t mbar)
{
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(z), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap *map, int x, int y, int z, uint32_t src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                 ::"l"(map), "r"(x), "r"(y), "r"(z), "r"(src) : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_fence_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// byte offset of row r, 16-byte chunk q of a dense 64-byte-row tile under SWIZZLE_64B
__device__ __forceinline__ uint32_t swz64(uint32_t o) { return o ^ (((o >> 7) & 3u) << 4); }

template <typename T, int N, int W, int OP, int MINB, int EX = 16>
__global__ void __launch_bounds__(W * Shape<N, EX>::TPT, MINB)
tma_cols_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, TmaColArgs a,
                const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N, EX>;
    using L = TmaColSmem<C, N, W, EX>;
    constexpr int E = S::E, TPT = S::TPT;
    constexpr bool TWO = OP == PIPE_POISSON || OP == PIPE_DIFFUSE;
    constexpr bool INV1 = OP == PIPE_INV_SCALED;
    static_assert(TPT <= 32 || W <= 15, "one named barrier per line");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // aligned by an offset from the __shared__ array (keeps the shared address space:
    // LDS/STS, not generic loads and stores)
    unsigned char *base = smem_raw + ((1024u - (tma_smem(smem_raw) & 1023u)) & 1023u);
    const uint32_t mbar0 = tma_smem(base + 2 * L::SLOT);

    const int tid = threadIdx.x;
    const int c = tid / TPT, t = tid % TPT;
    const LineSync<TPT> lsync{1 + c};
    constexpr int X2 = 2 * W;                 // box width in reals
    auto issue = [&](int64_t tile, int slot) {
        const int64_t b = tile / a.groups;
        const int x = (int)((tile - b * a.groups) * X2);
        const uint32_t mb = mbar0 + 8 * slot;
        tma_mbar_expect(mb, (uint32_t)L::DENSE);
        const uint32_t dst = tma_smem(base + slot * L::SLOT);
#pragma unroll
        for (int k = 0; k < L::NBOX; ++k) tma_load3(dst + k * L::BOXR * 64, &tin, x, k * L::BOXR, (int)b, mb);
    };

    using TwP = std::conditional_t<(EX > 16), TwL1<N, C, EX>, TwReg<N, C, EX>>;   // radix 32: no room for TwReg
    TwP twp;
    if constexpr (EX > 16) twp = TwP{tw, t};
    else twp.load(tw, t);
    if (tid == 0) {
        tma_mbar_init(mbar0, 1);
        tma_mbar_init(mbar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tin) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tout) : "memory");
    }
    __syncthreads();
    pdl_wait();

    int64_t tile = blockIdx.x;
    if (tid == 0 && tile < a.ntiles) issue(tile, 0);
    for (int it = 0; tile < a.ntiles; ++it, tile += gridDim.x) {
        const int slot = it & 1;
        const int64_t next = tile + gridDim.x;
        if (next >= a.ntiles) pdl_trigger();
        if (tid == 0 && next < a.ntiles) {
            tma_wait_read0();                 // the other slot's store has read its smem
            issue(next, slot ^ 1);
        }
        tma_mbar_wait(mbar0 + 8 * slot, (uint32_t)(it >> 1) & 1u);
        unsigned char *sb = base + slot * L::SLOT;
        const uint32_t cofs = (uint32_t)(c * sizeof(C));
        C v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = *reinterpret_cast<const C *>(sb + swz64((uint32_t)(t + TPT * e) * 64u + cofs));
        if constexpr (OP == PIPE_INV_SCALED) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], tab.scale);
        }
        __syncthreads();                      // the tile is in registers: the slot is the exchange buffer
        SmemView<C, S::LOGE, 1> sm{reinterpret_cast<C *>(sb) + c * L::PS::S};
        fft_tw<N, INV1, EX>(v, sm, t, twp, lsync);
        if constexpr (TWO) {
            const int64_t bb = tile / a.groups;
            int64_t col = (tile - bb * a.groups) * W + c;
            if (col >= a.ncols) col = 0;
            if constexpr (OP == PIPE_POISSON) {
                const T kxa = tab.kx2[col];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const T k2 = kxa + __ldg(&tab.ky2[t + TPT * e]);
                    v[e] = cscale(v[e], poisson_mul(k2, tab.scale));   // -1/|k|^2, k = 0 zeroed
                }
            } else if (tab.ey2d) {                   // four-step By pass: the factor of batch (block) bb
                const T *m = tab.ey2d + bb * N;
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + t + TPT * e));
            } else {
                const T exa = tab.ex[col];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cscale(v[e], exa * __ldg(&tab.ey[t + TPT * e]));
            }
            fft_tw<N, true, EX>(v, sm, t, twp, lsync);
        }
        __syncthreads();                      // every line is done with the exchange buffer
#pragma unroll
        for (int e = 0; e < E; ++e) *reinterpret_cast<C *>(sb + swz64((uint32_t)(t + TPT * e) * 64u + cofs)) = v[e];
        tma_fence_smem();
        __syncthreads();
        if (tid == 0) {
            const int64_t b = tile / a.groups;
            const int x = (int)((tile - b * a.groups) * X2);
            const uint32_t src = tma_smem(sb);
#pragma unroll
            for (int k = 0; k < L::NBOX; ++k) tma_store3(&tout, x, k * L::BOXR, (int)b, src + k * L::BOXR * 64);
            tma_commit();
        }
    }
    if (tid == 0) tma_wait0();
}

} // namespace fftpde


namespace fftpde {

// Cluster-pair variant: a cluster of two CTAs per column a, CTA rank f owns
// field f (0: U, 1: V) in ~70 KB of shared memory, so two clusters' CTAs share
// an SM and one CTA's TMA traffic overlaps another's transforms.  After the
// forward transforms the pair meets at a cluster barrier and each CTA reads its
// partner's spectrum straight from the partner's shared memory (DSMEM) for the
// oscillator update; a second barrier frees the buffers for the inverse.
template <typename C, int N, int EX> struct TmaWave2Smem {
    static constexpr int RAW = Shape<N, EX>::PADDED;
    static constexpr size_t LINE = ((size_t)RAW * sizeof(C) + 127) / 128 * 128;
    static constexpr int BOXR = N < 256 ? N : 256;
    static constexpr int NBOX = N / BOXR;
    static constexpr size_t BYTES = LINE + 128 + 16;
};

__device__ __forceinline__ double2 ld_cluster(uint32_t a)
{
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ float2 ld_cluster_f(uint32_t a)
{
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
    return v;
}

#ifndef FFTPDE_WAVE2_NA
#define FFTPDE_WAVE2_NA 0    // 1: the propagator rows (read once per column) bypass L1 so the twiddle table stays there
#endif
__device__ __forceinline__ double ld_stream(const double *p)
{
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float *p)
{
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

template <typename T, int N, int EX, int MINB>
__global__ void __launch_bounds__(Shape<N, EX>::TPT, MINB)
tma_wave2_cols_kernel(const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mv, int64_t ncols,
                      const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab,
                      typename cplx_t<T>::type *gU, typename cplx_t<T>::type *gV, int64_t gstride)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N, EX>;
    using L = TmaWave2Smem<C, N, EX>;
    constexpr int E = S::E, TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((128u - (tma_smem(smem_raw) & 127u)) & 127u);
    C *line = reinterpret_cast<C *>(base);
    const uint32_t mbar = tma_smem(base + L::LINE);
    const int t = threadIdx.x;
    const uint32_t f = cl_rank();                          // field of this CTA
    const int64_t cid = blockIdx.x / 2;
    const int64_t bz = cid / ncols;
    const int64_t a = cid - bz * ncols;
    const CUtensorMap *map = f ? &mv : &mu;
    const SyncCTA sync{};
    if (t == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
    }
    __syncthreads();
#ifndef FFTPDE_WAVE2_PF
#define FFTPDE_WAVE2_PF 0    // 1 / 2: prefetch this column's propagator rows into L2 / L1 ahead of the transform
#endif
#if FFTPDE_WAVE2_PF
    {   // the rows C[|a|][.] and S[|a|][.] (plan constants: no dependence on the previous launch) are read
        // once per column between the two cluster barriers; fetch their 128-byte lines now
        const int64_t qa0 = a <= tab.nfold - a ? a : tab.nfold - a;
        const T *r0 = tab.wC + qa0 * tab.qpitch, *r1 = (f ? tab.wS2 : tab.wS1) + qa0 * tab.qpitch;
        constexpr int PER = 128 / (int)sizeof(T);
        for (int i = t * PER; i <= N / 2; i += TPT * PER) {
#if FFTPDE_WAVE2_PF == 2
            asm volatile("prefetch.global.L1 [%0];" ::"l"(r0 + i) : "memory");
            asm volatile("prefetch.global.L1 [%0];" ::"l"(r1 + i) : "memory");
#else
            asm volatile("prefetch.global.L2 [%0];" ::"l"(r0 + i) : "memory");
            asm volatile("prefetch.global.L2 [%0];" ::"l"(r1 + i) : "memory");
#endif
        }
    }
#endif
    pdl_wait();
    if (t == 0) {
        tma_mbar_expect(mbar, (uint32_t)(N * sizeof(C)));
        const uint32_t d = tma_smem(base);
#pragma unroll
        for (int k = 0; k < L::NBOX; ++k) tma_load3(d + k * L::BOXR * (int)sizeof(C), map, (int)(2 * a), k * L::BOXR, (int)bz, mbar);
#ifndef FFTPDE_WAVE2_TPF
#define FFTPDE_WAVE2_TPF 0   // > 0: L2-prefetch (TMA) the column of the cluster that many clusters ahead (148 = one wave)
#endif
#if FFTPDE_WAVE2_TPF
        const int64_t pc = cid + FFTPDE_WAVE2_TPF;
        if (pc < (int64_t)(gridDim.x / 2)) {
            const int64_t pz = pc / ncols, pa = pc - pz * ncols;
#pragma unroll
            for (int k = 0; k < L::NBOX; ++k)
                asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map),
                             "r"((int)(2 * pa)), "r"(k * L::BOXR), "r"((int)pz) : "memory");
        }
#endif
    }
    pdl_trigger();
    tma_mbar_wait(mbar, 0);
    C v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = line[t + TPT * e];
    __syncthreads();
    SmemView<C, S::LOGE, 1> sm{line};
#ifndef FFTPDE_WAVE2_SPLIT
#define FFTPDE_WAVE2_SPLIT 1    // radix-32 middle-stage twiddles as products of two table values (C3 wave pass 0.559 -> 0.553 ms)
#endif
#if FFTPDE_TWPOW
    using TwP = std::conditional_t<FFTPDE_WAVE2_SPLIT != 0, TwL1PowSplit<N, C, EX>, TwL1Pow<N, C, EX>>;   // last radix 4: w, w^2, w^3 from one load
#else
    using TwP = TwL1<N, C, EX>;
#endif
    TwP twp;
    twp.tw = tw;
    twp.t = t;
    fft_tw<N, false, EX>(v, sm, t, twp, sync);
#pragma unroll
    for (int e = 0; e < E; ++e) line[t + TPT * e] = v[e];
    cl_arrive_release();                                   // my spectrum is visible to the partner
    cl_wait_acquire();
    {
        const uint32_t peer = mapa_rank(tma_smem(base), f ^ 1u);
        const int64_t qa = a <= tab.nfold - a ? a : tab.nfold - a;   // |fold(a)|
        const T *pC = tab.wC + qa * tab.qpitch, *pS = (f ? tab.wS2 : tab.wS1) + qa * tab.qpitch;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int b = t + TPT * e;
            const int qb = b <= N - b ? b : N - b;
#if FFTPDE_WAVE2_NA
            const T cc = ld_stream(pC + qb), ss = ld_stream(pS + qb);
#else
            const T cc = __ldg(pC + qb), ss = __ldg(pS + qb);
#endif
            C o;
            if constexpr (sizeof(T) == 8) o = ld_cluster(peer + (uint32_t)(b * sizeof(C)));
            else o = ld_cluster_f(peer + (uint32_t)(b * sizeof(C)));
            // U: C U + S1 V;  V: S2 U + C V
            v[e] = C{cc * v[e].x + ss * o.x, cc * v[e].y + ss * o.y};
        }
    }
    // done reading the partner's buffer.  The arrive must be a release: under
    // the PTX memory model a relaxed barrier.cluster.arrive does not order the
    // preceding ld.shared::cluster reads, so the partner could pass its wait
    // and overwrite `line` (the fft_tw below) while a remote read of it is
    // still in flight (write-after-read race).  The release costs a
    // few percent of the wave pass (r01: 274 vs 284 ms per 500 steps).
    cl_arrive_release();
    cl_wait_acquire();
    fft_tw<N, true, EX>(v, sm, t, twp, sync);
#ifndef FFTPDE_WAVE2_LSUST
#define FFTPDE_WAVE2_LSUST 0   // 1: the result column leaves through st.global from the registers (the LSU), so the
#endif                         // TMA unit only carries the column loads (it is request-rate bound on 16-byte rows)
#if FFTPDE_WAVE2_LSUST
    {
        C *g = (f ? gV : gU) + bz * gstride + a + (int64_t)t * ncols;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            C *q = g + (int64_t)(TPT * e) * ncols;
            if constexpr (sizeof(T) == 8)
                asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(q), "d"(v[e].x), "d"(v[e].y) : "memory");
            else
                asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(q), "f"(v[e].x), "f"(v[e].y) : "memory");
        }
    }
#else
#ifndef FFTPDE_WAVE2_LSUQ
#define FFTPDE_WAVE2_LSUQ 4    // 4096-point columns: the last 4 of the 16 256-row boxes leave through st.global from
#endif                         // the registers, the rest through the TMA unit, which is request-rate bound on 16-byte
                               // rows (C3 wave pass 0.553 -> 0.544 ms; 2 boxes equal, all 16 boxes 0.658 ms; run r02v)
    constexpr int LSUQ = N == 4096 ? FFTPDE_WAVE2_LSUQ : 0;
    constexpr int KT = L::NBOX - LSUQ;                      // boxes stored by the TMA unit
    constexpr int ET = KT * L::BOXR / TPT;                  // slots e < ET lie in those boxes
    static_assert(LSUQ == 0 || (L::BOXR % TPT == 0 && KT > 0), "box / slot split");
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (e < ET) line[t + TPT * e] = v[e];
    tma_fence_smem();
    __syncthreads();
    if (t == 0) {
        const uint32_t src = tma_smem(base);
#pragma unroll
        for (int k = 0; k < KT; ++k) tma_store3(map, (int)(2 * a), k * L::BOXR, (int)bz, src + k * L::BOXR * (int)sizeof(C));
        tma_commit();
    }
    if constexpr (LSUQ > 0) {
        C *g = (f ? gV : gU) + bz * gstride + a + (int64_t)t * ncols;
#pragma unroll
        for (int e = ET; e < E; ++e) {
            C *q = g + (int64_t)(TPT * e) * ncols;
            if constexpr (sizeof(T) == 8)
                asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(q), "d"(v[e].x), "d"(v[e].y) : "memory");
            else
                asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(q), "f"(v[e].x), "f"(v[e].y) : "memory");
        }
    }
    if (t == 0) tma_wait_read0();
#endif
}


} // namespace fftpde
