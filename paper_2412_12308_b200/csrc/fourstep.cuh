// fourstep.cuh -- the high-index DFT pass of the 2D four-step (Bailey) solve
// of the 32768 x 32768 complex128 diffusion (C5), sm_100a.
//
// Both axes are split N = P Q with P = 1024, Q = 32 (PAPER.md:262-273's row /
// column split of the 2D sum, applied once more inside each axis):
//   x = n1 + P n2, kx = k1 + Q k2;   y = m1 + P m2, ky = l1 + Q l2
//   X[k1 + Q k2] = sum_{n1} w_P^{n1 k2} [ w_N^{n1 k1} sum_{n2} x[n1 + P n2] w_Q^{n2 k1} ]
// (eq:DFT).  One diffusion step (separable, R26)
// is then four passes over the field in HBM, each reading and writing it once:
//   AA     (this kernel)  for every (m1, n1): the Q-point DFTs over n2 and over
//                         m2 with their twiddles w_N^{n1 k1}, w_N^{m1 l1}
//   Bx     (line pass)    1024-point rows of fixed k1: DFT over n1, times
//                         e^{-D kx^2 dt}/nx at kx = k1 + Q k2, inverse DFT
//   By     (line pass)    1024-point column segments of fixed l1: the same along y
//   AA^-1  (this kernel)  conjugate twiddles, inverse Q-point DFTs: the
//                         physical field u (materialised every step, R8)
// AA^-1 of step s and AA of step s+1 run as one pass (MID): one read, the
// physical field written, the next step's AA-domain field written.
//
// A tile is (m1, 4 consecutive n1) x all (m2, n2): 32 x 32 x 4 points (64 KiB),
// moved by one 4D tensor-memory-accelerator box per direction (64-byte row
// segments; no thread issues a global access), transformed along n2 by thread
// (m2, w) and along m2 by thread (k1, w), each a radix-32 DFT in registers.
#pragma once
#include <cuda.h>
#include "fft_core.cuh"
#include "tmacols.cuh"
#include "line.cuh"
#include "launch.h"

namespace fftpde {

struct FsGeom {
    static constexpr int N = 32768, P = 1024, Q = 32, W = 4;
    static constexpr int NT = Q * W;                       // 128 threads
    static constexpr int TILE = Q * Q * W;                 // 4096 points
    static constexpr int NCHUNK = P / W;                   // 256 n1-chunks per m1
    static constexpr int NTILES = P * NCHUNK;              // 262144 tiles
};
#ifndef FFTPDE_FS_MINB
#define FFTPDE_FS_MINB 3
#endif
#ifndef FFTPDE_FS_NBUF
#define FFTPDE_FS_NBUF 1
#endif
#ifndef FFTPDE_FS_TWP
#define FFTPDE_FS_TWP 33
#endif
#ifndef FFTPDE_FS_B3TW
#define FFTPDE_FS_B3TW 1    // b3_kernel: the 1024-point twiddles from shared memory
#endif
#ifndef FFTPDE_FS_SWZ
#define FFTPDE_FS_SWZ 1
#endif
#ifndef FFTPDE_FS_XSEL
#define FFTPDE_FS_XSEL 1
#endif
// NB = 1: one tile per CTA, several CTAs per SM (the scheduler overlaps one CTA's
// TMA traffic with another's transforms); NB = 2: persistent CTAs with the next
// tile's load in flight
template <int NB> struct FsCfg {
    static constexpr int NBUF = NB;
    static constexpr int MINB = NB == 1 ? FFTPDE_FS_MINB : 1;
    // the tile's twiddles: x [w][k1] at row pitch TWP = Q + 1 (the four w rows of one k1
    // fall in distinct banks: the x-pass loads of a warp are one wavefront, not four),
    // then y [l1]; TWB = the bytes they bring
    static constexpr int TWP = FFTPDE_FS_TWP;
    static constexpr int TWS = FsGeom::W * TWP + FsGeom::Q;
    static constexpr uint32_t TWB = (uint32_t)(FsGeom::W * FsGeom::Q + FsGeom::Q) * 16;
    static constexpr size_t BYTES = (size_t)NB * (FsGeom::TILE + TWS) * 16 + 128 + 64;   // + alignment slack + mbarriers
};
enum FsOp { FS_FWD = 0, FS_INV = 1, FS_MID = 2, FS_COPY = 3, FS_COPY3 = 4 };   // COPY*: traffic-only (experiments)
// a 128-thread group's named barrier (id >= 1; 0 is __syncthreads)
struct SyncGroup {
    int id;
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
};

__device__ __forceinline__ void tma_load4(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                          uint32_t mbar)
{
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                 "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void tma_store4(const CUtensorMap *map, int c0, int c1, int c2, int c3, uint32_t src)
{
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(src) : "memory");
}

__device__ __forceinline__ void tma_prefetch4(const CUtensorMap *map, int c0, int c1, int c2, int c3)
{
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_prefetch3(const CUtensorMap *map, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2) : "memory");
}
// ---- the distributed four-step (sharded plans, R28) -------------------
// P ranks, M = P_fs / P (m1 or n1 values per rank).  Every rank's part of the field
// is the 5D array [B][Q][M][Q][M] = [blk][l1|m2][m1_l][k1|n2][n1_l]:
//   Y-part (xmode 0, rank r): m1 = r M + m1_l, blk = q, n1 = q M + n1_l  (all x, rows of one m1 range)
//   X-part (xmode 1, rank q): n1 = q M + n1_l, blk = r, m1 = r M + m1_l  (all y, columns of one n1 range)
// so the global array is G[r][q][..] and the Y -> X exchange is the all-to-all of
// its first two indices (block q of rank r's Y-part -> block r of rank q's X-part).
// At P = 1 both parts are the single-GPU layout [y = m1 + P l1][x = n1 + P k1].
struct FsPart {
    int M, P, rank, xmode;
    int ntiles;    // tiles of this pass on this rank
    int nb;        // AA: tiles per value of the tile's leading index
    int rows;      // Bx: local rows (Q M)
    int ngroup;    // By: 4-column groups per 1024-row block (Q M / W)
    int lgM, lgNb, lgMW, lgNg;   // log2 of M, nb, M / W and of the B pass's tiles per line class
    int topeer;    // B pass: store the result into the peers' other part (the exchange fused, R28)
};
// the peers' Y-parts as By store maps ({2 Q M doubles, M, Q, P}, boxes of 64 B x min(M, 256) rows)
struct FsPeerMaps {
    CUtensorMap m[kFsMaxPeerMaps];
};
struct FsTile { int m1, chunk, cx, cm, cb; };     // global m1 and n1-chunk; tensor coordinates
template <bool DIST> __device__ __forceinline__ FsTile fs_tile(int tile, const FsPart &pt)
{
    using G = FsGeom;
    FsTile t;
    if constexpr (!DIST) {
        t.m1 = tile / G::NCHUNK;
        t.chunk = tile % G::NCHUNK;
        t.cx = 2 * G::W * t.chunk;
        t.cm = t.m1;
        t.cb = 0;
    } else {
        const int a = tile >> pt.lgNb, b = tile & ((1 << pt.lgNb) - 1);
        t.m1 = pt.xmode ? a : (pt.rank << pt.lgM) + a;
        t.chunk = pt.xmode ? (pt.rank << pt.lgMW) + b : b;
        t.cx = 2 * G::W * (t.chunk & ((1 << pt.lgMW) - 1));
        t.cm = t.m1 & (pt.M - 1);
        t.cb = pt.xmode ? t.m1 >> pt.lgM : t.chunk >> pt.lgMW;
    }
    return t;
}
__device__ __forceinline__ void tma_load5(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                          uint32_t mbar)
{
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                 "r"(c4), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void tma_store5(const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4, uint32_t src)
{
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src) : "memory");
}
template <bool DIST> __device__ __forceinline__ void fs_tile_load(uint32_t dst, const CUtensorMap *map, const FsTile &t,
                                                                  uint32_t mb)
{
    if constexpr (DIST) tma_load5(dst, map, t.cx, 0, t.cm, 0, t.cb, mb);
    else tma_load4(dst, map, t.cx, 0, t.cm, 0, mb);
}
template <bool DIST> __device__ __forceinline__ void fs_tile_store(const CUtensorMap *map, const FsTile &t, uint32_t src)
{
    if constexpr (DIST) tma_store5(map, t.cx, 0, t.cm, 0, t.cb, src);
    else tma_store4(map, t.cx, 0, t.cm, 0, src);
}

#ifndef FFTPDE_FS_PF
#define FFTPDE_FS_PF 0      // L2 prefetch of the tile one wave ahead: measured +3% (578 vs 561 ms per solve), off
#endif

// Tables: tw[a][b] = w_N^{a b}, a < P, b < Q (both axes: x and y have the same N).
// Tile smem layout [row index r][col index c][w] = (r * Q + c) * W + w, where r is
// m2 (physical) or l1 (AA domain) and c is n2 or k1.

// Thread `lead` issues the loads of a tile (TMA box) and of its twiddles into slot
// S / ts, completing on mbarrier `mb`.
template <typename Cfg, bool DIST>
__device__ __forceinline__ void aa_load(const CUtensorMap *min, const double2 *tw, const FsTile &ti, double2 *S,
                                        double2 *ts, uint32_t mb)
{
    using G = FsGeom;
    constexpr int Q = G::Q, W = G::W, TWP = Cfg::TWP;
    const int m1 = ti.m1, chunk = ti.chunk;
    tma_mbar_expect(mb, (uint32_t)(G::TILE * 16) + Cfg::TWB);
    fs_tile_load<DIST>(tma_smem(S), min, ti, mb);
    if constexpr (TWP == Q) {
        bulk_g2s(tma_smem(ts), tw + (size_t)chunk * W * Q, W * Q * 16, mb);     // w_N^{n1 k1}, 4 n1
    } else {
#pragma unroll
        for (int i = 0; i < W; ++i) bulk_g2s(tma_smem(ts + i * TWP), tw + ((size_t)chunk * W + i) * Q, Q * 16, mb);
    }
    bulk_g2s(tma_smem(ts + W * TWP), tw + (size_t)m1 * Q, Q * 16, mb);           // w_N^{m1 l1}
}

// The work on one landed tile by 128 threads (r, w) = (tid / W, tid % W), `sync`
// their barrier, `lead` the thread that issues the stores.  On return the last
// store is committed (the caller waits for its read before reusing the slot).
template <int OP, typename Cfg, bool DIST, typename Sync>
__device__ __forceinline__ void aa_tile(double2 *S, const double2 *ts, int r, int w, bool lead, const FsTile &ti,
                                        const CUtensorMap *mout, const CUtensorMap *mphys, Sync sync)
{
    using G = FsGeom;
    constexpr int Q = G::Q, W = G::W;
    const double2 *twx = ts + w * Cfg::TWP;                // w_N^{n1 k1}
    const double2 *twy = ts + W * Cfg::TWP;                // w_N^{m1 l1}
    double2 v[Q];
    // The intermediate between the x and y DFTs is kept row-swizzled: element
    // (row, col) at (row, col ^ (row & 1)).  An x-pass warp covers 8 rows x 4 w of
    // one col, two rows per quarter-warp; dense, those two rows hit the same
    // banks (two wavefronts per quarter), swizzled they fill both 64-byte halves.
    // The TMA-facing layouts (tile in, physical field and AA domain out) stay dense.
    const int rb = FFTPDE_FS_SWZ ? (r & 1) : 0;
    double2 *const xe = S + (r * Q + rb) * W + w;          // x pass, row r: even cols at xe[n W]
    double2 *const xo = S + (r * Q - rb) * W + w;          //                odd cols at xo[n W]
    double2 *const ye = S + r * W + w;                     // y pass, col r: even rows at ye[m Q W]
    double2 *const yo = S + (FFTPDE_FS_SWZ ? (r ^ 1) : r) * W + w;   //      odd rows at yo[m Q W]
    auto X = [&](int n) -> double2 & { return (n & 1) ? xo[n * W] : xe[n * W]; };
    auto Y = [&](int m) -> double2 & { return (m & 1) ? yo[m * Q * W] : ye[m * Q * W]; };

    auto xpass_fwd = [&]() {      // v[n2] (thread (m2, w)) -> v[k1] = w^{n1 k1} DFT_n2
        dft_r<Q, false>(v);
#pragma unroll
        for (int k = 1; k < Q; ++k) v[k] = cmulw<false>(v[k], twx[k]);
    };
    auto ypass_fwd = [&]() {      // thread (k1, w): rows m2 -> l1
#pragma unroll
        for (int m = 0; m < Q; ++m) v[m] = Y(m);
        dft_r<Q, false>(v);
#pragma unroll
        for (int l = 1; l < Q; ++l) v[l] = cmulw<false>(v[l], twy[l]);
#pragma unroll
        for (int l = 0; l < Q; ++l) S[(l * Q + r) * W + w] = v[l];
    };
    auto store_tile = [&](const CUtensorMap *map) {
        tma_fence_smem();
        sync();
        if (lead) {
            fs_tile_store<DIST>(map, ti, tma_smem(S));
            tma_commit();
        }
    };

    if constexpr (OP == FS_COPY) {                         // the AA / AA^-1 traffic with no arithmetic
        store_tile(mout);
    } else if constexpr (OP == FS_COPY3) {                 // the MID traffic: two stores of the tile
        store_tile(mphys);
        store_tile(mout);
    } else if constexpr (OP == FS_FWD) {
#pragma unroll
        for (int n = 0; n < Q; ++n) v[n] = S[(r * Q + n) * W + w];
        xpass_fwd();
#pragma unroll
        for (int k = 0; k < Q; ++k) X(k) = v[k];
        sync();
        ypass_fwd();
        store_tile(mout);
    } else {
        // ---- AA^-1: thread (k1, w): rows l1 -> m2 with w^{-m1 l1} (own slots only)
#pragma unroll
        for (int l = 0; l < Q; ++l) v[l] = S[(l * Q + r) * W + w];
#pragma unroll
        for (int l = 1; l < Q; ++l) v[l] = cmulw<true>(v[l], twy[l]);
        dft_r<Q, true>(v);
#pragma unroll
        for (int m = 0; m < Q; ++m) Y(m) = v[m];
        sync();
        // thread (m2, w): k1 -> n2 with w^{-n1 k1} (own slots only)
#pragma unroll
        for (int k = 0; k < Q; ++k) v[k] = X(k);
#pragma unroll
        for (int k = 1; k < Q; ++k) v[k] = cmulw<true>(v[k], twx[k]);
        dft_r<Q, true>(v);
        // the physical tile, dense for the TMA store: odd rows write col n ^ 1 in
        // store n, so each quarter-warp fills both 64-byte halves (conflict-free)
#pragma unroll
        for (int n = 0; n < Q; ++n) {
            if (FFTPDE_FS_XSEL) X(n) = rb ? v[n ^ 1] : v[n];
            else S[(r * Q + n) * W + w] = v[n];
        }
        if constexpr (OP == FS_INV) {
            store_tile(mout);
        } else {
            store_tile(mphys);                             // the physical field of this step
            // ---- AA of the next step, from the registers
            xpass_fwd();
            if (lead) tma_wait_read0();                    // the store has read the slot
            sync();
#pragma unroll
            for (int k = 0; k < Q; ++k) X(k) = v[k];
            sync();
            ypass_fwd();
            store_tile(mout);
        }
    }
}

struct SyncBlock { __device__ __forceinline__ void operator()() const { __syncthreads(); } };

template <int OP, int NB, bool DIST = false>
__global__ void __launch_bounds__(FsGeom::NT, FsCfg<NB>::MINB)
aa_kernel(const __grid_constant__ CUtensorMap min, const __grid_constant__ CUtensorMap mout,
          const __grid_constant__ CUtensorMap mphys, const double2 *__restrict__ tw, const FsPart pt)
{
    using G = FsGeom;
    using Cfg = FsCfg<NB>;
    constexpr int W = G::W, NBUF = Cfg::NBUF;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // 128-byte aligned tile slots (offset kept in the shared window: LDS/STS, not generic loads)
    const uint32_t pad = (128u - (tma_smem(smem_raw) & 127u)) & 127u;
    double2 *S0 = reinterpret_cast<double2 *>(smem_raw + pad);
    double2 *TWS0 = S0 + NBUF * G::TILE;                   // per slot: [w][k1] x twiddles, then [l1] y twiddles
    const uint32_t mbar0 = tma_smem(TWS0 + NBUF * Cfg::TWS);
    const int tid = threadIdx.x;
    const int w = tid % W, r = tid / W;                   // (m2 | k1, w) of this thread
    if (tid == 0) {
        for (int i = 0; i < NBUF; ++i) tma_mbar_init(mbar0 + 8u * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto load = [&](int t, int slot) {
        aa_load<Cfg, DIST>(&min, tw, fs_tile<DIST>(t, pt), S0 + slot * G::TILE, TWS0 + slot * Cfg::TWS, mbar0 + 8u * slot);
    };
    pdl_wait();
    const int ntiles = DIST ? pt.ntiles : G::NTILES;
    int tile = blockIdx.x;
    if (tid == 0 && tile < ntiles) load(tile, 0);
    if (!DIST && NBUF == 1 && FFTPDE_FS_PF && tid == 0) {           // the tile one wave of resident CTAs ahead -> L2
        const int pf = tile + 3 * 148;
        if (pf < G::NTILES) tma_prefetch4(&min, 2 * W * (pf % G::NCHUNK), 0, pf / G::NCHUNK, 0);
    }
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const int slot = it % NBUF;
        const int next = tile + gridDim.x;
        if (tid == 0) {
            if (NBUF > 1 && next < ntiles) {
                tma_wait_read0();                          // the last store from that slot has read it
                load(next, (it + 1) % NBUF);
            } else if (next >= ntiles) {
                pdl_trigger();
            }
        }
        tma_mbar_wait(mbar0 + 8u * slot, (uint32_t)(it / NBUF) & 1u);
        aa_tile<OP, Cfg, DIST>(S0 + slot * G::TILE, TWS0 + slot * Cfg::TWS, r, w, tid == 0, fs_tile<DIST>(tile, pt),
                               &mout, &mphys, SyncBlock{});
    }
    if (tid == 0) tma_wait_read0();                        // smem stays valid until the stores have read it
}



// ---- By: the 1024-point column segments of the AA-domain field (block l1 = rows
// [1024 l1, 1024 l1 + 1024)), forward DFT over m1, times e^{-D ky^2 dt}/ny at
// ky = l1 + Q l2, inverse DFT; a tile of 4 adjacent columns (64 KiB) arrives as
// 4 TMA boxes of 256 rows x 64 bytes and leaves the same way, one tile per CTA,
// several CTAs per SM (the line pass issued 32 strided 16-byte loads per thread).
struct ByGeom {
    static constexpr int L = 1024, E = 32, W = 4, BOXR = 256;
    static constexpr int NT = W * (L / E);                         // 128 threads
    using LS = LineSmem<double2, L, E, W, true>;
    static constexpr size_t TILE_BYTES = (size_t)L * W * 16;       // 64 KiB dense
    static constexpr size_t XCH_BYTES = (size_t)W * LS::S * 16;    // exchange buffers
    static constexpr size_t BUF = TILE_BYTES > XCH_BYTES ? TILE_BYTES : XCH_BYTES;
    static constexpr size_t BYTES = BUF + 128 + 16;
    static constexpr int NGROUP = FsGeom::N / W;                   // 8192 column groups per block
};

template <int MINB>
__global__ void __launch_bounds__(ByGeom::NT, MINB)
by_kernel(const __grid_constant__ CUtensorMap map, const double2 *__restrict__ tw32, const double *__restrict__ my2d)
{
    using G = ByGeom;
    constexpr int L = G::L, E = G::E, W = G::W, TPT = L / E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t pad = (128u - (tma_smem(smem_raw) & 127u)) & 127u;
    double2 *S = reinterpret_cast<double2 *>(smem_raw + pad);
    const uint32_t mbar = tma_smem(reinterpret_cast<unsigned char *>(S) + G::BUF);
    const int tid = threadIdx.x;
    const int c = tid % W, t = tid / W;
    const int l1 = (int)(blockIdx.x / G::NGROUP), grp = (int)(blockIdx.x % G::NGROUP);
    const int x0 = 2 * W * grp;                                    // tensor coordinate (doubles)
    if (tid == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    if (tid == 0) {
        tma_mbar_expect(mbar, (uint32_t)G::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < L / G::BOXR; ++k)
            tma_load3(tma_smem(S) + k * G::BOXR * W * 16, &map, x0, 1024 * l1 + k * G::BOXR, 0, mbar);
        if (FFTPDE_FS_PF) {                                        // the tile one wave ahead -> L2
            const int pf = (int)blockIdx.x + 2 * 148;
            if (pf < FsGeom::Q * G::NGROUP) {
                const int pl1 = pf / G::NGROUP, pg = pf % G::NGROUP;
#pragma unroll
                for (int k = 0; k < L / G::BOXR; ++k) tma_prefetch3(&map, 2 * W * pg, 1024 * pl1 + k * G::BOXR, 0);
            }
        }
    }
    pdl_trigger();
    const TwL1<L, double2, E> twp{tw32, t};
    const SmemView<double2, Shape<L, E>::LOGE, 1> sm{S + c * G::LS::S};
    const SyncCTA sync{};
    double2 v[E];
    tma_mbar_wait(mbar, 0);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = S[(t + TPT * e) * W + c];
    __syncthreads();                                               // the tile buffer becomes the exchange buffers
    fft_tw<L, false, E>(v, sm, t, twp, sync);                      // v[e] = X[l2 = t + 32 e]
    {
        const double *m = my2d + (size_t)l1 * L + t;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + TPT * e));
    }
    fft_tw<L, true, E>(v, sm, t, twp, sync);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) S[(t + TPT * e) * W + c] = v[e];
    tma_fence_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < L / G::BOXR; ++k)
            tma_store3(&map, x0, 1024 * l1 + k * G::BOXR, 0, tma_smem(S) + k * G::BOXR * W * 16);
        tma_commit();
        tma_wait_read0();
    }
}


// ---- Bx: 1024-point row segments of the AA-domain field (32 per grid row, line
// class k1 = segment % 32), forward DFT over n1, times e^{-D kx^2 dt}/nx at
// kx = k1 + Q k2, inverse DFT; four consecutive segments (64 KiB contiguous) per
// CTA arrive as one bulk copy and leave as one; one warp per segment (radix 32 x 32,
// warp-synchronous exchange).
struct BxGeom {
    static constexpr int L = 1024, E = 32, W = 4;
    static constexpr int NT = W * (L / E);                         // 128 threads
    static constexpr int RAW = Shape<L, E>::PADDED;                // 1056
    static constexpr size_t TILE_BYTES = (size_t)L * W * 16;       // 64 KiB dense
    static constexpr size_t XCH_BYTES = (size_t)W * RAW * 16;
    static constexpr size_t BUF = TILE_BYTES > XCH_BYTES ? TILE_BYTES : XCH_BYTES;
    static constexpr size_t BYTES = BUF + 128 + 16;
    static constexpr int64_t NTILES = (int64_t)FsGeom::N * FsGeom::Q / W;   // 262144
};

template <int MINB>
__global__ void __launch_bounds__(BxGeom::NT, MINB)
bx_kernel(double2 *f, const double2 *__restrict__ tw32, const double *__restrict__ mx2d)
{
    using G = BxGeom;
    constexpr int L = G::L, E = G::E, W = G::W, TPT = L / E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t pad = (128u - (tma_smem(smem_raw) & 127u)) & 127u;
    double2 *S = reinterpret_cast<double2 *>(smem_raw + pad);
    const uint32_t mbar = tma_smem(reinterpret_cast<unsigned char *>(S) + G::BUF);
    const int tid = threadIdx.x;
    const int c = tid / TPT, t = tid % TPT;
    double2 *g = f + (int64_t)blockIdx.x * (W * L);
    const int k1 = (int)((int64_t)blockIdx.x * W + c) % FsGeom::Q;  // line class
    if (tid == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    if (tid == 0) {
        tma_mbar_expect(mbar, (uint32_t)G::TILE_BYTES);
        bulk_g2s(tma_smem(S), g, (uint32_t)G::TILE_BYTES, mbar);
        if (FFTPDE_FS_PF && (int64_t)blockIdx.x + 2 * 148 < G::NTILES)   // the tile one wave ahead -> L2
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + (int64_t)2 * 148 * W * L),
                         "r"((uint32_t)G::TILE_BYTES) : "memory");
    }
    pdl_trigger();
    const TwL1<L, double2, E> twp{tw32, t};
    const SmemView<double2, Shape<L, E>::LOGE, 1> sm{S + c * G::RAW};
    const SyncWarp sync{};
    double2 v[E];
    tma_mbar_wait(mbar, 0);
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = S[c * L + t + TPT * e];
    __syncthreads();                                               // the tile buffer becomes the exchange buffers
    fft_tw<L, false, E>(v, sm, t, twp, sync);                      // v[e] = X[k2 = t + 32 e]
    {
        const double *m = mx2d + (size_t)k1 * L + t;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + TPT * e));
    }
    fft_tw<L, true, E>(v, sm, t, twp, sync);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) S[c * L + t + TPT * e] = v[e];
    tma_fence_smem();
    __syncthreads();
    if (tid == 0) {
        bulk_s2g(g, tma_smem(S), (uint32_t)G::TILE_BYTES);
        tma_commit();
        tma_wait_read0();
    }
}


// ---- B3: Bx or By as a persistent pass: one CTA per SM made of two independent
// 4-warp groups and three 64 KiB tile slots.  Tile j of the CTA (global tile
// blockIdx.x + j gridDim.x) sits in slot j % 3 and is transformed by group j % 2;
// the group that finishes tile j stores it, and as soon as the store has read the
// slot it loads tile j + 3 there.  Two tiles are in the transforms while the third
// is in flight from HBM, so neither group waits for a load once the pipe is full
// (the one-tile-per-CTA passes above spend a quarter of their stalls there).
// Per tile the work is that of by_kernel (COLS) or bx_kernel (rows), one warp per
// line on either axis: the By tile arrives under the 64-byte hardware swizzle, so
// lane t reading rows t + 32 e of column c hits eight distinct 16-byte bank groups
// per phase, and the exchanges are warp-synchronous (no CTA barrier per stage).
// Bx tiles by class (FFTPDE_FS_BXCLS): tile t holds segment s = t / (N/W) of the W
// grid rows W (t mod N/W) .. + W-1 -- four lines of ONE diffusion-factor class, and a
// CTA's successive tiles (t + 148 j) keep that class for ~55 tiles, so the class's
// 8 KiB factor row stays in L1 (tiles of four consecutive segments of one row cycle
// through all 32 classes: 8 GB of factor reads from L2 per pass)
#ifndef FFTPDE_FS_BXCLS
#define FFTPDE_FS_BXCLS 1     // C5 505.6 -> 504.0 ms per solve (Bx 7.79 -> 7.76 ms; SM clock under the power cap 1665 -> 1680 MHz)
#endif
__device__ __forceinline__ int64_t bx_class(int64_t tile) { return tile / (FsGeom::N / FsGeom::W); }
__device__ __forceinline__ int64_t bx_line(int64_t tile, int c)
{
    const int64_t yb = tile % (FsGeom::N / FsGeom::W);
    return (yb * FsGeom::W + c) * FsGeom::Q + bx_class(tile);   // line = grid row * 32 + segment
}

#ifndef FFTPDE_FSD_BXK
#define FFTPDE_FSD_BXK 1
#endif
template <bool COLS> struct B3Geom {
    static constexpr int L = 1024, E = 32, W = 4, BOXR = 256;
    static constexpr int GT = W * (L / E);                          // 128 threads per group
    static constexpr int NG = 2, NT = NG * GT, NSLOT = 3;
    static constexpr int PITCH = Shape<L, E>::PADDED;
    static constexpr size_t TILE_BYTES = (size_t)L * W * 16;       // 64 KiB dense
    static constexpr size_t XCH_BYTES = (size_t)W * PITCH * 16;
    static constexpr size_t SLOT = ((TILE_BYTES > XCH_BYTES ? TILE_BYTES : XCH_BYTES) + 1023) / 1024 * 1024;
    static constexpr int TWN = Shape<L, E>::TW_SIZE;               // the twiddle table staged in smem
    static constexpr size_t TWBYTES = FFTPDE_FS_B3TW ? (size_t)TWN * 16 : 0;
    static constexpr size_t BYTES = NSLOT * SLOT + TWBYTES + 1024 + 8 * NSLOT + 4 * NSLOT;
    static constexpr int NGROUP = FsGeom::N / W;                   // column groups per block (COLS)
    static constexpr int NTILES = FsGeom::Q * NGROUP;              // 262144 on either axis
};

// DIST (sharded plans, R28): Bx on a Y-part (lines of P segments of M points, one
// per block q: P bulk copies per line each way), By on an X-part (the 4D map
// {2 Q M doubles, M, Q, P}: 1024 rows of block l1 = P runs of M rows, boxes of 256 rows).
// topeer (DIST): the exchange fused into the epilogue.  Block q of this rank's
// Y-part is block `rank` of rank q's X-part at the same offset inside the block
// (and the other way round), so Bx stores the tile's run of block q (4 M points)
// with one bulk copy into peers.p[q], and By stores its rows of m1 block r with
// TMA boxes through pmaps.m[r] (the peers' Y-parts).
template <bool COLS, bool DIST = false>
__global__ void __launch_bounds__(B3Geom<COLS>::NT, 1)
b3_kernel(const __grid_constant__ CUtensorMap map, double2 *f, const double2 *__restrict__ tw32,
          const double *__restrict__ m2d, const FsPart pt, const PeerPtrs peers,
          const __grid_constant__ FsPeerMaps pmaps)
{
    using G = B3Geom<COLS>;
    const int64_t ntiles = DIST ? (int64_t)pt.ntiles : (int64_t)G::NTILES;
    const int ngroup = DIST ? (COLS ? pt.ngroup : pt.rows / G::W) : G::NGROUP;   // tiles per line class
    // Bx (DIST): the tile arrives as [q][c][n1_l] (segment q of line c at (q W + c) M).
    // FFTPDE_FSD_BXK: a tile = 4 consecutive k1 of one row (runs of 4 M points per
    // block q; loopback P = 8 with 4 rows of one k1 -- 2 KiB runs at 64 KiB stride --
    // cost 226 ms of Bx per solve against 157 at P = 1); else 4 rows of one k1
    auto bxi = [&](int c, int n1) { return (((n1 >> pt.lgM) << 2) + c) * pt.M + (n1 & (pt.M - 1)); };
    auto bxk = [&](int ti) { return FFTPDE_FSD_BXK ? (ti & (FsGeom::Q / G::W - 1)) * G::W : ti >> pt.lgNg; };
    auto bxr = [&](int ti) { return FFTPDE_FSD_BXK ? ti / (FsGeom::Q / G::W) : (ti & (ngroup - 1)) << 2; };
    constexpr int L = G::L, E = G::E, W = G::W, TPT = L / E, NS = G::NSLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t pad = (1024u - (tma_smem(smem_raw) & 1023u)) & 1023u;   // the swizzle pattern's alignment
    unsigned char *base = smem_raw + pad;
    double2 *const twS = reinterpret_cast<double2 *>(base + NS * G::SLOT);   // [TWN] twiddles (FFTPDE_FS_B3TW)
    const uint32_t mbar0 = tma_smem(base + NS * G::SLOT + G::TWBYTES);
    // issued[s] = the CTA-local index of the last tile loaded into slot s: a group
    // waits on a slot's mbarrier only once its own tile's load was issued, so the
    // parity it waits for is never two phases ahead of the barrier
    volatile int *issued = reinterpret_cast<volatile int *>(base + NS * G::SLOT + G::TWBYTES + 8 * NS);
    const int grp = threadIdx.x / G::GT, tid = threadIdx.x % G::GT;
    const int c = tid / TPT, t = tid % TPT;                        // line c of the tile, lane t
    const SyncGroup gsync{1 + grp};
    auto slot_ptr = [&](int s) { return reinterpret_cast<double2 *>(base + s * G::SLOT); };
    auto load = [&](int64_t tile, int s) {
        const uint32_t mb = mbar0 + 8u * s;
        tma_mbar_expect(mb, (uint32_t)G::TILE_BYTES);
        if constexpr (COLS && DIST) {
            const int l1 = (int)tile >> pt.lgNg, g = (int)tile & (ngroup - 1);
#pragma unroll
            for (int k = 0; k < L / G::BOXR; ++k)
                tma_load4(tma_smem(slot_ptr(s)) + k * G::BOXR * W * 16, &map, 2 * W * g, (k * G::BOXR) & (pt.M - 1), l1,
                          (k * G::BOXR) >> pt.lgM, mb);
        } else if constexpr (COLS) {
            const int l1 = (int)(tile / G::NGROUP), g = (int)(tile % G::NGROUP);
#pragma unroll
            for (int k = 0; k < L / G::BOXR; ++k)
                tma_load3(tma_smem(slot_ptr(s)) + k * G::BOXR * W * 16, &map, 2 * W * g, 1024 * l1 + k * G::BOXR, 0, mb);
        } else if constexpr (DIST) {       // one 5D box: [q][4 lines][n1_l] (bx_map_part)
            const int ti = (int)tile;
            tma_load5(tma_smem(slot_ptr(s)), &map, 0, 0, bxk(ti), bxr(ti), 0, mb);
        } else if constexpr (FFTPDE_FS_BXCLS) {
#pragma unroll
            for (int c = 0; c < W; ++c)
                bulk_g2s(tma_smem(slot_ptr(s)) + c * L * 16, f + bx_line(tile, c) * L, (uint32_t)(L * 16), mb);
        } else {
            bulk_g2s(tma_smem(slot_ptr(s)), f + tile * (W * L), (uint32_t)G::TILE_BYTES, mb);
        }
    };
    pdl_wait();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) tma_mbar_init(mbar0 + 8u * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < NS; ++s) {
            const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
            issued[s] = s;
            if (tile < ntiles) load(tile, s);
        }
    }
    if constexpr (FFTPDE_FS_B3TW)
        for (int i = threadIdx.x; i < G::TWN; i += G::NT) twS[i] = tw32[i];
    __syncthreads();
    pdl_trigger();
#ifndef FFTPDE_FS_B3SPLIT
#define FFTPDE_FS_B3SPLIT 1    // By: last-stage twiddles as products of two table values (8.09 -> 7.93 ms; Bx +0.8%: off)
#endif
    using TwS = std::conditional_t<FFTPDE_FS_B3SPLIT != 0 && COLS, TwSmemVSplit<L, E>, TwSmemV<L, E>>;
    using TwP = std::conditional_t<FFTPDE_FS_B3TW != 0, TwS, TwL1<L, double2, E>>;
    TwP twp;
    if constexpr (FFTPDE_FS_B3TW) { twp.base = tma_smem(twS); twp.t = t; }
    else twp = TwP{tw32, t};
    for (int j = grp;; j += G::NG) {
        const int64_t tile = blockIdx.x + (int64_t)j * gridDim.x;
        if (tile >= ntiles) break;
        const int s = j % NS;
        double2 *S = slot_ptr(s);
        while (issued[s] != j) {}
        tma_mbar_wait(mbar0 + 8u * s, (uint32_t)(j / NS) & 1u);
        double2 v[E];
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = COLS ? *reinterpret_cast<const double2 *>(
                                                     reinterpret_cast<const unsigned char *>(S) + swz64((uint32_t)(t + TPT * e) * 64u + 16u * c))
                                          : DIST ? S[bxi(c, t + TPT * e)]
                                               : S[c * L + t + TPT * e];
        gsync();                                                   // the tile slot becomes the exchange buffers
        const SmemView<double2, Shape<L, E>::LOGE, 1> sm{S + c * G::PITCH};
        const double *m;
        if constexpr (DIST && !COLS && FFTPDE_FSD_BXK) m = m2d + (size_t)(bxk((int)tile) + c) * L + t;   // class k1 of line c
        else if constexpr (DIST) m = m2d + (size_t)((int)tile >> pt.lgNg) * L + t;        // class l1 / k1
        else if constexpr (COLS) m = m2d + (size_t)(tile / G::NGROUP) * L + t;          // class l1
        else if constexpr (FFTPDE_FS_BXCLS) m = m2d + (size_t)bx_class(tile) * L + t;   // one class per tile
        else m = m2d + (size_t)((tile * W + c) % FsGeom::Q) * L + t;                     // class k1
        const SyncWarp wsync{};
        fft_tw<L, false, E>(v, sm, t, twp, wsync);
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + TPT * e));
        fft_tw<L, true, E>(v, sm, t, twp, wsync);
        gsync();                                                   // every line's exchanges are done
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if constexpr (COLS)
                *reinterpret_cast<double2 *>(reinterpret_cast<unsigned char *>(S) + swz64((uint32_t)(t + TPT * e) * 64u + 16u * c)) = v[e];
            else if constexpr (DIST) S[bxi(c, t + TPT * e)] = v[e];
            else S[c * L + t + TPT * e] = v[e];
        }
        tma_fence_smem();
        gsync();
        if (tid == 0) {
            if constexpr (COLS && DIST) {
                const int l1 = (int)tile >> pt.lgNg, g = (int)tile & (ngroup - 1);
                if (pt.topeer) {                   // rows of m1 block r -> rank r's Y-part, block `rank`
                    const int br = pt.M < G::BOXR ? pt.M : G::BOXR;
                    for (int j = 0; j < L / br; ++j) {
                        const int r = (j * br) >> pt.lgM;
                        tma_store4(&pmaps.m[r], 2 * W * g, (j * br) & (pt.M - 1), l1, pt.rank, tma_smem(S) + j * br * W * 16);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < L / G::BOXR; ++k)
                        tma_store4(&map, 2 * W * g, (k * G::BOXR) & (pt.M - 1), l1, (k * G::BOXR) >> pt.lgM,
                                   tma_smem(S) + k * G::BOXR * W * 16);
                }
            } else if constexpr (COLS) {
                const int l1 = (int)(tile / G::NGROUP), g = (int)(tile % G::NGROUP);
#pragma unroll
                for (int k = 0; k < L / G::BOXR; ++k)
                    tma_store3(&map, 2 * W * g, 1024 * l1 + k * G::BOXR, 0, tma_smem(S) + k * G::BOXR * W * 16);
            } else if constexpr (DIST) {
                const int ti = (int)tile;
                if (pt.topeer) {                   // block q's run (4 k1 x M points) -> rank q's X-part, block `rank`
                    const int64_t off = (((int64_t)pt.rank * pt.rows + bxr(ti)) * FsGeom::Q + bxk(ti)) * pt.M;
                    for (int q = 0; q < pt.P; ++q)
                        bulk_s2g(reinterpret_cast<double2 *>(peers.p[q]) + off, tma_smem(S) + q * W * pt.M * 16,
                                 (uint32_t)(W * pt.M * 16));
                } else {
                    tma_store5(&map, 0, 0, bxk(ti), bxr(ti), 0, tma_smem(S));
                }
            } else if constexpr (FFTPDE_FS_BXCLS) {
#pragma unroll
                for (int c = 0; c < W; ++c) bulk_s2g(f + bx_line(tile, c) * L, tma_smem(S) + c * L * 16, (uint32_t)(L * 16));
            } else {
                bulk_s2g(f + tile * (W * L), tma_smem(S), (uint32_t)G::TILE_BYTES);
            }
            tma_commit();
            const int64_t nt = blockIdx.x + (int64_t)(j + NS) * gridDim.x;
            tma_wait_read0();                                      // the slot is free once the store has read it
            if (nt < ntiles) load(nt, s);
            issued[s] = j + NS;
        }
    }
    if (tid == 0) {
        if (DIST && pt.topeer) tma_wait0();                        // the peer stores are performed
        else tma_wait_read0();
    }
}


// ---- BB: the Bx and By passes fused over L2-resident blocks.  A block (l1, k1) =
// rows [1024 l1, +1024) x columns [1024 k1, +1024) of the AA domain (16 MiB) holds
// 1024 whole Bx lines (row segment k1 of each of its rows) and 1024 whole By lines
// (column segments of block l1): it is closed under both passes.  The CTAs of the
// persistent, cooperatively launched grid form `teams`; a team takes blocks
// b = team, team + teams, ...: its Bx lines (one warp per line), a team barrier,
// its By tiles (4 columns x 1024 rows by TMA), a team barrier.  With teams x 16 MiB
// inside the 126 MB L2, the By pass reads what Bx wrote from L2 and HBM sees one
// read and one write of the field for both passes (32 B/pt instead of 64).
struct BbGeom {
    static constexpr int L = 1024, E = 32, NT = 128;
    static constexpr int NB = 1024;                                  // blocks (32 x 32)
    static constexpr size_t BYTES = ByGeom::BUF + 128 + 16;
};

// team barrier over global memory: release my CTA's writes, count in, wait for the
// generation to move (acquire), then order later async-proxy (TMA) reads after it
__device__ __forceinline__ void team_sync(unsigned *cnt, unsigned *gen, unsigned size, unsigned &mygen)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned g = mygen;
        if (atomicAdd(cnt, 1u) == size - 1) {
            atomicExch(cnt, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
                if (v == g) __nanosleep(64);
            } while (v == g);
        }
        mygen = g + 1;
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
}

template <int MINB>
__global__ void __launch_bounds__(BbGeom::NT, MINB)
bb_kernel(const __grid_constant__ CUtensorMap map, double2 *f, const double2 *__restrict__ tw32,
          const double *__restrict__ mx2d, const double *__restrict__ my2d, unsigned *sync, int teams)
{
    using G = ByGeom;
    constexpr int L = G::L, E = G::E, W = G::W, TPT = L / E;
    constexpr int64_t N = FsGeom::N;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t pad = (128u - (tma_smem(smem_raw) & 127u)) & 127u;
    double2 *S = reinterpret_cast<double2 *>(smem_raw + pad);
    const uint32_t mbar = tma_smem(reinterpret_cast<unsigned char *>(S) + G::BUF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int team = (int)blockIdx.x % teams, member = (int)blockIdx.x / teams;
    const unsigned tsize = (gridDim.x - (unsigned)team + (unsigned)teams - 1) / (unsigned)teams;
    unsigned *cnt = sync + 2 * team, *gen = cnt + 1;
    unsigned mygen = 0;
    if (tid == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const TwL1<L, double2, E> twx{tw32, lane};
    const SmemView<double2, Shape<L, E>::LOGE, 1> smx{S + warp * Shape<L, E>::PADDED};
    const SyncWarp wsync{};
    const int c = tid % W, t = tid / W;                              // By thread layout
    const TwL1<L, double2, E> twy{tw32, t};
    const SmemView<double2, Shape<L, E>::LOGE, 1> smy{S + c * G::LS::S};
    const SyncCTA csync{};
    uint32_t tphase = 0;
    for (int b = team; b < BbGeom::NB; b += teams) {
        const int l1 = b / FsGeom::Q, k1 = b % FsGeom::Q;
        // ---- Bx: row segment k1 of the block's 1024 rows, one warp per line
        {
            const double *m = mx2d + (size_t)k1 * L + lane;
            for (int r = member * 4 + warp; r < L; r += (int)tsize * 4) {
                double2 *g = f + (int64_t)(1024 * l1 + r) * N + 1024 * k1 + lane;
                double2 v[E];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = g[TPT * e];
                fft_tw<L, false, E>(v, smx, lane, twx, wsync);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + TPT * e));
                fft_tw<L, true, E>(v, smx, lane, twx, wsync);
#pragma unroll
                for (int e = 0; e < E; ++e) g[TPT * e] = v[e];
            }
        }
        team_sync(cnt, gen, tsize, mygen);
        // ---- By: 4-column tiles of the block's columns, rows [1024 l1, +1024)
        {
            const double *m = my2d + (size_t)l1 * L + t;
            for (int gi = member; gi < L / W; gi += (int)tsize) {
                const int x0 = 2 * (1024 * k1 + W * gi);
                if (tid == 0) {
                    tma_mbar_expect(mbar, (uint32_t)G::TILE_BYTES);
#pragma unroll
                    for (int k = 0; k < L / G::BOXR; ++k)
                        tma_load3(tma_smem(S) + k * G::BOXR * W * 16, &map, x0, 1024 * l1 + k * G::BOXR, 0, mbar);
                }
                tma_mbar_wait(mbar, tphase);
                tphase ^= 1u;
                double2 v[E];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = S[(t + TPT * e) * W + c];
                __syncthreads();
                fft_tw<L, false, E>(v, smy, t, twy, csync);
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(m + TPT * e));
                fft_tw<L, true, E>(v, smy, t, twy, csync);
                __syncthreads();
#pragma unroll
                for (int e = 0; e < E; ++e) S[(t + TPT * e) * W + c] = v[e];
                tma_fence_smem();
                __syncthreads();
                if (tid == 0) {
#pragma unroll
                    for (int k = 0; k < L / G::BOXR; ++k)
                        tma_store3(&map, x0, 1024 * l1 + k * G::BOXR, 0, tma_smem(S) + k * G::BOXR * W * 16);
                    tma_commit();
                    tma_wait_read0();                                // the tile buffer is free again
                }
                __syncthreads();
            }
        }
        if (tid == 0) tma_wait0();                                   // this block's By stores are done
        team_sync(cnt, gen, tsize, mygen);
    }
}

} // namespace fftpde
