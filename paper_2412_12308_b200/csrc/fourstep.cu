// fourstep.cu -- launcher of the four-step AA pass (fourstep.cuh).
#include <cuda.h>
#include <cstring>
#include <algorithm>
#include "fourstep.cuh"
#include "dispatch.cuh"

namespace fftpde {

#ifndef FFTPDE_FS_PROMO_AA
#define FFTPDE_FS_PROMO_AA CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
#ifndef FFTPDE_FS_PROMO_BY
#define FFTPDE_FS_PROMO_BY CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
// The four-step passes move their tiles with tensor maps: without the driver's
// encoder (or with FFTPDE_TMA=0) the plan keeps the round-1 cluster passes.
bool fourstep_supported(int64_t nx, int64_t ny, int64_t batch, int elem_bytes)
{
    return elem_bytes == 16 && nx == FsGeom::N && ny == FsGeom::N && batch == 1 && tma_encoder() != nullptr;
}

// The field as the 4D tensor {2 n1 (doubles), n2, m1, m2} of a [y = m1 + P m2][x = n1 + P n2]
// grid; boxes of {2 W doubles, Q, 1, Q}: one tile per box.
static bool fs_map(CUtensorMap &m, const void *p)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)(2 * G::P), (cuuint64_t)G::Q, (cuuint64_t)G::P, (cuuint64_t)G::Q};
    cuuint64_t strides[3] = {(cuuint64_t)G::P * 16, (cuuint64_t)G::N * 16, (cuuint64_t)G::P * G::N * 16};
    cuuint32_t box[4] = {(cuuint32_t)(2 * G::W), (cuuint32_t)G::Q, 1, (cuuint32_t)G::Q};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, FFTPDE_FS_PROMO_AA,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the rank's part of the distributed four-step (R28) as the 5D tensor
// {2 M doubles (n1_l), Q, M (m1_l), Q, P (blk)}; boxes of {2 W doubles, Q, 1, Q, 1}
static bool fs_map5(CUtensorMap &m, const void *p, int M, int P)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t r = (cuuint64_t)M * 16;
    cuuint64_t dims[5] = {(cuuint64_t)(2 * M), (cuuint64_t)G::Q, (cuuint64_t)M, (cuuint64_t)G::Q, (cuuint64_t)P};
    cuuint64_t strides[4] = {r, r * G::Q, r * G::Q * M, r * G::Q * M * G::Q};
    cuuint32_t box[5] = {(cuuint32_t)(2 * G::W), (cuuint32_t)G::Q, 1, (cuuint32_t)G::Q, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, FFTPDE_FS_PROMO_AA,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int OP, bool DIST = false>
static cudaError_t aa_n(const CUtensorMap &mi, const CUtensorMap &mo, const CUtensorMap &mp, const void *tw,
                        cudaStream_t st, const FsPart &pt = FsPart{})
{
    using G = FsGeom;
    using Cfg = FsCfg<FFTPDE_FS_NBUF>;
    auto k = aa_kernel<OP, FFTPDE_FS_NBUF, DIST>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, Cfg::BYTES);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, G::NT, Cfg::BYTES);
    if (e != cudaSuccess) return e;
    const int64_t ntiles = DIST ? pt.ntiles : G::NTILES;
    const dim3 grid(Cfg::NBUF == 1 ? (unsigned)ntiles    // one tile per CTA
                                   : (unsigned)std::min<int64_t>(ntiles, (int64_t)std::max(occ, 1) * sm_count()));
    e = launch_fam(PDL_FOURSTEP, k, grid, dim3(G::NT), Cfg::BYTES, st, mi, mo, mp, (const double2 *)tw, pt);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_aa(int op, const void *in, void *out, void *phys, const void *tw, cudaStream_t st)
{
    CUtensorMap mi, mo, mp;
    if (!fs_map(mi, in)) return cudaErrorNotSupported;
    if (out == in) mo = mi;
    else if (!fs_map(mo, out)) return cudaErrorNotSupported;
    if (!phys) mp = mo;
    else if (!fs_map(mp, phys)) return cudaErrorNotSupported;
    switch (op) {
    case FS_FWD: return aa_n<FS_FWD>(mi, mo, mp, tw, st);
    case FS_INV: return aa_n<FS_INV>(mi, mo, mp, tw, st);
    case FS_MID: return aa_n<FS_MID>(mi, mo, mp, tw, st);
    default: return cudaErrorInvalidValue;
    }
}

FsPart fs_part(int P, int rank, int xmode, int pass)
{
    using G = FsGeom;
    FsPart t{};
    t.M = G::P / P;
    t.P = P;
    t.rank = rank;
    t.xmode = xmode;
    t.rows = G::Q * t.M;
    t.ngroup = G::Q * t.M / G::W;
    t.nb = xmode ? t.M / G::W : G::NCHUNK;
    t.ntiles = pass == 0 ? G::NTILES / P : (int)((int64_t)G::Q * t.ngroup);   // AA | B passes: 262144 / P tiles
    auto lg = [](int v) { int l = 0; while ((1 << l) < v) ++l; return l; };
    t.lgM = lg(t.M);
    t.lgNb = lg(t.nb);
    t.lgMW = lg(t.M / G::W);
    t.lgNg = lg(t.ngroup);          // Bx: rows / W = Q M / W, By: ngroup (the same count)
    return t;
}

bool fs_dist_supported(int P)
{
    // M = 1024 / P points per rank along the split index, a multiple of the tile
    // width W = 4, and P <= 32 so that a rank's row slab holds whole m2 rows of 1024
    return P >= 1 && P <= 32 && (P & (P - 1)) == 0 && tma_encoder() != nullptr;
}

cudaError_t launch_aa_part(int op, int P, int rank, int xmode, const void *in, void *out, void *phys, const void *tw,
                           cudaStream_t st)
{
    const FsPart pt = fs_part(P, rank, xmode, 0);
    CUtensorMap mi, mo, mp;
    if (!fs_map5(mi, in, pt.M, P)) return cudaErrorNotSupported;
    if (out == in) mo = mi;
    else if (!fs_map5(mo, out, pt.M, P)) return cudaErrorNotSupported;
    if (!phys) mp = mo;
    else if (!fs_map5(mp, phys, pt.M, P)) return cudaErrorNotSupported;
    switch (op) {
    case FS_FWD: return aa_n<FS_FWD, true>(mi, mo, mp, tw, st, pt);
    case FS_INV: return aa_n<FS_INV, true>(mi, mo, mp, tw, st, pt);
    case FS_MID: return aa_n<FS_MID, true>(mi, mo, mp, tw, st, pt);
    default: return cudaErrorInvalidValue;
    }
}


#ifndef FFTPDE_FS_BY_TMA
#define FFTPDE_FS_BY_TMA 1
#endif
#ifndef FFTPDE_FS_BYT_MINB
#define FFTPDE_FS_BYT_MINB 2
#endif
// the field as a 3D tensor {2 N doubles, N rows, 1}; boxes of 64 bytes x 256 rows
static bool by_map(CUtensorMap &m, const void *p, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)(2 * G::N), (cuuint64_t)G::N, 1};
    cuuint64_t strides[2] = {(cuuint64_t)G::N * 16, (cuuint64_t)G::N * G::N * 16};
    cuuint32_t box[3] = {(cuuint32_t)(2 * ByGeom::W), (cuuint32_t)ByGeom::BOXR, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz, FFTPDE_FS_PROMO_BY,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static cudaError_t launch_by_tma(void *f, const void *tw32, const double *my2d, cudaStream_t st)
{
    CUtensorMap m;
    if (!by_map(m, f)) return cudaErrorNotSupported;
    auto k = by_kernel<FFTPDE_FS_BYT_MINB>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, ByGeom::BYTES);
    if (e != cudaSuccess) return e;
    e = launch_fam(PDL_FOURSTEP, k, dim3((unsigned)(FsGeom::Q * ByGeom::NGROUP)), dim3(ByGeom::NT), ByGeom::BYTES, st,
                   m, (const double2 *)tw32, my2d);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}


// The persistent three-slot B passes (b3_kernel): bit 0 Bx, bit 1 By
#ifndef FFTPDE_FS_B3
#define FFTPDE_FS_B3 3      // Bx and By persistent (C5 512 vs 525 ms per 20-step solve against by_kernel / line Bx)
#endif
// an X-part as the 4D tensor {2 Q M doubles, M rows (m1_l), Q (l1), P (blk)}; boxes of
// 64 bytes x 256 rows (min(M, 256) rows x max(1, 256 / M) blocks)
static bool by_map_part(CUtensorMap &m, const void *p, int M, int P)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t row = (cuuint64_t)G::Q * M * 16;
    cuuint64_t dims[4] = {(cuuint64_t)(2 * G::Q * M), (cuuint64_t)M, (cuuint64_t)G::Q, (cuuint64_t)P};
    cuuint64_t strides[3] = {row, row * M, row * M * G::Q};
    cuuint32_t box[4] = {(cuuint32_t)(2 * ByGeom::W), (cuuint32_t)std::min(M, ByGeom::BOXR), 1,
                         (cuuint32_t)std::max(1, ByGeom::BOXR / M)};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, FFTPDE_FS_PROMO_BY,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// a Y-part for Bx as the 5D tensor {2 MI doubles, M / MI, Q (k1), Q M (rows), P (q)},
// MI = min(M, 128) points; one box = a tile: {2 MI, M / MI, 4 k1, 1 row, P} (FFTPDE_FSD_BXK)
static bool bx_map_part(CUtensorMap &m, const void *p, int M, int P)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    const int MI = std::min(M, 128);
    const cuuint64_t e = 16;
    cuuint64_t dims[5] = {(cuuint64_t)(2 * MI), (cuuint64_t)(M / MI), (cuuint64_t)G::Q, (cuuint64_t)G::Q * M,
                          (cuuint64_t)P};
    cuuint64_t strides[4] = {e * MI, e * M, e * M * G::Q, e * M * G::Q * G::Q * M};
    cuuint32_t box[5] = {(cuuint32_t)(2 * MI), (cuuint32_t)(M / MI), FFTPDE_FSD_BXK ? (cuuint32_t)G::W : 1,
                         FFTPDE_FSD_BXK ? 1 : (cuuint32_t)G::W, (cuuint32_t)P};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, FFTPDE_FS_PROMO_BY,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the peer Y-part q as a By store target: by_map_part with boxes of min(M, 256) rows of one block
static bool by_map_peer(CUtensorMap &m, const void *p, int M, int P)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t row = (cuuint64_t)G::Q * M * 16;
    cuuint64_t dims[4] = {(cuuint64_t)(2 * G::Q * M), (cuuint64_t)M, (cuuint64_t)G::Q, (cuuint64_t)P};
    cuuint64_t strides[3] = {row, row * M, row * M * G::Q};
    cuuint32_t box[4] = {(cuuint32_t)(2 * ByGeom::W), (cuuint32_t)std::min(M, ByGeom::BOXR), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, FFTPDE_FS_PROMO_BY,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool COLS, bool DIST = false>
static cudaError_t launch_b3(void *f, const void *tw32, const double *m2d, cudaStream_t st, const FsPart &pt = FsPart{},
                             const PeerPtrs *peers = nullptr)
{
    using G = B3Geom<COLS>;
    CUtensorMap m;
    if (DIST && COLS) {
        if (!by_map_part(m, f, pt.M, pt.P)) return cudaErrorNotSupported;
    } else if (!DIST && !by_map(m, f, CU_TENSOR_MAP_SWIZZLE_64B)) {
        return cudaErrorNotSupported;
    } else if (DIST && !bx_map_part(m, f, pt.M, pt.P)) {
        return cudaErrorNotSupported;
    }
    PeerPtrs pp{};
    static FsPeerMaps pm;                                    // copied into the launch's parameters
    std::memset(&pm, 0, sizeof pm);
    if (DIST && pt.topeer) {
        if (!peers || pt.P > kMaxPeers || (COLS && pt.P > kFsMaxPeerMaps)) return cudaErrorNotSupported;
        pp = *peers;
        if (COLS)
            for (int r = 0; r < pt.P; ++r)
                if (!by_map_peer(pm.m[r], pp.p[r], pt.M, pt.P)) return cudaErrorNotSupported;
    }
    auto k = b3_kernel<COLS, DIST>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, G::BYTES);
    if (e != cudaSuccess) return e;
    static std::atomic<int> occ_cache{0};
    int occ = occ_cache.load(std::memory_order_relaxed);
    if (occ == 0) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, G::NT, G::BYTES);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        occ_cache.store(occ, std::memory_order_relaxed);
    }
    const unsigned grid = (unsigned)std::min<int64_t>(DIST ? pt.ntiles : G::NTILES, (int64_t)occ * sm_count());
    e = launch_fam(PDL_FOURSTEP, k, dim3(grid), dim3(G::NT), G::BYTES, st, m, (double2 *)f, (const double2 *)tw32, m2d,
                   pt, pp, pm);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
// the B pass of a rank's part (R28): Bx on a Y-part (cols false), By on an X-part (cols true)
cudaError_t launch_fs_b_part(bool cols, int P, int rank, void *f, const void *tw32, const double *m2d, cudaStream_t st,
                             const PeerPtrs *peers)
{
    FsPart pt = fs_part(P, rank, cols ? 1 : 0, 1);
    pt.topeer = peers != nullptr;
    return cols ? launch_b3<true, true>(f, tw32, m2d, st, pt, peers) : launch_b3<false, true>(f, tw32, m2d, st, pt, peers);
}
static int fs_b3_mask()
{
    static const int v = [] { const char *e = std::getenv("FFTPDE_FS_B3"); return e ? std::atoi(e) : FFTPDE_FS_B3; }();
    return v;
}


#ifndef FFTPDE_FS_BX_PIPE
#define FFTPDE_FS_BX_PIPE 0   // the persistent pipe pass for Bx: measured 9.7 vs 8.0 ms per launch, off
#endif
#ifndef FFTPDE_FS_BX_BULK
#define FFTPDE_FS_BX_BULK 0
#endif
#ifndef FFTPDE_FS_BXB_MINB
#define FFTPDE_FS_BXB_MINB 2
#endif
static cudaError_t launch_bx_bulk(void *f, const void *tw32, const double *mx2d, cudaStream_t st)
{
    auto k = bx_kernel<FFTPDE_FS_BXB_MINB>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, BxGeom::BYTES);
    if (e != cudaSuccess) return e;
    e = launch_fam(PDL_FOURSTEP, k, dim3((unsigned)BxGeom::NTILES), dim3(BxGeom::NT), BxGeom::BYTES, st,
                   (double2 *)f, (const double2 *)tw32, mx2d);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}


#ifndef FFTPDE_FS_BB
#define FFTPDE_FS_BB 0
#endif
#ifndef FFTPDE_FS_TEAMS
#define FFTPDE_FS_TEAMS 6
#endif
// Bx + By fused over L2-resident blocks (bb_kernel): a cooperative launch of the
// resident grid; `sync` holds 2 counters per team, zeroed before every launch.
// Opt-in (FFTPDE_FS_BB=1): measured slower than the two passes (C5 B passes 18.8-20.5
// vs 16.5 ms per step for 2-12 teams, r02): halving their HBM traffic does not pay
// because the B passes are bound by their FP64 work and latency (ncu: HBM 66%, FP64
// pipe 50%), and the per-block team barriers add tails.
cudaError_t launch_fs_bb(void *f, const void *tw32, const double *mx2d, const double *my2d, void *sync,
                         cudaStream_t st)
{
    CUtensorMap m;
    if (!by_map(m, f)) return cudaErrorNotSupported;
    auto k = bb_kernel<2>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, BbGeom::BYTES);
    if (e != cudaSuccess) return e;
    static std::atomic<int> occ_cache{0};
    int occ = occ_cache.load();
    if (!occ) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, BbGeom::NT, BbGeom::BYTES);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorNotSupported;
        occ_cache.store(occ);
    }
    int teams = FFTPDE_FS_TEAMS;
    if (const char *s = std::getenv("FFTPDE_FS_TEAMS")) teams = std::max(1, atoi(s));
    e = cudaMemsetAsync(sync, 0, 2 * sizeof(unsigned) * (size_t)teams, st);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    int grid = occ * sm_count();
    if (const char *s = std::getenv("FFTPDE_FS_BB_GRID")) grid = std::max(teams, std::min(grid, atoi(s)));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(BbGeom::NT);
    cfg.dynamicSmemBytes = BbGeom::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, m, (double2 *)f, (const double2 *)tw32, mx2d, my2d, (unsigned *)sync, teams);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
bool fs_bb_enabled()
{
    static const bool on = [] { const char *e = std::getenv("FFTPDE_FS_BB"); return e ? e[0] != '0' : FFTPDE_FS_BB != 0; }();
    return on;
}

#ifndef FFTPDE_FS_BY_W
#define FFTPDE_FS_BY_W 4
#endif
#ifndef FFTPDE_FS_BY_E
#define FFTPDE_FS_BY_E 32
#endif
#ifndef FFTPDE_FS_BY_MINB
#define FFTPDE_FS_BY_MINB 2
#endif
#ifndef FFTPDE_FS_BX_W
#define FFTPDE_FS_BX_W 1
#endif
#ifndef FFTPDE_FS_BX_E
#define FFTPDE_FS_BX_E 32
#endif
#ifndef FFTPDE_FS_BX_MINB
#define FFTPDE_FS_BX_MINB 4
#endif
// The B passes: 1024-point line diffusion with the 2D factor (OpTables::ey2d).
// Bx: rows of 1024 points (32 per grid row), line class = row % 32;
// By: 32 blocks of 1024 rows, W adjacent columns per CTA, class = block.
cudaError_t launch_fs_b(bool cols, void *f, const void *tw32, const void *tw16, const OpTables<double> &tab,
                        cudaStream_t st)
{
    using G = FsGeom;
    if (fs_b3_mask() & (cols ? 2 : 1)) {
        const cudaError_t e = cols ? launch_b3<true>(f, tw32, tab.ey2d, st) : launch_b3<false>(f, tw32, tab.ey2d, st);
        if (e != cudaErrorNotSupported) return e;
    }
    if (!cols && FFTPDE_FS_BX_BULK) return launch_bx_bulk(f, tw32, tab.ey2d, st);
    if (!cols && FFTPDE_FS_BX_PIPE) {      // persistent double-buffered pipe pass (radix 16, 4 rows per tile)
        OpTables<double> t = tab;
        PipeArgs a{(int64_t)G::N * G::Q, 1024, 1, (int64_t)G::N * G::N, 1, 0, PIPE_DIFFUSE, nullptr};
        return pipe_n<double, 1024, false, PIPE_DIFFUSE>(f, f, a, tw16, t, st);
    }
    if (!cols)
        return line_n<double, 1024, FFTPDE_FS_BX_E, FFTPDE_FS_BX_W, false, LN_DIFFUSE, FFTPDE_FS_BX_MINB>(
            f, f, nullptr, (int64_t)G::N * G::Q, 1024, 1, (int64_t)G::N * G::N, 1, FFTPDE_FS_BX_E == 32 ? tw32 : tw16,
            tab, st, PeerOut{}, PDL_FOURSTEP);
    if (FFTPDE_FS_BY_TMA) {
        const cudaError_t e = launch_by_tma(f, tw32, tab.ey2d, st);
        if (e != cudaErrorNotSupported) return e;
    }
    return line_n<double, 1024, FFTPDE_FS_BY_E, FFTPDE_FS_BY_W, true, LN_DIFFUSE, FFTPDE_FS_BY_MINB>(
        f, f, nullptr, G::N, 1, G::N, (int64_t)1024 * G::N, G::Q, FFTPDE_FS_BY_E == 32 ? tw32 : tw16, tab, st,
        PeerOut{}, PDL_FOURSTEP);
}

} // namespace fftpde
