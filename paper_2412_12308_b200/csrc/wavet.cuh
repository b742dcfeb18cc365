// wavet.cuh -- the wave solve (C3) on a transposed internal spectrum (sm_100a).
//
// The wave step (eq:OmegaZero / eq:OmegaNonZero) couples the two
// fields only in k-space: per step, forward transforms of U and V, the 2x2
// oscillator update (C, S1; S2, C) at every k, inverse transforms.  Between the
// row pass and the column pass the fields live in the solver's own scratch, so
// their layout is free: here the row-transformed spectrum is stored TRANSPOSED,
// T[kx][y] (y fastest).  The column pass then reads every column as one
// contiguous 64 KiB run (one bulk copy each way), instead of 4096 rows of 16
// bytes -- a pattern that copies at 2.2 TB/s on B200 against 5.4 TB/s for
// 32-byte granules (tools/exp_c3_gran.cu).  The row pass pays for the transpose
// in 32-byte granules: a cluster pair owns the row pair (y0, y0+1); CTA c holds
// row y0+c in registers but moves the tile T[kx in half c][y0..y0+1] (2048 x 32
// bytes, TMA boxes of 256 x 32 B), the other row's half travelling over DSMEM
// (st.async into the partner, completing on its mbarrier).
//
// wavet_rows_kernel<OP> (one row pair per cluster, 2 x 128 threads, radix 32):
//   FWD: physical rows -> forward row FFT -> T          (the first step)
//   MID: T -> inverse row FFT -> physical rows (u materialised) -> forward -> T
//   INV: T -> inverse row FFT -> physical rows          (the last step)
// wavet_cols_kernel (one column kx per cluster pair, CTA f = field f): bulk load
// of T[kx][*], forward column FFT, the partner's spectrum over DSMEM for the
// oscillator update (as tma_wave2_cols_kernel), inverse, bulk store.
#pragma once
#include "tmacols.cuh"

namespace fftpde {

template <int NX> struct WaveTRowGeom {
    static constexpr int E = 32, TPT = NX / E;                      // 128 threads per row
    static constexpr int H = NX / 2;                                // kx half per CTA
    static constexpr int BOXK = 256, NBOX = H / BOXK;               // TMA boxes of 256 kx x 32 bytes
    static constexpr size_t TILE = (size_t)H * 32;                  // [H][2] complex128
    static constexpr size_t XCH = (size_t)Shape<NX, E>::PADDED * 16;
    static constexpr size_t LINE = ((TILE > XCH ? TILE : XCH) + 127) / 128 * 128;
    static constexpr size_t RECV = (size_t)H * 16;
    static constexpr size_t BYTES = LINE + RECV + 128 + 64;         // + alignment, 4 mbarriers
    static_assert(H % (TPT * 1) == 0 && H / TPT == E / 2, "half a row = e < E/2");
};

__device__ __forceinline__ void mbar_remote_arrive_relaxed(uint32_t cluster_addr)
{
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void fence_release_cta_to_cluster()
{
    asm volatile("fence.release.sync_restrict::shared::cta.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t mbar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n"
                 "W%=:\n\t"
                 "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W%=;\n}" ::"r"(mbar), "r"(parity) : "memory");
    asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}

// Rows: grid = 2 x ny/2 CTAs in clusters of 2; cluster p owns rows 2p, 2p+1.
// tmap: T viewed as [nx][ny] complex128, box {2 complex (y, y+1), 256 kx}.
template <int NX, int OP>
__global__ void __launch_bounds__(WaveTRowGeom<NX>::TPT, 1)
wavet_rows_kernel(const __grid_constant__ CUtensorMap tmap, const double2 *__restrict__ phys_in,
                  double2 *phys_out, int64_t ny, const double2 *__restrict__ tw)
{
    using G = WaveTRowGeom<NX>;
    using S = Shape<NX, G::E>;
    constexpr int E = G::E, TPT = G::TPT, H = G::H, HE = E / 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((128u - (tma_smem(smem_raw) & 127u)) & 127u);
    double2 *tile = reinterpret_cast<double2 *>(base);             // [H][2] granules, then the exchange buffer
    double2 *recv = reinterpret_cast<double2 *>(base + G::LINE);    // the partner's push of my row's other half
    const uint32_t full = tma_smem(base + G::LINE + G::RECV);
    const uint32_t recv1 = full + 8, freed = full + 16, recv2 = full + 24;
    const int t = threadIdx.x;
    const uint32_t c = cl_rank();                                   // my row: y0 + c; my kx half: c
    const int64_t y0 = 2 * (int64_t)(blockIdx.x / 2);
    const int64_t y = y0 + c;
    constexpr bool IN_T = OP != WT_FWD, OUT_T = OP != WT_INV;
    if (t == 0) {
        tma_mbar_init(full, 1);
        tma_mbar_init(recv1, 1);
        tma_mbar_init(freed, 1);
        tma_mbar_init(recv2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncthreads();
    cl_arrive_relaxed();                                            // my mbarriers exist
    pdl_wait();
    if (t == 0) {
        if constexpr (IN_T) {
            tma_mbar_expect(full, (uint32_t)G::TILE);
            tma_mbar_expect(recv1, (uint32_t)G::RECV);
#pragma unroll
            for (int k = 0; k < G::NBOX; ++k)
                tma_load3(tma_smem(tile) + k * G::BOXK * 32, &tmap, (int)(2 * y0), (int)(c * H + k * G::BOXK), 0, full);
        }
        if constexpr (OUT_T) tma_mbar_expect(recv2, (uint32_t)G::RECV);
    }
    pdl_trigger();
    const uint32_t peer = c ^ 1u;
    cl_wait_acquire();                                              // the partner's mbarriers exist
    double2 v[E];
    if constexpr (IN_T) {
        tma_mbar_wait(full, 0);
        // push the partner's row in my kx half: tile[kl][peer] -> partner's recv[kl]
        const uint32_t precv = mapa_rank(tma_smem(recv), peer), pm = mapa_rank(recv1, peer);
#pragma unroll
        for (int e = 0; e < HE; ++e) {
            const int kl = t + TPT * e;
            st_async(precv + (uint32_t)(kl * 16), tile[2 * kl + peer], pm);
        }
        // my row: kx = t + TPT e; e < HE is kx < H (half 0)
#pragma unroll
        for (int e = 0; e < E; ++e)
            if ((e < HE) == (c == 0)) v[e] = tile[2 * (t + TPT * (e % HE)) + c];
        tma_mbar_wait(recv1, 0);
#pragma unroll
        for (int e = 0; e < E; ++e)
            if ((e < HE) != (c == 0)) v[e] = recv[t + TPT * (e % HE)];
        __syncthreads();                                            // the tile is free: exchange buffer
    } else {
        const double2 *src = phys_in + y * NX;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = src[t + TPT * e];
    }
    const SmemView<double2, S::LOGE, 1> sm{tile};
    const SyncCTA sync{};
#if FFTPDE_TWPOW
    const TwL1Pow<NX, double2, E> twp{{tw, t}};
#else
    const TwL1<NX, double2, E> twp{tw, t};
#endif
    if constexpr (IN_T) {
        fft_tw<NX, true, E>(v, sm, t, twp, sync);                   // inverse along x (unscaled)
        double2 *dst = opaque_ptr(phys_out + y * NX);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[t + TPT * e] = v[e];        // u of this step, materialised
    }
    if constexpr (OUT_T) {
        fft_tw<NX, false, E>(v, sm, t, twp, sync);                  // forward along x (the next step)
        // my tile is free (fft_tw ends with a barrier): tell the partner it may push into it
        if (t == 0) {
            fence_release_cta_to_cluster();
            mbar_remote_arrive_relaxed(mapa_rank(freed, peer));
        }
        // my values in my half -> my tile[kl][c]; the rest -> the partner's tile[kl][c]
#pragma unroll
        for (int e = 0; e < E; ++e)
            if ((e < HE) == (c == 0)) tile[2 * (t + TPT * (e % HE)) + c] = v[e];
        mbar_wait_cluster(freed, 0);
        const uint32_t ptile = mapa_rank(tma_smem(tile), peer), pm = mapa_rank(recv2, peer);
#pragma unroll
        for (int e = 0; e < E; ++e)
            if ((e < HE) != (c == 0)) st_async(ptile + (uint32_t)((2 * (t + TPT * (e % HE)) + c) * 16), v[e], pm);
        tma_mbar_wait(recv2, 0);                                    // the partner's row is in my tile
        tma_fence_smem();
        __syncthreads();
        if (t == 0) {
#pragma unroll
            for (int k = 0; k < G::NBOX; ++k)
                tma_store3(&tmap, (int)(2 * y0), (int)(c * H + k * G::BOXK), 0, tma_smem(tile) + k * G::BOXK * 32);
            tma_commit();
            tma_wait_read0();
        }
    }
}

// Columns of the transposed spectra: column kx of field f is T_f[kx][0..NY).
template <int NY> struct WaveTColGeom {
    static constexpr int E = 32, TPT = NY / E;
    static constexpr size_t LINE = ((size_t)Shape<NY, E>::PADDED * 16 + 127) / 128 * 128;
    static constexpr size_t BYTES = LINE + 128 + 16;
};

template <int NY>
__global__ void __launch_bounds__(WaveTColGeom<NY>::TPT, 1)
wavet_cols_kernel(double2 *TU, double2 *TV, const double2 *__restrict__ tw, OpTables<double> tab)
{
    using G = WaveTColGeom<NY>;
    using S = Shape<NY, G::E>;
    constexpr int E = G::E, TPT = G::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((128u - (tma_smem(smem_raw) & 127u)) & 127u);
    double2 *line = reinterpret_cast<double2 *>(base);
    const uint32_t mbar = tma_smem(base + G::LINE);
    const int t = threadIdx.x;
    const uint32_t f = cl_rank();
    const int64_t a = blockIdx.x / 2;                               // kx
    double2 *col = (f ? TV : TU) + a * NY;
    const SyncCTA sync{};
    if (t == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    if (t == 0) {
        bulk_expect(mbar, (uint32_t)(NY * 16));
        bulk_g2s(tma_smem(base), col, (uint32_t)(NY * 16), mbar);
    }
    pdl_trigger();
    tma_mbar_wait(mbar, 0);
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = line[t + TPT * e];
    __syncthreads();
    const SmemView<double2, S::LOGE, 1> sm{line};
#if FFTPDE_TWPOW
    const TwL1Pow<NY, double2, E> twp{{tw, t}};
#else
    const TwL1<NY, double2, E> twp{tw, t};
#endif
    fft_tw<NY, false, E>(v, sm, t, twp, sync);
#pragma unroll
    for (int e = 0; e < E; ++e) line[t + TPT * e] = v[e];
    cl_arrive_release();                                            // my spectrum is visible to the partner
    cl_wait_acquire();
    {
        const uint32_t peer = mapa_rank(tma_smem(base), f ^ 1u);
        const int64_t qa = a <= tab.nfold - a ? a : tab.nfold - a;
        const double *pC = tab.wC + qa * tab.qpitch, *pS = (f ? tab.wS2 : tab.wS1) + qa * tab.qpitch;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int b = t + TPT * e;
            const int qb = b <= NY - b ? b : NY - b;
            const double cc = __ldg(pC + qb), ss = __ldg(pS + qb);
            const double2 o = ld_cluster(peer + (uint32_t)(b * 16));
            v[e] = double2{cc * v[e].x + ss * o.x, cc * v[e].y + ss * o.y};   // U: C U + S1 V; V: S2 U + C V
        }
    }
    cl_arrive_release();                                            // done reading the partner's line
    cl_wait_acquire();
    fft_tw<NY, true, E>(v, sm, t, twp, sync);
#pragma unroll
    for (int e = 0; e < E; ++e) line[t + TPT * e] = v[e];
    tma_fence_smem();
    __syncthreads();
    if (t == 0) {
        bulk_s2g(col, tma_smem(base), (uint32_t)(NY * 16));
        tma_commit();
        tma_wait_read0();
    }
}

} // namespace fftpde
