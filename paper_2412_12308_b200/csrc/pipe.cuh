// pipe.cuh -- persistent, double-buffered line-FFT pass (rows or columns).
//
// One CTA per SM slot loops over tiles of W lines (rows along x, or columns
// along y).  While tile i is transformed from shared-memory buffer A, the
// loads of tile i+1 are already in flight into buffer B (cp.async, one
// 16 B / 8 B copy per element, issued by the thread that will consume it), so
// HBM reads overlap the FP64 butterflies; results go straight from registers
// to global memory.  A buffer doubles as the transform's exchange buffer once
// its tile has been read into registers.
//
// Per line: a forward transform along the line (eq:DFT sign
// +), optionally the k-space operator of the column pass and the inverse
// transform (conjugate kernel).
#pragma once
#include <type_traits>
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

// PIPE_INV is the unscaled inverse (row pass); PIPE_INV_SCALED multiplies by
// tab.scale = 1/(nx ny) first (standalone inverse column pass).
// PIPE_MID (rows): the inverse transform of step s (stored to out2: the
// materialised physical field) followed by the forward transform of step s+1
// (stored to out), one HBM read for both.
enum PipeOp { PIPE_FWD = 0, PIPE_INV_SCALED = 1, PIPE_POISSON = 2, PIPE_DIFFUSE = 3, PIPE_INV = 4, PIPE_MID = 5 };

template <int BYTES> __device__ __forceinline__ void cp_async_n(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Shared-memory pitch (elements) of one line buffer: the padded line, plus an
// offset so that the lines sharing one 128-byte smem phase use distinct banks.
template <typename C, int N, int W, bool COLS, int NBUF = 2> struct PipeSmem {
    static constexpr int LPP = 128 / (int)sizeof(C);           // elements per smem phase
    static constexpr int TPT = Shape<N>::TPT;
    static constexpr int RAW = Shape<N>::PADDED;
    static constexpr int LINES_PER_PHASE = COLS ? (W < LPP ? W : LPP) : (TPT < LPP ? LPP / TPT : 1);
    static constexpr int S = LINES_PER_PHASE <= 1 ? RAW
                           : ((RAW + LPP - 1) / LPP) * LPP + LPP / LINES_PER_PHASE;
    static constexpr size_t BUF = (size_t)W * S * sizeof(C);
    static constexpr size_t BYTES = NBUF * BUF;
};

struct PipeArgs {
    int64_t nlines;       // lines per grid (rows: ny, columns: nx)
    int64_t line_stride;  // elements between consecutive lines (rows: nx, columns: 1)
    int64_t elem_stride;  // elements between consecutive points of a line (rows: 1, columns: nx)
    int64_t batch_stride; // elements between grids
    int64_t ntiles;       // batch * ceil(nlines / W)
    int64_t groups;       // ceil(nlines / W)
    int op;               // PipeOp
    void *out2;           // PIPE_MID: physical-field output (same layout as out)
};

// Per-line barrier: the TPT threads of line c (line-major thread layout).
template <int TPT> struct LineSync {
    int id;
    __device__ __forceinline__ void operator()() const
    {
        if constexpr (TPT <= 32) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(TPT) : "memory");
    }
};

// Threads are laid out line-major for the transforms (thread t of line c =
// c*TPT + t), so each line synchronises on its own barrier (a warp barrier when
// TPT <= 32) and the W lines of a tile progress independently.  Column tiles
// are loaded and stored column-fastest (W*sizeof(C)-byte row segments), with
// the results staged through the tile buffer for the store.
// BULK (rows only): each line of a tile arrives as ONE bulk copy (cp.async.bulk,
// the 1D form of the tensor memory accelerator) issued by the line's first
// thread and counted on a per-(slot, line) mbarrier, instead of E 16-byte
// cp.async per thread: no per-element copy instructions in the memory pipeline.
// The row lands dense at the start of its line buffer and is read dense.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
// the reverse: shared -> global, completion tracked by the issuing thread's bulk async-group
__device__ __forceinline__ void bulk_s2g(void *dst, uint32_t src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_expect(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_wait(uint32_t mbar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n"
                 "BW%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra BW%=;\n}" ::"r"(mbar), "r"(parity) : "memory");
}

template <typename T, int N, int W, bool COLS, int OP, int NBUF, int MINB = 1, bool TWREG = false, bool BULK = false>
__global__ void __launch_bounds__(W * Shape<N>::TPT, MINB)
pipe_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out, PipeArgs a,
            const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab, PeerOut po)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N>;
    using L = PipeSmem<C, N, W, COLS, NBUF>;
    constexpr int E = S::E, TPT = S::TPT;
    static_assert(TPT <= 32 || W <= 15, "one named barrier per line");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *buf0 = reinterpret_cast<C *>(smem_raw);

    const int tid = threadIdx.x;
    const int c = tid / TPT, t = tid % TPT;                  // transform layout (line-major)
    const int lc = COLS ? tid % W : c;                        // load/store layout
    const int lt = COLS ? tid / W : t;
    const int64_t estep = (int64_t)TPT * a.elem_stride;
    constexpr bool INV1 = OP == PIPE_INV || OP == PIPE_INV_SCALED || OP == PIPE_MID;   // first transform inverse
    constexpr bool TWO = OP == PIPE_POISSON || OP == PIPE_DIFFUSE;   // forward, operator, inverse
    const LineSync<TPT> lsync{1 + c};

    // global offset of element lt of line lc of tile `tile`; -1 if past the end
    auto line_base = [&](int64_t tile, int cc, int tt) -> int64_t {
        const int64_t b = tile / a.groups;
        const int64_t line = (tile - b * a.groups) * W + cc;
        if (line >= a.nlines) return -1;
        return b * a.batch_stride + line * a.line_stride + (int64_t)tt * a.elem_stride;
    };
    auto buf = [&](int slot, int cc) { return buf0 + (size_t)slot * (L::BUF / sizeof(C)) + cc * L::S; };
    static_assert(!BULK || !COLS, "bulk copies load whole rows");
    // BULK: mbarrier of (slot, line) at the end of the ring buffers
    const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(smem_raw + (BULK ? L::BYTES : 0));
    auto issue = [&](int64_t tile, int slot) {
        if constexpr (BULK) {
            if (t == 0) {
                const int64_t base = line_base(tile, c, 0);
                if (base >= 0) {
                    const uint32_t mb = mbar0 + 8u * (uint32_t)(slot * W + c);
                    bulk_expect(mb, (uint32_t)(N * sizeof(C)));
                    bulk_g2s((uint32_t)__cvta_generic_to_shared(buf(slot, c)), in + base, (uint32_t)(N * sizeof(C)), mb);
                }
            }
            return;
        }
        const int64_t base = line_base(tile, lc, lt);
        if (base >= 0) {
            C *dst = buf(slot, lc) + padidx(lt, S::LOGE);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int o = TPT % E == 0 ? SmemView<C, S::LOGE, 1>::off(TPT * e)
                                           : padidx(lt + TPT * e, S::LOGE) - padidx(lt, S::LOGE);
                cp_async_n<sizeof(C)>(dst + o, in + base + e * estep);
            }
        }
        cp_async_commit();
    };

    using TwP = std::conditional_t<TWREG, TwReg<N, C>, TwL1<N, C>>;
    TwP twp;
    if constexpr (TWREG) twp.load(tw, t);
    else twp = TwL1<N, C>{tw, t};
    if constexpr (BULK) {
        if (tid < NBUF * W) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar0 + 8u * tid) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncthreads();
    }
    pdl_wait();

    // ring of NBUF tile buffers: tile i lives in slot i % NBUF; the loads of the
    // next NBUF-1 tiles are in flight while tile i is transformed
    int64_t tile = blockIdx.x;
#pragma unroll
    for (int j = 0; j < NBUF - 1; ++j) {
        const int64_t pre = tile + (int64_t)j * gridDim.x;
        if (pre < a.ntiles) issue(pre, j);
        else cp_async_commit();
    }
    for (int it = 0; tile < a.ntiles; ++it, tile += gridDim.x) {
        const int slot = it % NBUF;
        const int64_t next = tile + (int64_t)(NBUF - 1) * gridDim.x;
        if (tile + gridDim.x >= a.ntiles) pdl_trigger();   // this CTA's last tile
        if constexpr (BULK) {
            if (NBUF > 1 && next < a.ntiles) issue(next, (it + NBUF - 1) % NBUF);
            if (NBUF == 1 && it == 0) issue(tile, 0);
            if (line_base(tile, c, 0) >= 0) bulk_wait(mbar0 + 8u * (uint32_t)(slot * W + c), (uint32_t)(it / NBUF) & 1u);
        } else if constexpr (NBUF > 1) {
            if (next < a.ntiles) issue(next, (it + NBUF - 1) % NBUF);
            else cp_async_commit();                  // keep the group count uniform
            cp_async_wait<NBUF - 1>();               // this thread's copies of `tile` landed
        } else {
            if (it == 0) { if (tile < a.ntiles) issue(tile, 0); else cp_async_commit(); }
            cp_async_wait<0>();
        }
        if constexpr (COLS) __syncthreads();         // copies were issued in the other layout

        SmemView<C, S::LOGE, 1> sm{buf(slot, c)};
        C v[E];
        if constexpr (BULK) {                        // the row arrived dense
            const C *rp = buf(slot, c);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = rp[t + TPT * e];
        } else if constexpr (TPT % E == 0) {         // inactive lines read (unused) garbage
            const C *rp = sm.ptr(t);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = rp[decltype(sm)::off(TPT * e)];
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = sm.at(t + TPT * e);
        }
        if constexpr (OP == PIPE_INV_SCALED) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = cscale(v[e], tab.scale);
        }
        lsync();                                     // the line's inputs are read: buffer reusable
        fft_tw<N, INV1>(v, sm, t, twp, lsync);
        if constexpr (TWO) {
            // k-space operator at (a, b): the line is column a, element e is row b
            int64_t col = (tile - (tile / a.groups) * a.groups) * W + c;
            if (col >= a.nlines) col = 0;
            if constexpr (OP == PIPE_POISSON) {
                const T kxa = tab.kx2[col];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const T k2 = kxa + __ldg(&tab.ky2[t + TPT * e]);
                    const T m = poisson_mul(k2, tab.scale);     // -1/|k|^2, k = 0 zeroed
                    v[e] = cscale(v[e], m);
                }
            } else if (tab.ey2d) {                   // four-step B pass: factor of line class cls
                const int64_t cls = COLS ? tile / a.groups : col % tab.ey2d_mod;
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = cscale(v[e], __ldg(&tab.ey2d[cls * N + t + TPT * e]));
            } else {
                const T exa = tab.ex[col];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const T m = exa * __ldg(&tab.ey[t + TPT * e]);      // exp(-D|k|^2 dt)/(nx ny)
                    v[e] = cscale(v[e], m);
                }
            }
            fft_tw<N, true>(v, sm, t, twp, lsync);
        }
        if constexpr (OP == PIPE_MID) {
            static_assert(!COLS, "PIPE_MID is a row pass");
            const int64_t base = line_base(tile, c, t);
            if (base >= 0) {
                C *dst = opaque_ptr(reinterpret_cast<C *>(a.out2) + base);
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
            }
            fft_tw<N, false>(v, sm, t, twp, lsync);
        }
        if constexpr (!COLS) {
            const int64_t base = line_base(tile, c, t);
            if (base >= 0 && po.p[0]) {              // rows scattered into the peers' column slabs
                const int64_t k = (tile - (tile / a.groups) * a.groups) * W + c;
#pragma unroll
                for (int e = 0; e < E; ++e) *opaque_ptr(peer_row_dst<C>(po, k, t + TPT * e)) = v[e];
            } else if (base >= 0) {
                C *dst = opaque_ptr(out + base);
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
            }
        } else {
            // stage through the (free) tile buffer, store column-fastest
            if constexpr (TPT % E == 0) {
                C *wp = sm.ptr(t);
#pragma unroll
                for (int e = 0; e < E; ++e) wp[decltype(sm)::off(TPT * e)] = v[e];
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) sm.at(t + TPT * e) = v[e];
            }
            __syncthreads();
            const int64_t base = line_base(tile, lc, lt);
            if (base >= 0 && po.p[0]) {              // scattered into the owners' row slabs
                const C *src = buf(slot, lc) + padidx(lt, S::LOGE);
                const int64_t col = (tile - (tile / a.groups) * a.groups) * W + lc;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int o = TPT % E == 0 ? SmemView<C, S::LOGE, 1>::off(TPT * e)
                                               : padidx(lt + TPT * e, S::LOGE) - padidx(lt, S::LOGE);
                    *opaque_ptr(peer_col_dst<C>(po, lt + TPT * e, col)) = src[o];
                }
            } else if (base >= 0) {
                const C *src = buf(slot, lc) + padidx(lt, S::LOGE);
                C *dst = opaque_ptr(out + base);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int o = TPT % E == 0 ? SmemView<C, S::LOGE, 1>::off(TPT * e)
                                               : padidx(lt + TPT * e, S::LOGE) - padidx(lt, S::LOGE);
                    dst[e * estep] = src[o];
                }
            }
            if constexpr (NBUF > 1) __syncthreads();     // slot is refilled by the next issue
        }
        if constexpr (NBUF == 1) {
            if constexpr (!COLS) lsync();
            else __syncthreads();
            const int64_t nxt = tile + gridDim.x;
            if (nxt < a.ntiles) issue(nxt, 0);       // the buffer is free after the last use
        }
    }
    if constexpr (!BULK) cp_async_wait<0>();
}

} // namespace fftpde
