// tpipe.cuh -- row pass with a transposed-spectrum side (sm_100a).
//
// Multi-step solves keep the row spectrum TRANSPOSED in the workspace,
// T[b][a][k] = P^x_{a,k} (the x-transform of row k at wavenumber a, PAPER.md:
// 262-266), so the y-pass "forward along y, k-space operator, inverse along y"
// (PAPER.md:266-273 + the multiplier of eq:SolutionPoisson / solCalorFourier)
// becomes a pass over contiguous lines of T.  This kernel is the x-pass on the
// other side of that layout:
//   TP_FWD_T : natural rows in        -> forward x-transform -> T columns out
//   TP_MID_T : T columns in -> inverse x-transform -> natural rows (the
//              materialised physical field, out2) -> forward x-transform of the
//              next step -> T columns out
//   TP_INV_T : T columns in -> inverse x-transform -> natural rows out
// A tile is W consecutive rows k; on the T side each (a, k0..k0+W-1) is a
// W*sizeof(C)-byte segment (>= 32 B: whole sectors), loaded with cp.async and
// stored through the tile buffer column-fastest, like the column pass.
// Persistent CTAs, NBUF-deep cp.async ring as in pipe.cuh.
#pragma once
#include "../../paper_2412_12308_b200/csrc/pipe.cuh"

namespace fftpde {

enum TPipeOp { TP_FWD_T = 0, TP_MID_T = 1, TP_INV_T = 2 };

struct TPipeArgs {
    int64_t nrows;    // rows per grid (ny)
    int64_t nx, ny;   // natural row length (== N) and column length
    int64_t bs_nat;   // elements between grids of the natural arrays
    int64_t bs_t;     // elements between grids of the transposed spectrum
    int64_t ntiles;   // batch * groups
    int64_t groups;   // ceil(nrows / W)
    void *out2;       // TP_MID_T: physical-field output (natural layout)
};

template <typename T, int N, int W, int OP, int NBUF, bool TWREG>
__global__ void __launch_bounds__(W * Shape<N>::TPT, 1)
tpipe_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out, TPipeArgs a,
             const typename cplx_t<T>::type *__restrict__ tw)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N>;
    using L = PipeSmem<C, N, W, true, NBUF>;
    constexpr int E = S::E, TPT = S::TPT;
    constexpr bool IN_T = OP != TP_FWD_T, OUT_T = OP != TP_INV_T;
    static_assert(TPT <= 32 || W <= 15, "one named barrier per line");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *buf0 = reinterpret_cast<C *>(smem_raw);

    const int tid = threadIdx.x;
    const int c = tid / TPT, t = tid % TPT;        // transform layout (line-major)
    const int lc = tid % W, lt = tid / W;          // transposed-side layout (row-fastest)
    const LineSync<TPT> lsync{1 + c};

    auto tile_rows = [&](int64_t tile, int64_t &b) -> int64_t {   // first row k0 of the tile
        b = tile / a.groups;
        return (tile - b * a.groups) * W;
    };
    auto buf = [&](int slot, int cc) { return buf0 + (size_t)slot * (L::BUF / sizeof(C)) + cc * L::S; };
    auto issue = [&](int64_t tile, int slot) {
        int64_t b;
        const int64_t k0 = tile_rows(tile, b);
        if constexpr (IN_T) {
            if (k0 + lc < a.nrows) {
                const C *src = in + b * a.bs_t + (int64_t)lt * a.ny + k0 + lc;
                C *dst = buf(slot, lc) + padidx(lt, S::LOGE);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int o = TPT % E == 0 ? SmemView<C, S::LOGE, 1>::off(TPT * e)
                                               : padidx(lt + TPT * e, S::LOGE) - padidx(lt, S::LOGE);
                    cp_async_n<sizeof(C)>(dst + o, src + (int64_t)e * TPT * a.ny);
                }
            }
        } else {
            if (k0 + c < a.nrows) {
                const C *src = in + b * a.bs_nat + (k0 + c) * a.nx + t;
                C *dst = buf(slot, c) + padidx(t, S::LOGE);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int o = TPT % E == 0 ? SmemView<C, S::LOGE, 1>::off(TPT * e)
                                               : padidx(t + TPT * e, S::LOGE) - padidx(t, S::LOGE);
                    cp_async_n<sizeof(C)>(dst + o, src + e * TPT);
                }
            }
        }
        cp_async_commit();
    };

    using TwP = std::conditional_t<TWREG, TwReg<N, C>, TwL1<N, C>>;
    TwP twp;
    if constexpr (TWREG) twp.load(tw, t);
    else twp = TwL1<N, C>{tw, t};

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
        if constexpr (NBUF > 1) {
            if (next < a.ntiles) issue(next, (it + NBUF - 1) % NBUF);
            else cp_async_commit();
            cp_async_wait<NBUF - 1>();
        } else {
            if (it == 0) { if (tile < a.ntiles) issue(tile, 0); else cp_async_commit(); }
            cp_async_wait<0>();
        }
        if constexpr (IN_T) __syncthreads();        // copies were issued in the other layout
        int64_t b;
        const int64_t k0 = tile_rows(tile, b);
        const bool active = k0 + c < a.nrows;

        SmemView<C, S::LOGE, 1> sm{buf(slot, c)};
        C v[E];
        if constexpr (TPT % E == 0) {
            const C *rp = sm.ptr(t);
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = rp[decltype(sm)::off(TPT * e)];
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = sm.at(t + TPT * e);
        }
        lsync();
        fft_tw<N, IN_T>(v, sm, t, twp, lsync);     // inverse when coming from the spectrum
        if constexpr (OP == TP_MID_T) {
            if (active) {
                C *dst = opaque_ptr(reinterpret_cast<C *>(a.out2) + b * a.bs_nat + (k0 + c) * a.nx + t);
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e * TPT] = v[e];
            }
            fft_tw<N, false>(v, sm, t, twp, lsync);
        }
        if constexpr (!OUT_T) {
            if (active) {
                C *dst = opaque_ptr(out + b * a.bs_nat + (k0 + c) * a.nx + t);
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e * TPT] = v[e];
            }
            // the next issue refills other lines' buffers (transposed-side layout)
            if constexpr (NBUF > 1) __syncthreads();
        } else {
            // stage through the (free) tile buffer, store row-fastest into T
            if constexpr (TPT % E == 0) {
                C *wp = sm.ptr(t);
#pragma unroll
                for (int e = 0; e < E; ++e) wp[decltype(sm)::off(TPT * e)] = v[e];
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) sm.at(t + TPT * e) = v[e];
            }
            __syncthreads();
            if (k0 + lc < a.nrows) {
                const C *src = buf(slot, lc) + padidx(lt, S::LOGE);
                C *dst = opaque_ptr(out + b * a.bs_t + (int64_t)lt * a.ny + k0 + lc);
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int o = TPT % E == 0 ? SmemView<C, S::LOGE, 1>::off(TPT * e)
                                               : padidx(lt + TPT * e, S::LOGE) - padidx(lt, S::LOGE);
                    dst[(int64_t)e * TPT * a.ny] = src[o];
                }
            }
            if constexpr (NBUF > 1) __syncthreads();
        }
        if constexpr (NBUF == 1) {
            __syncthreads();
            const int64_t nxt = tile + gridDim.x;
            if (nxt < a.ntiles) issue(nxt, 0);
        }
    }
    cp_async_wait<0>();
}

} // namespace fftpde
