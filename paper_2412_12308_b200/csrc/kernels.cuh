// kernels.cuh -- pass kernels of the 2D FFT-PDE hot path (sm_100a).
//
// A solve step is three HBM passes:
//   row_fft      : forward transform along x of every row
//   col_fused    : forward transform along y of W adjacent columns, the k-space
//                  operator (with 1/(nx ny) folded in), inverse transform along y
//                  (PAPER.md:266-273 + eq:SolutionPoisson / solCalorFourier /
//                  eq:OmegaZero-NonZero)
//   row_fft      : inverse transform along x (conjugate in/out)
// and a single-CTA kernel (small_solve) keeps a whole small grid in shared
// memory for one HBM round trip (C1).
#pragma once
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

// conj-on-the-fly load/store helpers
template <typename C> __device__ __forceinline__ C ld(const C *p, bool cj)
{
    C v = *p;
    return cj ? cconj(v) : v;
}

// Smem pitch (in complex elements) of one column buffer so that W columns
// accessed by the lanes of one shared-memory phase hit distinct banks:
// a phase is 128 B = LPP elements; column c starts at c*S with S = LPP/W mod LPP.
template <typename C, int N, int W> struct ColSmem {
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int RAW = Shape<N>::PADDED;
    static constexpr int S = W == 1 ? RAW : ((RAW + LPP - 1) / LPP) * LPP + (W >= LPP ? 1 : LPP / W);
    static constexpr size_t BYTES = (size_t)W * S * sizeof(C);
};

// ---------------------------------------------------------------------------
// Row pass: ROWS rows of length N per CTA, Shape<N>::TPT threads per row.
// in/out may alias (each thread reads its own elements before writing them).
template <typename T, int N, int ROWS>
__global__ void __launch_bounds__(ROWS * Shape<N>::TPT)
row_fft_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out,
               int64_t ny, int64_t stride, int64_t total_rows, int conj_io,
               const typename cplx_t<T>::type *__restrict__ tw)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N>;
    constexpr int E = S::E, TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);

    const int lr = threadIdx.x / TPT;
    const int t = threadIdx.x - lr * TPT;
    const int64_t r = (int64_t)blockIdx.x * ROWS + lr;
    const bool active = r < total_rows;
    const int64_t b = active ? r / ny : 0;
    const int64_t y = active ? r - b * ny : 0;
    const int64_t off = b * stride + y * N;
    const bool cj = conj_io != 0;

    C v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? ld(in + off + t + TPT * e, cj) : C{0, 0};

    SmemView<C, S::LOGE, 1> sm{smem + lr * S::PADDED};
    if (TPT >= 32) fft_forward<N>(v, sm, t, tw, SyncCTA{});
    else fft_forward<N>(v, sm, t, tw, SyncWarp{});

    if (active) {
        C *dst = opaque_ptr(out + off + t);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[TPT * e] = cj ? cconj(v[e]) : v[e];
    }
}

// ---------------------------------------------------------------------------
// Column pass, general: op in {COL_FWD, COL_INV, COL_POISSON, COL_DIFFUSE}.
// CTA = W adjacent columns x all N rows; thread (c, t) = threadIdx.x = c + W t.
template <typename T, int N, int W>
__global__ void __launch_bounds__(W * Shape<N>::TPT)
col_fused_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out,
                 int64_t nx, int64_t stride, int op,
                 const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N>;
    using CS = ColSmem<C, N, W>;
    constexpr int E = S::E, TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);

    const int c = threadIdx.x % W;
    const int t = threadIdx.x / W;
    const int64_t a = (int64_t)blockIdx.x * W + c;
    const bool active = a < nx;
    const int64_t base = (int64_t)blockIdx.y * stride + (active ? a : 0) + (int64_t)t * nx;
    const int64_t estep = (int64_t)TPT * nx;          // element e of this thread: base + e*estep
    SmemView<C, S::LOGE, 1> sm{smem + c * CS::S};

    C v[E];
    if (op == COL_INV) {
        // standalone inverse along y: conj, scale by 1/(nx ny), forward, conj
#pragma unroll
        for (int e = 0; e < E; ++e)
            v[e] = active ? cscale(cconj(in[base + e * estep]), tab.scale) : C{0, 0};
        fft_forward<N>(v, sm, t, tw, SyncCTA{});
        if (active) {
            C *dst = opaque_ptr(out + base);
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e * estep] = cconj(v[e]);
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? in[base + e * estep] : C{0, 0};
    fft_forward<N>(v, sm, t, tw, SyncCTA{});
    if (op == COL_FWD) {
        if (active) {
            C *dst = opaque_ptr(out + base);
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e * estep] = v[e];
        }
        return;
    }
    // k-space operator at (a, b), b = t + TPT e; result conjugated for the inverse
    if (op == COL_POISSON) {
        const T kxa = active ? tab.kx2[a] : (T)1;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const T k2 = kxa + __ldg(&tab.ky2[t + TPT * e]);
            const T m = k2 == (T)0 ? (T)0 : -tab.scale / k2;          // -1/|k|^2, k = 0 zeroed
            v[e] = cconj(cscale(v[e], m));
        }
    } else {  // COL_DIFFUSE
        const T exa = active ? tab.ex[a] : (T)0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const T m = exa * __ldg(&tab.ey[t + TPT * e]);           // exp(-D|k|^2 dt)/(nx ny)
            v[e] = cconj(cscale(v[e], m));
        }
    }
    fft_forward<N>(v, sm, t, tw, SyncCTA{});
    if (active) {
        C *dst = opaque_ptr(out + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = cconj(v[e]);
    }
}

// Column pass for the wave step: both fields (U, V) of W columns, forward along
// y, the exact oscillator update, inverse along y.  In place.  One field is in
// registers at a time; the other's spectrum waits in a shared-memory stash
// (thread-private slots), so a thread holds 16 complex values, not 32.
template <typename C, int N, int W> struct WaveSmem {
    using CS = ColSmem<C, N, W>;
    static constexpr size_t XBYTES = CS::BYTES;                 // exchange buffers
    static constexpr size_t BYTES = XBYTES + (size_t)W * N * sizeof(C);   // + stash
};

template <typename T, int N, int W>
__global__ void __launch_bounds__(W * Shape<N>::TPT)
col_wave_kernel(typename cplx_t<T>::type *U, typename cplx_t<T>::type *V,
                int64_t nx, int64_t stride,
                const typename cplx_t<T>::type *__restrict__ tw, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<N>;
    using CS = ColSmem<C, N, W>;
    constexpr int E = S::E, TPT = S::TPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);
    C *stash = reinterpret_cast<C *>(smem_raw + WaveSmem<C, N, W>::XBYTES);

    const int c = threadIdx.x % W;
    const int t = threadIdx.x / W;
    const int64_t a = (int64_t)blockIdx.x * W + c;
    const bool active = a < nx;
    const int64_t base = (int64_t)blockIdx.y * stride + (active ? a : 0) + (int64_t)t * nx;
    const int64_t estep = (int64_t)TPT * nx;
    SmemView<C, S::LOGE, 1> sm{smem + c * CS::S};
    // stash slot of element e of this thread: column-interleaved, unit stride across threads
    auto slot = [&](int e) -> C & { return stash[(t + TPT * e) * W + c]; };

    C v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? U[base + e * estep] : C{0, 0};
    fft_forward<N>(v, sm, t, tw, SyncCTA{});
#pragma unroll
    for (int e = 0; e < E; ++e) slot(e) = v[e];                        // U^ -> stash
    asm volatile("" ::: "memory");
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = active ? V[base + e * estep] : C{0, 0};
    fft_forward<N>(v, sm, t, tw, SyncCTA{});
    asm volatile("" ::: "memory");   // keep the table loads below the transform (register pressure)
    // quadrant index: qa = |fold(a)|, qb = |fold(b)|
    const int64_t qa = active ? (a <= nx - a ? a : nx - a) : 0;
    const T *pC = tab.wC + qa * tab.qpitch;
    const T *pS1 = tab.wS1 + qa * tab.qpitch;
    const T *pS2 = tab.wS2 + qa * tab.qpitch;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int b = t + TPT * e;
        const int qb = b <= N - b ? b : N - b;
        const T cc = __ldg(pC + qb), s1 = __ldg(pS1 + qb), s2 = __ldg(pS2 + qb);
        const C uh = slot(e), vh = v[e];
        const C un = {cc * uh.x + s1 * vh.x, cc * uh.y + s1 * vh.y};   // C U + S1 V
        const C vn = {s2 * uh.x + cc * vh.x, s2 * uh.y + cc * vh.y};   // S2 U + C V
        slot(e) = cconj(un);
        v[e] = cconj(vn);
    }
    fft_forward<N>(v, sm, t, tw, SyncCTA{});                             // inverse of V
    if (active) {
        C *dst = opaque_ptr(V + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = cconj(v[e]);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = slot(e);
    fft_forward<N>(v, sm, t, tw, SyncCTA{});                             // inverse of U
    if (active) {
        C *dst = opaque_ptr(U + base);
#pragma unroll
        for (int e = 0; e < E; ++e) dst[e * estep] = cconj(v[e]);
    }
}

// ---------------------------------------------------------------------------
// Single-CTA solve of one small NX x NY grid per CTA (blockIdx.x = batch member),
// the whole grid resident in shared memory: rows -> columns -> operator ->
// inverse columns -> inverse rows, one HBM read and one HBM write.
template <typename C, int NX, int NY> struct SmallLayout {
    static constexpr int LPP = 128 / (int)sizeof(C);
    static constexpr int ROWLEN = Shape<NX>::PADDED;
    // row pitch: padded row, then offset so rows sharing a smem phase differ in bank
    static constexpr int PITCH = ((ROWLEN + LPP - 1) / LPP) * LPP + LPP / 2;
    static constexpr int THREADS_R = NY * Shape<NX>::TPT;
    static constexpr int THREADS_C = NX * Shape<NY>::TPT;
    static constexpr int THREADS = THREADS_R > THREADS_C ? THREADS_R : THREADS_C;
    static constexpr size_t BYTES = (size_t)NY * PITCH * sizeof(C);
};

template <typename T, int NX, int NY>
__global__ void __launch_bounds__(SmallLayout<typename cplx_t<T>::type, NX, NY>::THREADS)
small_solve_kernel(const typename cplx_t<T>::type *in, typename cplx_t<T>::type *out,
                   int64_t stride, int op,
                   const typename cplx_t<T>::type *__restrict__ twx,
                   const typename cplx_t<T>::type *__restrict__ twy, OpTables<T> tab)
{
    using C = typename cplx_t<T>::type;
    using L = SmallLayout<C, NX, NY>;
    using SX = Shape<NX>;
    using SY = Shape<NY>;
    static_assert(SX::E == SY::E, "small_solve needs one thread layout for rows and columns");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *g = reinterpret_cast<C *>(smem_raw);
    const int64_t off = (int64_t)blockIdx.x * stride;
    const int tid = threadIdx.x;

    const bool inv_only = op == COL_INV;
    // ---- phase 1: row transforms (forward, or conj-forward for the inverse)
    {
        const int row = tid / SX::TPT, t = tid % SX::TPT;
        const bool act = row < NY;
        C v[SX::E];
#pragma unroll
        for (int e = 0; e < SX::E; ++e)
            v[e] = act ? ld(in + off + (int64_t)row * NX + t + SX::TPT * e, inv_only) : C{0, 0};
        SmemView<C, SX::LOGE, 1> sm{g + (act ? row : 0) * L::PITCH};
        fft_forward<NX>(v, sm, t, twx, SyncCTA{});
        if (act) {
#pragma unroll
            for (int e = 0; e < SX::E; ++e) sm.at(t + SX::TPT * e) = inv_only ? cconj(v[e]) : v[e];
        }
        __syncthreads();
    }
    // ---- phase 2: column transforms (+ operator + inverse columns)
    {
        const int col = tid % NX, t = tid / NX;
        const bool act = t < SY::TPT;
        SmemView<C, 30, L::PITCH> sm{g + padidx(col, SX::LOGE)};
        C v[SY::E];
#pragma unroll
        for (int e = 0; e < SY::E; ++e) v[e] = act ? sm.at(t + SY::TPT * e) : C{0, 0};
        __syncthreads();
        if (inv_only) {
#pragma unroll
            for (int e = 0; e < SY::E; ++e) v[e] = cscale(cconj(v[e]), tab.scale);
        }
        fft_forward<NY>(v, sm, t, twy, SyncCTA{});
        if (op == COL_POISSON || op == COL_DIFFUSE) {
#pragma unroll
            for (int e = 0; e < SY::E; ++e) {
                const int b = t + SY::TPT * e;
                T m;
                if (op == COL_POISSON) {
                    const T k2 = tab.kx2[col] + tab.ky2[b];
                    m = k2 == (T)0 ? (T)0 : -tab.scale / k2;
                } else {
                    m = tab.ex[col] * tab.ey[b];
                }
                v[e] = cconj(cscale(v[e], m));
            }
            fft_forward<NY>(v, sm, t, twy, SyncCTA{});
#pragma unroll
            for (int e = 0; e < SY::E; ++e) v[e] = cconj(v[e]);
        } else if (inv_only) {
#pragma unroll
            for (int e = 0; e < SY::E; ++e) v[e] = cconj(v[e]);
        }
        if (act) {
#pragma unroll
            for (int e = 0; e < SY::E; ++e) sm.at(t + SY::TPT * e) = v[e];
        }
        __syncthreads();
    }
    if (op == COL_FWD || inv_only) {   // plain transform: write the grid
        for (int i = tid; i < NX * NY; i += L::THREADS) {
            const int row = i / NX, j = i % NX;
            out[off + i] = g[row * L::PITCH + padidx(j, SX::LOGE)];
        }
        return;
    }
    // ---- phase 3: inverse row transforms (conj, forward, conj)
    {
        const int row = tid / SX::TPT, t = tid % SX::TPT;
        const bool act = row < NY;
        SmemView<C, SX::LOGE, 1> sm{g + (act ? row : 0) * L::PITCH};
        C v[SX::E];
#pragma unroll
        for (int e = 0; e < SX::E; ++e) v[e] = act ? cconj(sm.at(t + SX::TPT * e)) : C{0, 0};
        __syncthreads();
        fft_forward<NX>(v, sm, t, twx, SyncCTA{});
        if (act) {
#pragma unroll
            for (int e = 0; e < SX::E; ++e) out[off + (int64_t)row * NX + t + SX::TPT * e] = cconj(v[e]);
        }
    }
}

} // namespace fftpde
