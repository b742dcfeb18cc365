// rc.cu -- real-to-complex / complex-to-real row passes.
//
// For a real row f_0 .. f_{n-1} (n = 2M) the spectrum is Hermitian,
// X_{n-a} = conj(X_a), so only X_0 .. X_M are kept (the "half spectrum").  The
// row is read as M complex values z_m = f_{2m} + i f_{2m+1} (the same bytes),
// transformed with the length-M Stockham FFT of fft_core.cuh (sign +, eq:DFT
// PAPER.md:119-124), and untangled with the even/odd split of eq:FFTpairodd
// (PAPER.md:199-224):  X_a = E_a + w_n^a O_a,  E = DFT_M(f_even), O = DFT_M(f_odd),
//   E_a = (Z_a + conj Z_{M-a}) / 2,   O_a = (Z_a - conj Z_{M-a}) / (2i),
// X_M = E_0 - O_0.  The inverse (unscaled, like every other inverse row pass)
// builds Z_a = (X_a + conj X_{M-a}) + i (X_a - conj X_{M-a}) w_n^{-a}, runs the
// conjugate length-M transform and stores Re/Im as f_{2m}, f_{2m+1}.
//   RC_FWD : real rows -> half-spectrum rows
//   RC_INV : half-spectrum rows -> real rows
//   RC_MID : half spectrum of step s -> real physical field (out2) -> half
//            spectrum of step s+1 (out); one read, two writes
//   RC_DIFF: real row -> half spectrum X_a -> X_a mul[a] -> real row (unscaled
//            inverse): the x factor of a separable operator, one read, one write
// Half-spectrum rows have `pitch` elements (>= M + 1; entries M+1.. are zeroed).
#include <cuda_runtime.h>
#include <stdint.h>
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

template <int TPT> struct RcSync {
    int id;
    __device__ __forceinline__ void operator()() const
    {
        if constexpr (TPT <= 32) __syncwarp();
        else asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(TPT) : "memory");
    }
};

template <typename T, int M, int W, int OP>
__global__ void __launch_bounds__(W * Shape<M>::TPT)
rc_rows_kernel(const void *in, void *out, void *out2, int64_t nrows, int64_t pitch,
               const typename cplx_t<T>::type *__restrict__ tw, const typename cplx_t<T>::type *__restrict__ twr,
               const T *__restrict__ mul)
{
    using C = typename cplx_t<T>::type;
    using S = Shape<M>;
    constexpr int E = S::E, TPT = S::TPT;
    constexpr int SP = S::PADDED;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);
    const int c = threadIdx.x / TPT, t = threadIdx.x % TPT;
    const int64_t row = (int64_t)blockIdx.x * W + c;
    const bool active = row < nrows;
    const int64_t r = active ? row : 0;
    const RcSync<TPT> sync{1 + c};
    SmemView<C, S::LOGE, 1> sm{smem + c * SP};
    const TwL1<M, C> twp{tw, t};

    C v[E];
    if constexpr (OP == RC_FWD || OP == RC_DIFF) {
        const C *z = reinterpret_cast<const C *>(in) + r * M;     // the real row as M complex pairs
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = z[t + TPT * e];
    } else {
        // Z_a = (X_a + conj X_{M-a}) + i (X_a - conj X_{M-a}) w_n^{-a}
        const C *x = reinterpret_cast<const C *>(in) + r * pitch;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int a = t + TPT * e;
            const C xa = x[a], xm = x[M - a];
            const C ev = {xa.x + xm.x, xa.y - xm.y};
            const C od = cmulw<true>(C{xa.x - xm.x, xa.y + xm.y}, twr[a]);
            v[e] = C{ev.x - od.y, ev.y + od.x};
        }
        fft_tw<M, true>(v, sm, t, twp, sync);                      // sum_a Z_a w_M^{-am} = n (f_2m + i f_2m+1)
        C *f = reinterpret_cast<C *>(OP == RC_INV ? out : out2) + r * M;
        if (active) {
#pragma unroll
            for (int e = 0; e < E; ++e) f[t + TPT * e] = v[e];
        }
        if constexpr (OP == RC_INV) return;
    }
    // forward: Z = DFT_M(z), then the even/odd untangle through shared memory
    fft_tw<M, false>(v, sm, t, twp, sync);
#pragma unroll
    for (int e = 0; e < E; ++e) sm.at(t + TPT * e) = v[e];
    sync();
    if constexpr (OP == RC_DIFF) {
        // X_a mul[a] (a < M) stays in registers, X_M mul[M] with the thread of a = 0
        C X[E];
        C XM = C{0, 0};
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int a = t + TPT * e;
            const C za = v[e], zm = sm.at(a == 0 ? 0 : M - a);
            const C ev = {(T)0.5 * (za.x + zm.x), (T)0.5 * (za.y - zm.y)};
            const C od = {(T)0.5 * (za.y + zm.y), (T)-0.5 * (za.x - zm.x)};
            const C wo = cmulw<false>(od, twr[a]);
            X[e] = cscale(C{ev.x + wo.x, ev.y + wo.y}, __ldg(mul + a));
            if (a == 0) XM = cscale(C{ev.x - od.x, ev.y - od.y}, __ldg(mul + M));
        }
        sync();                                                                   // Z is consumed
#pragma unroll
        for (int e = 0; e < E; ++e) sm.at(t + TPT * e) = X[e];
        sync();
        // inverse as RC_INV: Z_a = (X_a + conj X_{M-a}) + i (X_a - conj X_{M-a}) w_n^{-a}
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int a = t + TPT * e;
            const C xa = X[e], xm = a == 0 ? XM : sm.at(M - a);
            const C ev = {xa.x + xm.x, xa.y - xm.y};
            const C od = cmulw<true>(C{xa.x - xm.x, xa.y + xm.y}, twr[a]);
            v[e] = C{ev.x - od.y, ev.y + od.x};
        }
        sync();                                                                   // X is consumed
        fft_tw<M, true>(v, sm, t, twp, sync);
        C *f = reinterpret_cast<C *>(out) + r * M;
        if (active) {
#pragma unroll
            for (int e = 0; e < E; ++e) f[t + TPT * e] = v[e];
        }
        return;
    }
    C *x = reinterpret_cast<C *>(out) + r * pitch;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int a = t + TPT * e;
        const C za = v[e], zm = sm.at(a == 0 ? 0 : M - a);
        const C ev = {(T)0.5 * (za.x + zm.x), (T)0.5 * (za.y - zm.y)};          // (Z_a + conj Z_{M-a}) / 2
        const C od = {(T)0.5 * (za.y + zm.y), (T)-0.5 * (za.x - zm.x)};         // (Z_a - conj Z_{M-a}) / (2i)
        const C wo = cmulw<false>(od, twr[a]);
        if (active) x[a] = C{ev.x + wo.x, ev.y + wo.y};
        if (a == 0 && active) {
            x[M] = C{ev.x - od.x, ev.y - od.y};                                  // X_M = E_0 - O_0
            for (int64_t q = M + 1; q < pitch; ++q) x[q] = C{0, 0};
        }
    }
}

template <typename T, int M>
cudaError_t rc_rows_n(const void *in, void *out, void *out2, int64_t nrows, int64_t pitch, int op, const void *tw,
                      const void *twr, cudaStream_t st, const void *mul)
{
    using C = typename cplx_t<T>::type;
    constexpr int TPT = Shape<M>::TPT;
    constexpr int W = TPT >= 256 ? 1 : 256 / TPT;
    const size_t smem = (size_t)W * Shape<M>::PADDED * sizeof(C);
    const unsigned grid = (unsigned)((nrows + W - 1) / W);
    auto go = [&](auto k) -> cudaError_t {
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        k<<<grid, W * TPT, smem, st>>>(in, out, out2, nrows, pitch, (const C *)tw, (const C *)twr, (const T *)mul);
        return cudaGetLastError();
    };
    switch (op) {
    case RC_FWD: return go(rc_rows_kernel<T, M, W, RC_FWD>);
    case RC_INV: return go(rc_rows_kernel<T, M, W, RC_INV>);
    case RC_MID: return go(rc_rows_kernel<T, M, W, RC_MID>);
    case RC_DIFF: return mul ? go(rc_rows_kernel<T, M, W, RC_DIFF>) : cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
    }
}

template <typename T>
cudaError_t launch_rc_rows(int64_t nx, const void *in, void *out, void *out2, int64_t nrows, int64_t pitch, int op,
                           const void *tw, const void *twr, cudaStream_t st, const void *mul)
{
    switch (nx / 2) {
#define X(L) case L: return rc_rows_n<T, L>(in, out, out2, nrows, pitch, op, tw, twr, st, mul);
        X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_rc_rows<double>(int64_t, const void *, void *, void *, int64_t, int64_t, int,
                                            const void *, const void *, cudaStream_t, const void *);
template cudaError_t launch_rc_rows<float>(int64_t, const void *, void *, void *, int64_t, int64_t, int,
                                           const void *, const void *, cudaStream_t, const void *);

} // namespace fftpde
