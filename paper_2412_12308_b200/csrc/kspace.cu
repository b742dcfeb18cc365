// kspace.cu -- diagonal k-space operators between a forward and an inverse 2D
// transform, in place on a natural-order spectrum:
//   KOP_LAPLACIAN  X <- -(kx^2 + ky^2) X
//   KOP_DX         X <- -i kx X          (F{du/dx} = -i w F{u})
//   KOP_DY         X <- -i ky X
//   KOP_DIFFSRC    X <- E X + Phi S,  E = exp(-D k^2 dt),
//                  Phi = -expm1(-D k^2 dt)/(D k^2) (k != 0, D > 0), dt otherwise:
//                  one exact step of du^/dt = -D k^2 u^ + s^ (eq:DiffusionIVPFS,
//                  PAPER.md:369-376, with the constant forcing of a static source)
// kx, ky: signed angular wavenumbers 2 pi fold(a)/L, Nyquist at +N/2
// (R2, R4, R24); kx2, ky2 their squares as used by every other pass.
#include <cuda_runtime.h>
#include <stdint.h>
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

template <typename T>
__global__ void kop_kernel(typename cplx_t<T>::type *X, const typename cplx_t<T>::type *__restrict__ S,
                           int64_t nx, int64_t ny, int64_t batch, int64_t stride, int op,
                           const T *__restrict__ kx, const T *__restrict__ ky, const T *__restrict__ kx2,
                           const T *__restrict__ ky2, double D, double dt)
{
    using C = typename cplx_t<T>::type;
    const int64_t plane = nx * ny, n = plane * batch;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bi = i / plane, r = i - bi * plane;
        const int64_t b = r / nx, a = r - b * nx;
        const int64_t off = bi * stride + r;
        const C v = X[off];
        C o;
        if (op == KOP_LAPLACIAN) {
            const T m = -(kx2[a] + ky2[b]);
            o = C{m * v.x, m * v.y};
        } else if (op == KOP_DX || op == KOP_DY) {
            const T k = op == KOP_DX ? kx[a] : ky[b];
            o = C{k * v.y, -k * v.x};                          // (-i k)(x + i y)
        } else {                                               // KOP_DIFFSRC
            const double k2 = (double)kx2[a] + (double)ky2[b];
            const double x = D * k2 * dt;
            const double E = exp(-x);
            const double Phi = x > 0.0 ? -expm1(-x) / (D * k2) : dt;
            const C s = S[off];
            o = C{(T)(E * (double)v.x + Phi * (double)s.x), (T)(E * (double)v.y + Phi * (double)s.y)};
        }
        X[off] = o;
    }
}

template <typename T>
cudaError_t launch_kop(void *X, const void *S, int64_t nx, int64_t ny, int64_t batch, int64_t stride, int op,
                       const void *kx, const void *ky, const void *kx2, const void *ky2, double D, double dt,
                       cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    const int64_t n = nx * ny * batch;
    int64_t g = (n + 255) / 256;
    if (g > 148LL * 16) g = 148LL * 16;
    kop_kernel<T><<<(unsigned)(g < 1 ? 1 : g), 256, 0, st>>>((C *)X, (const C *)S, nx, ny, batch, stride, op,
                                                             (const T *)kx, (const T *)ky, (const T *)kx2,
                                                             (const T *)ky2, D, dt);
    return cudaGetLastError();
}

template cudaError_t launch_kop<double>(void *, const void *, int64_t, int64_t, int64_t, int64_t, int, const void *,
                                        const void *, const void *, const void *, double, double, cudaStream_t);
template cudaError_t launch_kop<float>(void *, const void *, int64_t, int64_t, int64_t, int64_t, int, const void *,
                                       const void *, const void *, const void *, double, double, cudaStream_t);

} // namespace fftpde
