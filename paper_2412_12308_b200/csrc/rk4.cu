// rk4.cu -- time-dependent source path: the wave
// equation u_tt = c^2 nabla^2 u + s(t, x, y) integrated in Fourier space,
//   du^/dt = v^,  dv^/dt = -kappa^2 u^ + s^(t),  kappa = c|k|
// (eq:SystemOfODEsForWaveEquation), with the classical RK4
// scheme and the paper's orbiting Gaussian source re-sampled
// and transformed at each stage time (R18-R22).
//
// Kernels:
//   src_kernel : s(t, x_j, y_k) = A cos(gamma t) exp(-(dx^2 + dy^2)/sigma^2),
//                dx, dy periodic minimum images of x_j - x0, y_k - y0 (the
//                host passes x0 = rs cos(Omega t), y0 = rs sin(Omega t),
//                amp = A cos(gamma t) in fp64)
//   rk4_kernel : one RK4 step of every Fourier mode given s^ at t, t + dt/2,
//                t + dt -- the four stage evaluations and their combination
//                (k1 + 2 k2 + 2 k3 + k4)/6 fused in registers: one read of the
//                state and the three source spectra, one write of the state
//   mean_kernel: u_bar = u^(0,0) / (nx ny) into the means record
#include <cuda_runtime.h>
#include <stdint.h>
#include "fft_core.cuh"
#include "launch.h"

namespace fftpde {

template <typename T>
__global__ void src_kernel(typename cplx_t<T>::type *s, int64_t nx, int64_t ny, SrcParams p)
{
    using C = typename cplx_t<T>::type;
    const int64_t n = nx * ny;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / nx, j = i - k * nx;
        const double x = p.xmin + (double)j * p.Lx / (double)nx;
        const double y = p.ymin + (double)k * p.Ly / (double)ny;
        double dx = x - p.x0, dy = y - p.y0;
        dx = dx - p.Lx * floor(dx / p.Lx + 0.5);
        dy = dy - p.Ly * floor(dy / p.Ly + 0.5);
        const double v = p.amp * exp(-(dx * dx + dy * dy) / (p.sigma * p.sigma));
        s[i] = C{(T)v, (T)0};
    }
}

template <typename T>
__global__ void rk4_kernel(typename cplx_t<T>::type *U, typename cplx_t<T>::type *V,
                           const typename cplx_t<T>::type *__restrict__ S0,
                           const typename cplx_t<T>::type *__restrict__ Sh,
                           const typename cplx_t<T>::type *__restrict__ S1, int64_t nx, int64_t ny,
                           const T *__restrict__ kx2, const T *__restrict__ ky2, T c2, T dt,
                           typename cplx_t<T>::type *mean_out, T inv_area)
{
    using C = typename cplx_t<T>::type;
    const int64_t n = nx * ny;
    const T h2 = (T)0.5 * dt, h6 = dt / (T)6;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / nx, a = i - b * nx;
        const T w2 = c2 * (kx2[a] + ky2[b]);                 // kappa^2
        const C u = U[i], v = V[i], s0 = S0[i], sh = Sh[i], s1 = S1[i];
        // k1 = f(t, y)
        const C k1u = v;
        const C k1v = C{s0.x - w2 * u.x, s0.y - w2 * u.y};
        // k2 = f(t + dt/2, y + dt/2 k1)
        const C u2 = C{u.x + h2 * k1u.x, u.y + h2 * k1u.y};
        const C k2u = C{v.x + h2 * k1v.x, v.y + h2 * k1v.y};
        const C k2v = C{sh.x - w2 * u2.x, sh.y - w2 * u2.y};
        // k3 = f(t + dt/2, y + dt/2 k2)
        const C u3 = C{u.x + h2 * k2u.x, u.y + h2 * k2u.y};
        const C k3u = C{v.x + h2 * k2v.x, v.y + h2 * k2v.y};
        const C k3v = C{sh.x - w2 * u3.x, sh.y - w2 * u3.y};
        // k4 = f(t + dt, y + dt k3)
        const C u4 = C{u.x + dt * k3u.x, u.y + dt * k3u.y};
        const C k4u = C{v.x + dt * k3v.x, v.y + dt * k3v.y};
        const C k4v = C{s1.x - w2 * u4.x, s1.y - w2 * u4.y};
        // y(t + dt) = y + dt/6 (k1 + 2 k2 + 2 k3 + k4)
        const C nu = C{u.x + h6 * (k1u.x + (T)2 * k2u.x + (T)2 * k3u.x + k4u.x),
                       u.y + h6 * (k1u.y + (T)2 * k2u.y + (T)2 * k3u.y + k4u.y)};
        const C nv = C{v.x + h6 * (k1v.x + (T)2 * k2v.x + (T)2 * k3v.x + k4v.x),
                       v.y + h6 * (k1v.y + (T)2 * k2v.y + (T)2 * k3v.y + k4v.y)};
        U[i] = nu;
        V[i] = nv;
        if (i == 0 && mean_out) *mean_out = C{nu.x * inv_area, nu.y * inv_area};
    }
}

template <typename T>
__global__ void mean_kernel(const typename cplx_t<T>::type *U, typename cplx_t<T>::type *out, T inv_area)
{
    using C = typename cplx_t<T>::type;
    const C u = U[0];
    *out = C{u.x * inv_area, u.y * inv_area};
}

static unsigned grid_for(int64_t n, int threads)
{
    int64_t g = (n + threads - 1) / threads;
    const int64_t cap = 148LL * 16;
    return (unsigned)(g < 1 ? 1 : g > cap ? cap : g);
}

template <typename T>
cudaError_t launch_source(void *s, int64_t nx, int64_t ny, const SrcParams &p, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    src_kernel<T><<<grid_for(nx * ny, 256), 256, 0, st>>>((C *)s, nx, ny, p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rk4(void *U, void *V, const void *S0, const void *Sh, const void *S1, int64_t nx, int64_t ny,
                       const void *kx2, const void *ky2, double c, double dt, void *mean_out, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    const T inv_area = (T)(1.0 / ((double)nx * (double)ny));
    rk4_kernel<T><<<grid_for(nx * ny, 256), 256, 0, st>>>((C *)U, (C *)V, (const C *)S0, (const C *)Sh,
                                                          (const C *)S1, nx, ny, (const T *)kx2, (const T *)ky2,
                                                          (T)(c * c), (T)dt, (C *)mean_out, inv_area);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_mean(const void *U, void *out, int64_t nx, int64_t ny, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    mean_kernel<T><<<1, 1, 0, st>>>((const C *)U, (C *)out, (T)(1.0 / ((double)nx * (double)ny)));
    return cudaGetLastError();
}

template cudaError_t launch_source<double>(void *, int64_t, int64_t, const SrcParams &, cudaStream_t);
template cudaError_t launch_source<float>(void *, int64_t, int64_t, const SrcParams &, cudaStream_t);
template cudaError_t launch_rk4<double>(void *, void *, const void *, const void *, const void *, int64_t, int64_t,
                                        const void *, const void *, double, double, void *, cudaStream_t);
template cudaError_t launch_rk4<float>(void *, void *, const void *, const void *, const void *, int64_t, int64_t,
                                       const void *, const void *, double, double, void *, cudaStream_t);
template cudaError_t launch_mean<double>(const void *, void *, int64_t, int64_t, cudaStream_t);
template cudaError_t launch_mean<float>(const void *, void *, int64_t, int64_t, cudaStream_t);

} // namespace fftpde
