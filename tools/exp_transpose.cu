// Transposed-layout probe on a 4096 x 4096 complex128 field: row-contiguous reads
// with 16 B scattered writes to T[a][k] (and the reverse gather), vs a plain copy.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_rows(const double2 *__restrict__ in, double2 *__restrict__ out, int n)
{
    for (int k = blockIdx.x; k < n; k += gridDim.x)
        for (int a = threadIdx.x; a < n; a += blockDim.x) out[(size_t)k * n + a] = in[(size_t)k * n + a];
}
// row k read contiguously, written to column k of T (16 B scatter)
__global__ void scatter_rows(const double2 *__restrict__ in, double2 *__restrict__ out, int n)
{
    for (int k = blockIdx.x; k < n; k += gridDim.x)
        for (int a = threadIdx.x; a < n; a += blockDim.x) out[(size_t)a * n + k] = in[(size_t)k * n + a];
}
// row k of the result gathered from column k of T (16 B gather), written contiguously
__global__ void gather_rows(const double2 *__restrict__ in, double2 *__restrict__ out, int n)
{
    for (int k = blockIdx.x; k < n; k += gridDim.x)
        for (int a = threadIdx.x; a < n; a += blockDim.x) out[(size_t)k * n + a] = in[(size_t)a * n + k];
}
// 2 rows per CTA: 32 B segments
__global__ void scatter_rows2(const double2 *__restrict__ in, double2 *__restrict__ out, int n)
{
    for (int k = 2 * blockIdx.x; k < n; k += 2 * gridDim.x)
        for (int i = threadIdx.x; i < 2 * n; i += blockDim.x) {
            const int a = i >> 1, r = i & 1;
            out[(size_t)a * n + k + r] = in[(size_t)(k + r) * n + a];
        }
}

template <typename F> float timeit(F f)
{
    for (int i = 0; i < 2; ++i) f();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
}

int main()
{
    const int n = 4096;
    const size_t bytes = (size_t)n * n * 16;
    double2 *A, *B;
    cudaMalloc(&A, bytes); cudaMalloc(&B, bytes);
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes);
    for (int grid : {148, 296, 592, 1184}) {
        for (int thr : {256, 512}) {
            float t0 = timeit([&] { copy_rows<<<grid, thr>>>(A, B, n); });
            float t1 = timeit([&] { scatter_rows<<<grid, thr>>>(A, B, n); });
            float t2 = timeit([&] { gather_rows<<<grid, thr>>>(A, B, n); });
            float t3 = timeit([&] { scatter_rows2<<<grid, thr>>>(A, B, n); });
            printf("grid %4d thr %3d: copy %7.1f us %5.0f GB/s | scatter16 %7.1f us %5.0f GB/s | gather16 %7.1f us %5.0f GB/s | scatter32 %7.1f us %5.0f GB/s\n",
                   grid, thr, t0 * 1e3, 2 * bytes / (t0 * 1e-3) / 1e9, t1 * 1e3, 2 * bytes / (t1 * 1e-3) / 1e9,
                   t2 * 1e3, 2 * bytes / (t2 * 1e-3) / 1e9, t3 * 1e3, 2 * bytes / (t3 * 1e-3) / 1e9);
        }
    }
    return 0;
}
