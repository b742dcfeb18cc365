// L2 bandwidth probe: copy of an L2-resident buffer (contiguous and 128 B-segment
// column tiles), and DSMEM throughput, on B200.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void copy_contig(const int4 *__restrict__ in, int4 *__restrict__ out, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}
__global__ void read_contig(const int4 *__restrict__ in, int4 *__restrict__ out, size_t n)
{
    int4 acc = {0, 0, 0, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        int4 v = __ldcg(in + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if (acc.x == 0x12345678) out[0] = acc;
}
// column tiles: rows of row_bytes, 128 B segments; tile = 128 B x R rows
__global__ void copy_cols(const int4 *__restrict__ in, int4 *__restrict__ out, long rows, long row_v, long seg_v)
{
    const long ncolblk = row_v / seg_v;
    for (long blk = blockIdx.x; blk < ncolblk; blk += gridDim.x)
        for (long i = threadIdx.x; i < rows * seg_v; i += blockDim.x) {
            long r = i / seg_v, v = i % seg_v;
            long idx = r * row_v + blk * seg_v + v;
            out[idx] = in[idx];
        }
}
// DSMEM: each CTA of a cluster reads its neighbour's smem buffer repeatedly
__global__ void __cluster_dims__(2, 1, 1) dsmem_read(int4 *out, int iters)
{
    extern __shared__ int4 buf[];
    cg::cluster_group cl = cg::this_cluster();
    const int nv = 64 * 1024 / 16;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) buf[i] = make_int4(i, i, i, i);
    cl.sync();
    int4 *rem = cl.map_shared_rank(buf, cl.block_rank() ^ 1);
    int4 acc = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it)
        for (int i = threadIdx.x; i < nv; i += blockDim.x) {
            int4 v = rem[(i + it) & (nv - 1)];
            acc.x ^= v.x; acc.y += v.y;
        }
    cl.sync();
    if (acc.x == 0x7777777) out[0] = acc;
}

template <typename F> float timeit(F f, int reps = 20)
{
    for (int i = 0; i < 3; ++i) f();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main()
{
    int4 *A, *B;
    cudaMalloc(&A, 1ull << 30); cudaMalloc(&B, 1ull << 30);
    cudaMemset(A, 1, 1ull << 30); cudaMemset(B, 1, 1ull << 30);
    for (size_t mb : {8, 16, 32, 48, 64, 128, 512}) {
        size_t n = (mb << 20) / 16;
        float t = timeit([&] { copy_contig<<<148 * 8, 256>>>(A, B, n); });
        float r = timeit([&] { read_contig<<<148 * 8, 256>>>(A, B, n); });
        printf("contig %4zu MiB: copy %8.2f us %7.0f GB/s (r+w) | read %8.2f us %7.0f GB/s\n", mb, t * 1e3,
               2.0 * (mb << 20) / (t * 1e-3) / 1e9, r * 1e3, 1.0 * (mb << 20) / (r * 1e-3) / 1e9);
    }
    // 128 B column tiles on a 1024-row x 16 KiB grid (16 MiB, L2) and 4096 x 64 KiB (256 MiB, HBM)
    {
        float t = timeit([&] { copy_cols<<<148 * 4, 256>>>(A, B, 1024, 1024, 8); });
        printf("cols128 16 MiB (1024 rows x 16 KiB): %8.2f us %7.0f GB/s\n", t * 1e3, 2.0 * (16 << 20) / (t * 1e-3) / 1e9);
        t = timeit([&] { copy_cols<<<148 * 4, 256>>>(A, B, 4096, 4096, 8); });
        printf("cols128 256 MiB (4096 rows x 64 KiB): %8.2f us %7.0f GB/s\n", t * 1e3, 2.0 * (256 << 20) / (t * 1e-3) / 1e9);
    }
    {
        cudaFuncSetAttribute(dsmem_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        const int iters = 64;
        float t = timeit([&] { dsmem_read<<<148, 1024, 64 * 1024>>>(B, iters); }, 5);
        const double bytes = 148.0 * iters * 64 * 1024;
        printf("dsmem read (148 CTAs x %d x 64 KiB): %8.2f us %7.0f GB/s total, %.1f B/clk/SM @1.965GHz %s\n", iters,
               t * 1e3, bytes / (t * 1e-3) / 1e9, bytes / (t * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
