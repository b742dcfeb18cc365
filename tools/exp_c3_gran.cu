// Copy ceiling of column-granule TMA patterns on a 4096^2 complex128 field (64 MiB
// rows of 64 KiB): a CTA moves a 64 KiB tile of G adjacent complex128 columns
// (G * 16 bytes wide) x 4096/G rows by TMA boxes of 256 rows, in and out, several
// CTAs per SM.  G = 1 is the C3 wave column pass's pattern; G = 2 / 4 the 32- and
// 64-byte granules of a column-pair / column-quad layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2412_12308_b200/csrc -Iinclude \
//        -o tools/exp_c3_gran tools/exp_c3_gran.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include "tmacols.cuh"
using namespace fftpde;
constexpr int NN = 4096;
__global__ void __launch_bounds__(128) gran_copy(const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mo, int G)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *S = smem_raw + ((128u - (tma_smem(smem_raw) & 127u)) & 127u);
    const uint32_t mbar = tma_smem(S + 65536);
    if (threadIdx.x == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int rows = NN / G, nb = rows / 256;
    const int ngx = NN / G;                           // column groups
    const int gx = blockIdx.x % ngx, part = blockIdx.x / ngx;   // part: which 4096/G-row slice
    const int x = 2 * G * gx, y0 = part * rows;
    if (threadIdx.x == 0) {
        tma_mbar_expect(mbar, 65536);
        for (int k = 0; k < nb; ++k) tma_load3(tma_smem(S) + k * 256 * G * 16, &mi, x, y0 + k * 256, 0, mbar);
    }
    tma_mbar_wait(mbar, 0);
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_fence_smem();
        for (int k = 0; k < nb; ++k) tma_store3(&mo, x, y0 + k * 256, 0, tma_smem(S) + k * 256 * G * 16);
        tma_commit();
        tma_wait_read0();
    }
}
// CTA q: column c = q % 2 of pair p = q / 2 (adjacent CTAs share the pair's sectors)
__global__ void __launch_bounds__(128) pair_copy(const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mo)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *S = smem_raw + ((128u - (tma_smem(smem_raw) & 127u)) & 127u);
    const uint32_t mbar = tma_smem(S + 65536);
    if (threadIdx.x == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int c = blockIdx.x % 2, pr = blockIdx.x / 2;
    if (threadIdx.x == 0) {
        tma_mbar_expect(mbar, 65536);
        for (int k = 0; k < NN / 256; ++k) tma_load3(tma_smem(S) + k * 256 * 16, &mi, 2 * c, k * 256, pr, mbar);
    }
    tma_mbar_wait(mbar, 0);
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_fence_smem();
        for (int k = 0; k < NN / 256; ++k) tma_store3(&mo, 2 * c, k * 256, pr, tma_smem(S) + k * 256 * 16);
        tma_commit();
        tma_wait_read0();
    }
}
static void map(CUtensorMap &m, void *p, int G)
{
    cuuint64_t dims[3] = {2 * NN, NN, 1};
    cuuint64_t strides[2] = {(cuuint64_t)NN * 16, (cuuint64_t)NN * NN * 16};
    cuuint32_t box[3] = {(cuuint32_t)(2 * G), 256, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}
int main()
{
    const size_t n = (size_t)NN * NN;
    const int F = 8;                                   // 8 fields (2 GiB) so that L2 does not hold them
    double2 *A, *B;
    cudaMalloc(&A, n * 16 * F);
    cudaMalloc(&B, n * 16 * F);
    cudaMemset(A, 0, n * 16 * F);
    cudaFuncSetAttribute(gran_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 256);
    cudaFuncSetAttribute(pair_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 256);
    for (int G : {1, 2, 4, 8}) {
        CUtensorMap mi[F], mo[F];
        for (int f = 0; f < F; ++f) { map(mi[f], A + f * n, G); map(mo[f], B + f * n, G); }
        const int tiles = (NN / G) * G;                // 4096 tiles of 64 KiB per field
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int f = 0; f < F; ++f) gran_copy<<<tiles, 128, 65536 + 256>>>(mi[f], mo[f], G);
        cudaEventRecord(e0);
        for (int r = 0; r < 4; ++r)
            for (int f = 0; f < F; ++f) gran_copy<<<tiles, 128, 65536 + 256>>>(mi[f], mo[f], G);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("granule %3d B (G=%d columns x %4d rows per tile): %.1f us per field  %6.0f GB/s  %s\n", 16 * G, G,
               NN / G, ms * 1e3 / 32, 2.0 * n * 16 * 32 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    // 16-byte boxes over a column-PAIR layout [p][y][2] (32-byte granules, the pair's
    // two columns read by two CTAs): a 64 KiB tile = one column c of pair p, 4096 rows
    // of 16 bytes at a 32-byte stride
    {
        CUtensorMap mi[F], mo[F];
        for (int f = 0; f < F; ++f) {
            for (int io = 0; io < 2; ++io) {
                cuuint64_t dims[3] = {4, NN, NN / 2};                 // {c re/im, y, p}
                cuuint64_t strides[2] = {32, (cuuint64_t)NN * 32};
                cuuint32_t box[3] = {2, 256, 1};
                cuuint32_t es[3] = {1, 1, 1};
                cuTensorMapEncodeTiled(io ? &mo[f] : &mi[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (io ? B : A) + f * n,
                                       dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
        }
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int f = 0; f < F; ++f) pair_copy<<<NN, 128, 65536 + 256>>>(mi[f], mo[f]);
        cudaEventRecord(e0);
        for (int r = 0; r < 4; ++r)
            for (int f = 0; f < F; ++f) pair_copy<<<NN, 128, 65536 + 256>>>(mi[f], mo[f]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("16 B boxes at a 32 B stride (column-pair layout, CTA = one column of a pair): %.1f us per field  %6.0f GB/s  %s\n",
               ms * 1e3 / 32, 2.0 * n * 16 * 32 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
