// Traffic ceiling of the four-step tile patterns (r02): the AA pass with its
// arithmetic removed (TMA box load + store of every 64 KiB tile; MID: two stores),
// the same with the arithmetic, and a contiguous copy, on a 32768^2 complex128 field.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2412_12308_b200/csrc \
//        -Iinclude -o tools/exp_aa_copy tools/exp_aa_copy.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include "fourstep.cuh"
#include "dispatch.cuh"
using namespace fftpde;
static bool map4(CUtensorMap &m, void *p)
{
    using G = FsGeom;
    cuuint64_t dims[4] = {(cuuint64_t)(2 * G::P), (cuuint64_t)G::Q, (cuuint64_t)G::P, (cuuint64_t)G::Q};
    cuuint64_t strides[3] = {(cuuint64_t)G::P * 16, (cuuint64_t)G::N * 16, (cuuint64_t)G::P * G::N * 16};
    cuuint32_t box[4] = {(cuuint32_t)(2 * G::W), (cuuint32_t)G::Q, 1, (cuuint32_t)G::Q};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, p, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <int OP> float run(const CUtensorMap &a, const CUtensorMap &b, const CUtensorMap &c, const double2 *tw)
{
    using Cfg = FsCfg<1>;
    auto k = aa_kernel<OP, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::BYTES);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int r = 0; r < 2; ++r) k<<<FsGeom::NTILES, FsGeom::NT, Cfg::BYTES>>>(a, b, c, tw);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<FsGeom::NTILES, FsGeom::NT, Cfg::BYTES>>>(a, b, c, tw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}
__global__ void copyk(const int4 *__restrict__ a, int4 *b, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main()
{
    const size_t n = (size_t)FsGeom::N * FsGeom::N;
    double2 *A, *B, *C, *tw;
    cudaMalloc(&A, n * 16);
    cudaMalloc(&B, n * 16);
    cudaMalloc(&C, n * 16);
    cudaMalloc(&tw, 32768 * 16);
    cudaMemset(A, 0, n * 16);
    cudaMemset(tw, 0, 32768 * 16);
    CUtensorMap ma, mb, mc;
    map4(ma, A);
    map4(mb, B);
    map4(mc, C);
    const double GB = n * 16 / 1e9;
    float t;
    t = run<FS_COPY>(ma, mb, mc, tw);   printf("AA tile copy (load+store)      %7.3f ms  %6.0f GB/s\n", t, 2 * GB / t * 1e3);
    t = run<FS_FWD>(ma, mb, mc, tw);    printf("AA forward (with arithmetic)   %7.3f ms  %6.0f GB/s\n", t, 2 * GB / t * 1e3);
    t = run<FS_COPY3>(ma, mb, mc, tw);  printf("MID tile copy (load+2 stores)  %7.3f ms  %6.0f GB/s\n", t, 3 * GB / t * 1e3);
    t = run<FS_MID>(ma, mb, mc, tw);    printf("MID (with arithmetic)          %7.3f ms  %6.0f GB/s\n", t, 3 * GB / t * 1e3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    copyk<<<148 * 8, 512>>>((const int4 *)A, (int4 *)B, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copyk<<<148 * 8, 512>>>((const int4 *)A, (int4 *)B, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1);
    t /= 5;
    printf("contiguous copy                %7.3f ms  %6.0f GB/s\n", t, 2 * GB / t * 1e3);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
