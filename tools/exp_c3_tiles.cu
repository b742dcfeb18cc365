// Traffic ceiling of 16-byte-wide four-step tiles on the C3 grid (4096^2 complex128):
// box {1 complex, 64 n2, 1 m1, 64 m2} (64 KiB) loaded and stored by TMA, one tile per
// CTA, several CTAs per SM; compared with a contiguous copy and with 64-row x 64-column
// blocks (1 KiB row segments, the B-pass pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2412_12308_b200/csrc -Iinclude \
//        -o tools/exp_c3_tiles tools/exp_c3_tiles.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include "fourstep.cuh"
using namespace fftpde;
constexpr int NN = 4096, PP = 64, QQ = 64;
__global__ void __launch_bounds__(128) tile_copy(const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mo, int w, int kind)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t pad = (128u - (tma_smem(smem_raw) & 127u)) & 127u;
    unsigned char *S = smem_raw + pad;
    const uint32_t mbar = tma_smem(S + 65536);
    if (threadIdx.x == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int c0, c1, c2, c3;
    if (kind == 0) {            // AA tile: (m1, n1 chunk of w) x all (m2, n2)
        const int nch = PP / w;
        c0 = 2 * w * (blockIdx.x % nch); c1 = 0; c2 = blockIdx.x / nch; c3 = 0;
    } else {                    // B block: 64 rows (m1) x 64 columns (n1) of block (m2, n2)
        c0 = 0; c1 = blockIdx.x % QQ; c2 = 0; c3 = blockIdx.x / QQ;
    }
    if (threadIdx.x == 0) {
        tma_mbar_expect(mbar, 65536);
        tma_load4(tma_smem(S), &mi, c0, c1, c2, c3, mbar);
    }
    tma_mbar_wait(mbar, 0);
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_fence_smem();
        tma_store4(&mo, c0, c1, c2, c3, tma_smem(S));
        tma_commit();
        tma_wait_read0();
    }
}
static void map(CUtensorMap &m, void *p, int w, int kind, CUtensorMapL2promotion pr)
{
    // {2 n1 doubles, n2, m1, m2}: x = n1 + 64 n2, y = m1 + 64 m2
    cuuint64_t dims[4] = {2 * PP, QQ, PP, QQ};
    cuuint64_t strides[3] = {(cuuint64_t)PP * 16, (cuuint64_t)NN * 16, (cuuint64_t)PP * NN * 16};
    cuuint32_t boxA[4] = {(cuuint32_t)(2 * w), QQ, 1, QQ};
    cuuint32_t boxB[4] = {2 * PP, 1, PP, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, p, dims, strides, kind == 0 ? boxA : boxB, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}
int main()
{
    const size_t n = (size_t)NN * NN;
    double2 *A, *B;
    cudaMalloc(&A, n * 16 * 8);     // 8 fields (2 GiB) so that L2 does not hold the data
    cudaMalloc(&B, n * 16 * 8);
    cudaMemset(A, 0, n * 16 * 8);
    cudaFuncSetAttribute(tile_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 256);
    const char *pn[] = {"none", "64B", "128B", "256B"};
    CUtensorMapL2promotion prs[] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    for (int kind = 0; kind < 2; ++kind)
        for (int w : {1, 2}) {
            if (kind == 1 && w == 2) continue;
            for (int pi = 0; pi < 4; ++pi) {
                CUtensorMap mi[8], mo[8];
                for (int f = 0; f < 8; ++f) { map(mi[f], A + f * n, w, kind, prs[pi]); map(mo[f], B + f * n, w, kind, prs[pi]); }
                const int tiles = kind == 0 ? PP * (PP / w) : QQ * QQ;
                const size_t sm = kind == 0 ? (size_t)w * 65536 / 1 : 65536;
                if (kind == 0 && w == 2) { printf("(w=2 boxes are 128 KiB: skipped)\n"); break; }
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                for (int f = 0; f < 8; ++f) tile_copy<<<tiles, 128, sm + 256>>>(mi[f], mo[f], w, kind);
                cudaEventRecord(e0);
                for (int r = 0; r < 4; ++r)
                    for (int f = 0; f < 8; ++f) tile_copy<<<tiles, 128, sm + 256>>>(mi[f], mo[f], w, kind);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                printf("%s w=%d promo %-4s: %.1f us per field  %6.0f GB/s  %s\n", kind == 0 ? "AA tile (16B x 64 x 64)" : "B block (64 x 1 KiB)  ",
                       w, pn[pi], ms * 1e3 / 32, 2.0 * n * 16 * 32 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}
