// Phase timestamps of the transposing row pass (rowt.cuh) on one CTA of cluster 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFFTPDE_ROWT_TRACE \
//        -Ipaper_2412_12308_b200/csrc -o tools/exp_rowt tools/exp_rowt.cu
//   ./tools/exp_rowt <clusters> <rows>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "rowt16.cuh"
using namespace fftpde;
__global__ void fill(double2 *p, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_double2((double)((i * 2654435761u) % 1000) * 1e-3, 0.0);
}
template <typename G, typename K> int run(K k, int argc, char **argv);
int main(int argc, char **argv)
{
    const int variant = argc > 3 ? atoi(argv[3]) : 16;
    if (variant == 32) return run<RowTGeom>(rowt_kernel<0>, argc, argv);
    if (variant == 1616) return run<RowT16Geom<16>>(rowt16_kernel<16>, argc, argv);
    return run<RowT16Geom<8>>(rowt16_kernel<8>, argc, argv);
}
template <typename G, typename K> int run(K k, int argc, char **argv)
{
    int ncl = argc > 1 ? atoi(argv[1]) : 1;
    const long nrows0 = argc > 2 ? atol(argv[2]) : 0;
    const long NA = nrows0 ? nrows0 : 8192;
    double2 *in, *out, *twA, *tw32;
    double *mul;
    cudaMalloc(&in, (size_t)NA * G::N * 16);
    cudaMalloc(&out, (size_t)NA * G::N * 16);
    cudaMalloc(&twA, (size_t)G::N * 16);
    cudaMalloc(&tw32, 4096 * 16);
    cudaMalloc(&mul, (size_t)G::N * 8);
    fill<<<1024, 256>>>(in, (size_t)NA * G::N);
    std::vector<double2> one(G::N, make_double2(1.0, 0.0));
    cudaMemcpy(twA, one.data(), G::N * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(tw32, one.data(), 4096 * 16, cudaMemcpyHostToDevice);
    std::vector<double> m(G::N, 1.0 / G::N);
    cudaMemcpy(mul, m.data(), G::N * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(G::NT);
    cfg.dynamicSmemBytes = G::BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = G::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(G::CL);
    int maxcl = 0;
    cudaOccupancyMaxActiveClusters(&maxcl, k, &cfg);
    printf("max active clusters %d (CL %d, %d threads, %zu B smem)\n", maxcl, G::CL, G::NT, G::BYTES);
    if (ncl <= 0) ncl = maxcl;
    const long nrows = nrows0 ? nrows0 : 2L * 64 * ncl;
    cfg.gridDim = dim3(G::CL * ncl);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, (const double2 *)in, out, (int64_t)nrows, (const double2 *)twA,
                                           (const double2 *)tw32, (const double *)mul);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("launch %d: %s  %.3f ms  (%.2f us per iteration, %ld rows, %d clusters)\n", r, cudaGetErrorString(e), ms,
               ms * 1e3 / (nrows / 2.0 / ncl), nrows, ncl);
    }
    long long tr[64][12];
    cudaMemcpyFromSymbol(tr, rowt_trace, sizeof(tr));
    const char *nm[] = {"loads+dftA", "twiddle A", "cl_wait E1", "send E1", "mbar E1", "phase B", "cl_wait E2",
                        "send E2", "mbar E2", "phase A'", "store+loop"};
    double acc[11] = {0};
    int cnt = 0;
    for (int i = 4; i < 60; ++i) {
        for (int p = 0; p < 10; ++p) acc[p] += tr[i][p + 1] - tr[i][p];
        acc[10] += tr[i + 1][0] - tr[i][10];
        ++cnt;
    }
    double tot = 0;
    for (int p = 0; p < 11; ++p) tot += acc[p] / cnt;
    for (int p = 0; p < 11; ++p) printf("  %-12s %8.0f cycles  %5.1f%%\n", nm[p], acc[p] / cnt, 100 * acc[p] / cnt / tot);
    printf("  total        %8.0f cycles per iteration\n", tot);
    return 0;
}
