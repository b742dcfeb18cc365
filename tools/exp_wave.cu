// Experiment harness: TMA wave column pass (one column of U and V per CTA) on the
// C3 shape (4096^2 c128, two fields), checked against col_wave_kernel.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I include tools/exp_wave.cu -o tools/exp_wave
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_2412_12308_b200/csrc/line.cuh"
#include "../paper_2412_12308_b200/csrc/pipe.cuh"
#include "../paper_2412_12308_b200/csrc/tmacols.cuh"
#include "../paper_2412_12308_b200/csrc/kernels.cuh"
#include <cudaTypedefs.h>
#include "experimental/tma_wave1.cuh"
using namespace fftpde;

static const char *g_filter = nullptr;
static int g_reps = 20;
static cudaStream_t g_stream = nullptr;

template <typename C> static void twiddles(int n, int emax, std::vector<C> &tw)
{
    int E = n < emax ? n : emax;
    tw.clear();
    auto put = [&](long M, long q) {
        long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)(q % M) / (long double)M;
        tw.push_back(C{(decltype(C{}.x))cosl(a), (decltype(C{}.x))sinl(a)});
    };
    long ns = 1;
    while (ns * E < n) {
        if (ns > 1)
            for (long m = 0; m < E; ++m)
                for (long k = 0; k < ns; ++k) put(ns * E, m * k);
        ns *= E;
    }
    if (ns > 1)
        for (long m = 0; m < n / ns; ++m)
            for (long j = 0; j < ns; ++j) put(n, m * j);
    if (tw.empty()) tw.push_back(C{1, 0});
}

template <typename C> static C *upload_tw(int n, int emax)
{
    std::vector<C> tw;
    twiddles(n, emax, tw);
    C *d;
    cudaMalloc(&d, tw.size() * sizeof(C));
    cudaMemcpy(d, tw.data(), tw.size() * sizeof(C), cudaMemcpyHostToDevice);
    return d;
}

template <typename T> static OpTables<T> make_tab(int nx, int ny)
{
    std::vector<T> kx(nx), ky(ny), ex(nx), ey(ny);
    for (int a = 0; a < nx; ++a) { int f = 2 * a <= nx ? a : a - nx; kx[a] = (T)((2 * M_PI * f) * (2 * M_PI * f)); ex[a] = (T)(exp(-1e-3 * kx[a] * 0.01) / ((double)nx * ny)); }
    for (int b = 0; b < ny; ++b) { int f = 2 * b <= ny ? b : b - ny; ky[b] = (T)((2 * M_PI * f) * (2 * M_PI * f)); ey[b] = (T)exp(-1e-3 * ky[b] * 0.01); }
    int qx = nx / 2 + 1, qy = ny / 2 + 1;
    std::vector<T> wc((size_t)qx * qy, (T)0.5), ws((size_t)qx * qy, (T)0.1);
    T *d[7];
    auto up = [&](std::vector<T> &v, int i) { cudaMalloc(&d[i], v.size() * sizeof(T)); cudaMemcpy(d[i], v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); };
    up(kx, 0); up(ky, 1); up(ex, 2); up(ey, 3); up(wc, 4); up(ws, 5); up(ws, 6);
    OpTables<T> t{};
    t.kx2 = d[0]; t.ky2 = d[1]; t.ex = d[2]; t.ey = d[3]; t.wC = d[4]; t.wS1 = d[5]; t.wS2 = d[6];
    t.qpitch = qy;
    t.nfold = nx;
    t.scale = (T)(1.0 / ((double)nx * ny));
    return t;
}

template <typename F> static float timeit(F launch, const char *name, double bytes, int occ, long grid)
{
    // launches captured into a CUDA graph: per-kernel time without the ~2 us
    // stream-launch quantum (graph kernel nodes cost ~0.6 us each)
    static cudaStream_t s = nullptr;
    if (!s) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaStream_t prev = g_stream;
    g_stream = s;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < g_reps; ++i) launch();
    cudaStreamEndCapture(s, &g);
    g_stream = prev;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= g_reps;
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaError_t err = cudaGetLastError();
    printf("%-58s occ %2d grid %6ld : %9.2f us  %7.0f GB/s %s\n", name, occ, grid, ms * 1e3,
           bytes / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
    fflush(stdout);
    return ms;
}


static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static CUtensorMap map16(void *p, long nx, long ny, CUtensorMapL2promotion prom)
{
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&g_encode, cudaEnableDefault, &q);
    }
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)(2 * nx), (cuuint64_t)ny, 1};
    cuuint64_t strides[2] = {(cuuint64_t)(nx * 16), (cuuint64_t)(nx * ny * 16)};
    cuuint32_t box[3] = {2, 256, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

template <int EX>
static void run_tma_wave(double2 *U, double2 *V, long n, const void *tw, const OpTables<double> &tab, CUtensorMapL2promotion prom,
                         const char *tag, bool time)
{
    using L = TmaWaveSmem<double2, 4096, EX>;
    auto k = tma_wave_cols_kernel<double, 4096, EX>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    CUtensorMap mu = map16(U, n, n, prom), mv = map16(V, n, n, prom);
    const int threads = 2 * Shape<4096, EX>::TPT;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    auto go = [&] { k<<<(unsigned)n, threads, L::BYTES, g_stream>>>(mu, mv, n, (const double2 *)tw, tab); };
    if (!time) { go(); return; }
    char name[128];
    snprintf(name, sizeof name, "%s TMA wave E=%d prom=%d", tag, EX, (int)prom);
    timeit(go, name, 4.0 * n * n * 16, occ, n);
}

template <int EX, int MINB>
static void run_tma_wave2(double2 *U, double2 *V, long n, const void *tw, const OpTables<double> &tab, const char *tag, bool time)
{
    using L = TmaWave2Smem<double2, 4096, EX>;
    auto k = tma_wave2_cols_kernel<double, 4096, EX, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    CUtensorMap mu = map16(U, n, n, CU_TENSOR_MAP_L2_PROMOTION_L2_256B), mv = map16(V, n, n, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const int threads = Shape<4096, EX>::TPT;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * n), 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = L::BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    auto go = [&] { cfg.stream = g_stream; cudaLaunchKernelEx(&cfg, k, mu, mv, (int64_t)n, (const double2 *)tw, tab, U, V, (int64_t)(n * n)); };
    if (!time) { go(); return; }
    char name[128];
    snprintf(name, sizeof name, "%s TMA wave2 E=%d minb=%d clusters=%d", tag, EX, MINB, ncl);
    timeit(go, name, 4.0 * n * n * 16, ncl, 2 * n);
}

static double maxrel(const double2 *A, const double2 *B, size_t cnt)
{
    std::vector<double2> a(cnt), b(cnt);
    cudaMemcpy(a.data(), A, cnt * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), B, cnt * 16, cudaMemcpyDeviceToHost);
    double m = 0, s = 0;
    for (size_t i = 0; i < cnt; ++i) {
        m = fmax(m, fabs(a[i].x - b[i].x) + fabs(a[i].y - b[i].y));
        s = fmax(s, fabs(b[i].x) + fabs(b[i].y));
    }
    return m / s;
}

int main(int argc, char **argv)
{
    if (argc > 1 && argv[1][0]) g_filter = argv[1];
    if (argc > 2) g_reps = atoi(argv[2]);
    const long n = 4096;
    const size_t cnt = (size_t)n * n;
    double2 *U, *V, *U2, *V2;
    cudaMalloc(&U, cnt * 16); cudaMalloc(&V, cnt * 16); cudaMalloc(&U2, cnt * 16); cudaMalloc(&V2, cnt * 16);
    std::vector<double2> h(cnt), g(cnt);
    for (size_t i = 0; i < cnt; ++i) { h[i] = {sin(0.37 * i), cos(0.11 * i)}; g[i] = {cos(0.23 * i), sin(0.05 * i + 1)}; }
    cudaMemcpy(U, h.data(), cnt * 16, cudaMemcpyHostToDevice); cudaMemcpy(V, g.data(), cnt * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(U2, h.data(), cnt * 16, cudaMemcpyHostToDevice); cudaMemcpy(V2, g.data(), cnt * 16, cudaMemcpyHostToDevice);
    OpTables<double> tab = make_tab<double>(n, n);
    void *t16 = upload_tw<double2>(n, 16), *t32 = upload_tw<double2>(n, 32), *t8 = upload_tw<double2>(n, 8);
    {   // reference: col_wave_kernel (single CTA per column, radix 16)
        using WS = WaveSmem<double2, 4096, 1>;
        auto k = col_wave_kernel<double, 4096, 1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WS::BYTES);
        k<<<dim3((unsigned)n, 1), Shape<4096>::TPT, WS::BYTES>>>(U, V, n, (long)cnt, (const double2 *)t16, tab);
    }
    run_tma_wave<16>(U2, V2, n, t16, tab, CU_TENSOR_MAP_L2_PROMOTION_NONE, "", false);
    cudaDeviceSynchronize();
    printf("TMA wave E16 vs col_wave: U %.3e V %.3e %s\n", maxrel(U2, U, cnt), maxrel(V2, V, cnt), cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(U2, h.data(), cnt * 16, cudaMemcpyHostToDevice); cudaMemcpy(V2, g.data(), cnt * 16, cudaMemcpyHostToDevice);
    run_tma_wave<32>(U2, V2, n, t32, tab, CU_TENSOR_MAP_L2_PROMOTION_NONE, "", false);
    cudaDeviceSynchronize();
    printf("TMA wave E32 vs col_wave: U %.3e V %.3e %s\n", maxrel(U2, U, cnt), maxrel(V2, V, cnt), cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(U2, h.data(), cnt * 16, cudaMemcpyHostToDevice); cudaMemcpy(V2, g.data(), cnt * 16, cudaMemcpyHostToDevice);
    run_tma_wave2<16, 2>(U2, V2, n, t16, tab, "", false);
    cudaDeviceSynchronize();
    printf("TMA wave2 E16 vs col_wave: U %.3e V %.3e %s\n", maxrel(U2, U, cnt), maxrel(V2, V, cnt), cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(U2, h.data(), cnt * 16, cudaMemcpyHostToDevice); cudaMemcpy(V2, g.data(), cnt * 16, cudaMemcpyHostToDevice);
    run_tma_wave2<32, 1>(U2, V2, n, t32, tab, "", false);
    cudaDeviceSynchronize();
    printf("TMA wave2 E32 vs col_wave: U %.3e V %.3e %s\n", maxrel(U2, U, cnt), maxrel(V2, V, cnt), cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(U2, h.data(), cnt * 16, cudaMemcpyHostToDevice); cudaMemcpy(V2, g.data(), cnt * 16, cudaMemcpyHostToDevice);
    run_tma_wave2<8, 2>(U2, V2, n, t8, tab, "", false);
    cudaDeviceSynchronize();
    printf("TMA wave2 E8 vs col_wave: U %.3e V %.3e %s\n", maxrel(U2, U, cnt), maxrel(V2, V, cnt), cudaGetErrorString(cudaGetLastError()));
    run_tma_wave2<16, 2>(U, V, n, t16, tab, "c3", true);
    run_tma_wave2<8, 2>(U, V, n, t8, tab, "c3", true);
    run_tma_wave2<8, 3>(U, V, n, t8, tab, "c3", true);
    run_tma_wave2<16, 3>(U, V, n, t16, tab, "c3", true);
    run_tma_wave2<16, 1>(U, V, n, t16, tab, "c3", true);
    run_tma_wave2<32, 1>(U, V, n, t32, tab, "c3", true);
    run_tma_wave2<32, 2>(U, V, n, t32, tab, "c3", true);
    {
        using WS = WaveSmem<double2, 4096, 1>;
        auto k = col_wave_kernel<double, 4096, 1>;
        timeit([&] { k<<<dim3((unsigned)n, 1), Shape<4096>::TPT, WS::BYTES, g_stream>>>(U, V, n, (long)cnt, (const double2 *)t16, tab); },
               "c3 col_wave W=1", 4.0 * cnt * 16, 1, n);
    }
    run_tma_wave<16>(U, V, n, t16, tab, CU_TENSOR_MAP_L2_PROMOTION_NONE, "c3", true);
    run_tma_wave<16>(U, V, n, t16, tab, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, "c3", true);
    run_tma_wave<16>(U, V, n, t16, tab, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "c3", true);
    run_tma_wave<32>(U, V, n, t32, tab, CU_TENSOR_MAP_L2_PROMOTION_NONE, "c3", true);
    run_tma_wave<32>(U, V, n, t32, tab, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, "c3", true);
    printf("done\n");
    return 0;
}
