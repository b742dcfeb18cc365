// Experiment: DSMEM-resident four-step row pass (row2d) vs the L2 two-level
// row pass (row2) on long complex128 rows: agreement and timing.
#include <cstdio>
#include <cstring>
#include <vector>
#include <cmath>
#include <random>
#include "experimental/row2.cuh"
#include "../paper_2412_12308_b200/csrc/row2d.cuh"
using namespace fftpde;
static const char *g_filter = nullptr;

static double2 root(long n, long m)
{
    long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)(((m % n) + n) % n) / (long double)n;
    return {(double)cosl(a), (double)sinl(a)};
}
static void stage_tw(long n, int emax, std::vector<double2> &tw)
{
    long E = n < emax ? n : emax;
    tw.clear();
    long ns = 1;
    while (ns * E < n) { if (ns > 1) for (long m = 0; m < E; ++m) for (long k = 0; k < ns; ++k) tw.push_back(root(ns * E, m * k)); ns *= E; }
    if (ns > 1) for (long m = 0; m < n / ns; ++m) for (long j = 0; j < ns; ++j) tw.push_back(root(n, m * j));
    if (tw.empty()) tw.push_back({1, 0});
}
template <typename T> T *up(const std::vector<T> &v) { T *d; cudaMalloc(&d, v.size() * sizeof(T)); cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); return d; }

template <typename F> float timeit(F f, int reps)
{
    for (int i = 0; i < 2; ++i) f();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

template <int P, int Q> struct Tabs {
    double2 *tP8, *tQ8, *tN, *tP16, *tQ16, *tS;
    Tabs()
    {
        constexpr long N = (long)P * Q;
        std::vector<double2> v;
        stage_tw(P, 8, v); tP8 = up(v);
        stage_tw(Q, 8, v); tQ8 = up(v);
        stage_tw(P, 16, v); tP16 = up(v);
        stage_tw(Q, 16, v); tQ16 = up(v);
        v.resize(N); for (long m = 0; m < N; ++m) v[m] = root(N, m); tN = up(v);
        v.clear();
        for (long a = 0; a < P; ++a) for (long l = 0; l < 16; ++l) v.push_back(root(N, a * l));
        for (long a = 0; a < P; ++a) for (long h = 0; h < Q / 16; ++h) v.push_back(root(N, 16 * a * h));
        for (long k = 0; k < Q; ++k) for (long l = 0; l < 16; ++l) v.push_back(root(N, k * l));
        for (long k = 0; k < Q; ++k) for (long h = 0; h < P / 16; ++h) v.push_back(root(N, 16 * k * h));
        tS = up(v);
    }
};

template <int P, int Q, int CL, int OP>
float run_new(const double2 *in, double2 *out, double2 *out2, long nrows, const Tabs<P, Q> &t, int reps, bool print)
{
    using G = Row2dGeom<double2, P, Q, CL>;
    auto k = row2d_kernel<double, P, Q, CL, OP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::BYTES);
    if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(G::NT, 1, 1);
    cfg.dynamicSmemBytes = G::BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    cfg.gridDim = dim3(CL, 1, 1);
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    long g = ncl < nrows ? ncl : nrows;
    if (g < 1) g = 1;
    cfg.gridDim = dim3((unsigned)(g * CL), 1, 1);
    const long N = (long)P * Q;
    auto f = [&] { cudaLaunchKernelEx(&cfg, k, in, out, out2, nrows, nrows, N * nrows, t.tP16, t.tQ16, t.tS, (const double *)nullptr); };
    float ms = timeit(f, reps);
    if (print) {
        const double bytes = (OP == R2D_MID ? 3.0 : 2.0) * N * nrows * 16;
        printf("row2d N=%ld CL=%d op=%d NT=%d smem=%zu clusters=%d(%s): %9.1f us %6.0f GB/s %s\n", N, CL, OP, G::NT, G::BYTES,
               ncl, cudaGetErrorString(e), ms * 1e3, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
    }
    return ms;
}

template <int P, int Q, bool INV>
float run_old(const double2 *in, double2 *out, long nrows, const Tabs<P, Q> &t, int reps)
{
    constexpr int EMAX = 8, CL = 8, NT = 256;
    using Sm = Row2Smem<double, P, Q, NT, EMAX>;
    auto k = row2_kernel<double, P, Q, INV, CL, NT, EMAX>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sm::BYTES);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(CL * nrows), 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = Sm::BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    const long N = (long)P * Q;
    auto f = [&] { cudaLaunchKernelEx(&cfg, k, in, out, nrows, nrows, N * nrows, t.tP8, t.tQ8, t.tN); };
    float ms = timeit(f, reps);
    printf("row2 (old) N=%ld inv=%d: %9.1f us %6.0f GB/s %s\n", N, INV, ms * 1e3, 2.0 * N * nrows * 16 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
    return ms;
}

static double rel(const std::vector<double2> &a, const std::vector<double2> &b)
{
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        double dx = a[i].x - b[i].x, dy = a[i].y - b[i].y;
        num += dx * dx + dy * dy;
        den += b[i].x * b[i].x + b[i].y * b[i].y;
    }
    return std::sqrt(num / den);
}

template <int P, int Q> void suite(long nrows_big)
{
    constexpr long N = (long)P * Q;
    Tabs<P, Q> t;
    // correctness on a few rows
    const long nr = 64;
    std::vector<double2> h(N * nr);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    for (auto &z : h) z = {nd(rng), nd(rng)};
    double2 *x = up(h), *y1, *y2, *y3;
    cudaMalloc(&y1, N * nr * 16); cudaMalloc(&y2, N * nr * 16); cudaMalloc(&y3, N * nr * 16);
    std::vector<double2> a(N * nr), b(N * nr), c(N * nr);
    run_old<P, Q, false>(x, y1, nr, t, 1);
    run_new<P, Q, 8, R2D_FWD>(x, y2, nullptr, nr, t, 1, false);
    cudaMemcpy(a.data(), y1, N * nr * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), y2, N * nr * 16, cudaMemcpyDeviceToHost);
    printf("N=%ld FWD new vs old rel %.3e\n", N, rel(b, a));
    run_new<P, Q, 16, R2D_FWD>(x, y2, nullptr, nr, t, 1, false);
    cudaMemcpy(b.data(), y2, N * nr * 16, cudaMemcpyDeviceToHost);
    printf("N=%ld FWD CL16 new vs old rel %.3e\n", N, rel(b, a));
    run_old<P, Q, true>(x, y1, nr, t, 1);
    run_new<P, Q, 8, R2D_INV>(x, y2, nullptr, nr, t, 1, false);
    cudaMemcpy(a.data(), y1, N * nr * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), y2, N * nr * 16, cudaMemcpyDeviceToHost);
    printf("N=%ld INV new vs old rel %.3e\n", N, rel(b, a));
    // MID: out2 = inv(x), out = fwd(inv(x)) -> out == N * x
    run_new<P, Q, 8, R2D_MID>(x, y2, y3, nr, t, 1, false);
    cudaMemcpy(b.data(), y2, N * nr * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), y3, N * nr * 16, cudaMemcpyDeviceToHost);
    for (auto &z : b) { z.x /= N; z.y /= N; }
    printf("N=%ld MID: phys vs old inv rel %.3e, fwd(inv(x))/N vs x rel %.3e\n", N, rel(c, a), rel(b, h));
    cudaFree(x); cudaFree(y1); cudaFree(y2); cudaFree(y3);
    // timing on nrows_big rows (256 MiB+)
    double2 *A, *B, *Cc;
    cudaMalloc(&A, N * nrows_big * 16); cudaMalloc(&B, N * nrows_big * 16); cudaMalloc(&Cc, N * nrows_big * 16);
    cudaMemset(A, 0, N * nrows_big * 16);
    run_old<P, Q, false>(A, B, nrows_big, t, 5);
    run_new<P, Q, 8, R2D_FWD>(A, B, nullptr, nrows_big, t, 5, true);
    run_new<P, Q, 16, R2D_FWD>(A, B, nullptr, nrows_big, t, 5, true);
    run_new<P, Q, 8, R2D_MID>(A, B, Cc, nrows_big, t, 5, true);
    run_new<P, Q, 16, R2D_MID>(A, B, Cc, nrows_big, t, 5, true);
    cudaFree(A); cudaFree(B); cudaFree(Cc);
}

int main(int argc, char **argv)
{
    if (argc > 1) g_filter = argv[1];
    suite<128, 256>(2048);   // 32768-point rows, 1 GiB
    suite<128, 128>(4096);   // 16384-point rows, 1 GiB
    return 0;
}
