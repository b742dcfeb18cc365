// Experiment: col2_kernel (cluster four-step column pass) launch variants on 4096^2 c128.
#include <cstdio>
#include <cstring>
#include <vector>
#include <cmath>
#include "../paper_2412_12308_b200/csrc/col2.cuh"
using namespace fftpde;
static const char *g_filter = nullptr;
static void stage_tw(long n, int emax, std::vector<double2> &tw)
{
    long E = n < emax ? n : emax;
    tw.clear();
    auto put = [&](long M, long q) { long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)(q % M) / (long double)M; tw.push_back({(double)cosl(a), (double)sinl(a)}); };
    long ns = 1;
    while (ns * E < n) { if (ns > 1) for (long m = 0; m < E; ++m) for (long k = 0; k < ns; ++k) put(ns * E, m * k); ns *= E; }
    if (ns > 1) for (long m = 0; m < n / ns; ++m) for (long j = 0; j < ns; ++j) put(n, m * j);
    if (tw.empty()) tw.push_back({1, 0});
}
template <typename T> T *up(const std::vector<T> &v) { T *d; cudaMalloc(&d, v.size() * sizeof(T)); cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); return d; }

template <int P, int Q, int OP, int CL, int NT, int MINB, int EMAX>
void var(Col2Args<double> g, OpTables<double> tab, long n, const char *tag)
{
    char name[128];
    snprintf(name, sizeof name, "%s op=%d CL=%d NT=%d MINB=%d E=%d", tag, OP, CL, NT, MINB, EMAX);
    if (g_filter && !strstr(name, g_filter)) return;
    using IA = Col2Items<double2, Q, NT, EMAX>;
    using IB = Col2Items<double2, P, NT, EMAX>;
    size_t sa = (size_t)IA::SLOTS * IA::SLOT_ELEMS * 16, sb = (size_t)IB::SLOTS * IB::SLOT_ELEMS * 16;
    size_t smem = sa > sb ? sa : sb;
    auto k = col2_kernel<double, P, Q, OP, CL, NT, MINB, EMAX>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(CL * g.nblocks), 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    for (int i = 0; i < 2; ++i) cudaLaunchKernelEx(&cfg, k, g, tab);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, k, g, tab);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    const double bytes = (OP == C2_WAVE ? 4.0 : 2.0) * (double)n * n * 16;
    printf("%-48s clusters %3d smem %6zu : %8.1f us %6.0f GB/s %s\n", name, ncl, smem, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
}

int main(int argc, char **argv)
{
    if (argc > 1) g_filter = argv[1];
    const long n = 4096;
    double2 *U, *V;
    cudaMalloc(&U, n * n * 16); cudaMalloc(&V, n * n * 16);
    cudaMemset(U, 0, n * n * 16); cudaMemset(V, 0, n * n * 16);
    std::vector<double2> tp; stage_tw(64, 8, tp); double2 *dtp = up(tp);
    std::vector<double2> tp16; stage_tw(64, 16, tp16); double2 *dtp16 = up(tp16);
    std::vector<double2> tn(n);
    for (long m = 0; m < n; ++m) { long double a = 2.0L * 3.14159265358979323846264338327950288L * m / n; tn[m] = {(double)cosl(a), (double)sinl(a)}; }
    double2 *dtn = up(tn);
    std::vector<double> k2(n);
    for (long a = 0; a < n; ++a) { long f = 2 * a <= n ? a : a - n; k2[a] = (2 * M_PI * f) * (2 * M_PI * f); }
    double *dk2 = up(k2);
    std::vector<double> q((n / 2 + 1) * (n / 2 + 1), 0.5); double *dq = up(q);
    OpTables<double> tab{}; tab.kx2 = dk2; tab.ky2 = dk2; tab.ex = dk2; tab.ey = dk2; tab.wC = dq; tab.wS1 = dq; tab.wS2 = dq;
    tab.qpitch = n / 2 + 1; tab.nfold = n; tab.scale = 1.0 / (n * n);
    Col2Args<double> g{U, V, U, n, n * n, n / 8, dtp, dtp, dtn};
    Col2Args<double> g16{U, V, U, n, n * n, n / 8, dtp16, dtp16, dtn};
    var<64, 64, C2_WAVE, 8, 256, 2, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 256, 1, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 512, 1, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 4, 512, 1, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 16, 256, 2, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 4, 256, 2, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 256, 3, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 128, 4, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 128, 3, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 128, 2, 8>(g, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 256, 2, 16>(g16, tab, n, "wave");
    var<64, 64, C2_WAVE, 8, 256, 1, 16>(g16, tab, n, "wave");
    var<64, 64, C2_POISSON, 8, 256, 2, 8>(g, tab, n, "poisson");
    var<64, 64, C2_POISSON, 8, 512, 1, 8>(g, tab, n, "poisson");
    var<64, 64, C2_POISSON, 8, 256, 3, 8>(g, tab, n, "poisson");
    var<64, 64, C2_POISSON, 8, 128, 4, 8>(g, tab, n, "poisson");
    var<64, 64, C2_POISSON, 8, 256, 2, 16>(g16, tab, n, "poisson");
    printf("done\n");
    return 0;
}
