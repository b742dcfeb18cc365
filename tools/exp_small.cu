// Experiment: 1024 x 1024 complex128 (C2) row and column pass variants (L2-resident field).
#include <cstdio>
#include <cstring>
#include <vector>
#include <cmath>
#include "../paper_2412_12308_b200/csrc/pipe.cuh"
#include "../paper_2412_12308_b200/csrc/col2.cuh"
using namespace fftpde;
static void stage_tw(long n, int emax, std::vector<double2>& tw) {
    long E = n < emax ? n : emax; tw.clear();
    auto put = [&](long M, long q) { long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)(q % M) / (long double)M; tw.push_back({(double)cosl(a), (double)sinl(a)}); };
    long ns = 1;
    while (ns * E < n) { if (ns > 1) for (long m = 0; m < E; ++m) for (long k = 0; k < ns; ++k) put(ns * E, m * k); ns *= E; }
    if (ns > 1) for (long m = 0; m < n / ns; ++m) for (long j = 0; j < ns; ++j) put(n, m * j);
    if (tw.empty()) tw.push_back({1, 0});
}
template <typename T> T* up(const std::vector<T>& v) { T* d; cudaMalloc(&d, v.size() * sizeof(T)); cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); return d; }
template <int W, bool COLS, int OP, int NBUF, int MINB, bool TWREG>
void var(const double2* in, double2* out, const double2* tw, OpTables<double> tab, const char* name, bool persistent) {
    constexpr int N = 1024;
    using L = PipeSmem<double2, N, W, COLS, NBUF>;
    auto k = pipe_kernel<double, N, W, COLS, OP, NBUF, MINB, TWREG>;
    PipeArgs a = COLS ? PipeArgs{N, 1, N, (long)N * N, N / W, N / W, OP} : PipeArgs{N, N, 1, (long)N * N, N / W, N / W, OP};
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int threads = W * Shape<N>::TPT;
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    long grid = persistent ? (long)occ * 148 : a.ntiles; if (grid > a.ntiles) grid = a.ntiles;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int i = 0; i < 5; ++i) k<<<grid, threads, L::BYTES, s>>>(in, out, a, tw, tab);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 50; ++i) k<<<grid, threads, L::BYTES, s>>>(in, out, a, tw, tab);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 50;
    printf("%-34s W=%2d occ %d grid %4ld: %6.2f us  %6.0f GB/s %s\n", name, W, occ, grid, ms * 1e3, 2.0 * 16 * N * N / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const long n = 1024;
    double2 *U, *V; cudaMalloc(&U, n * n * 16); cudaMalloc(&V, n * n * 16); cudaMemset(U, 0, n * n * 16); cudaMemset(V, 0, n * n * 16);
    std::vector<double2> t16; stage_tw(n, 16, t16); double2* dt16 = up(t16);
    std::vector<double> k2(n); for (long a = 0; a < n; ++a) { long f = 2 * a <= n ? a : a - n; k2[a] = (2 * M_PI * f) * (2 * M_PI * f); } double* dk2 = up(k2);
    OpTables<double> tab{}; tab.kx2 = dk2; tab.ky2 = dk2; tab.ex = dk2; tab.ey = dk2; tab.scale = 1.0 / (n * n);
    OpTables<double> tab1{}; tab1.scale = 1.0;
    var<4, false, PIPE_FWD, 2, 1, true>(U, V, dt16, tab1, "rows (current) persistent", true);
    var<4, false, PIPE_FWD, 2, 1, true>(U, V, dt16, tab1, "rows nonpersistent", false);
    var<4, false, PIPE_FWD, 1, 1, false>(U, V, dt16, tab1, "rows nbuf1", false);
    var<2, false, PIPE_FWD, 1, 1, false>(U, V, dt16, tab1, "rows nbuf1", false);
    var<1, false, PIPE_FWD, 1, 1, false>(U, V, dt16, tab1, "rows nbuf1", false);
    var<2, false, PIPE_FWD, 1, 2, false>(U, V, dt16, tab1, "rows nbuf1 minb2", false);
    var<1, false, PIPE_FWD, 1, 4, false>(U, V, dt16, tab1, "rows nbuf1 minb4", false);
    var<4, true, PIPE_DIFFUSE, 2, 1, true>(V, V, dt16, tab, "cols (current) persistent", true);
    var<4, true, PIPE_DIFFUSE, 1, 1, false>(V, V, dt16, tab, "cols nbuf1", false);
    var<8, true, PIPE_DIFFUSE, 1, 1, false>(V, V, dt16, tab, "cols nbuf1", false);
    var<2, true, PIPE_DIFFUSE, 1, 2, false>(V, V, dt16, tab, "cols nbuf1 minb2", false);
    var<4, true, PIPE_DIFFUSE, 1, 2, false>(V, V, dt16, tab, "cols nbuf1 minb2", false);
    var<1, false, PIPE_FWD, 2, 3, false>(U, V, dt16, tab1, "rows nbuf2 minb3", true);
    var<1, false, PIPE_FWD, 2, 4, false>(U, V, dt16, tab1, "rows nbuf2 minb4", true);
    var<2, true, PIPE_DIFFUSE, 2, 2, false>(V, V, dt16, tab, "cols nbuf2 minb2", true);
    var<8, true, PIPE_DIFFUSE, 1, 1, false>(V, V, dt16, tab, "cols nbuf1 W8", false);
    return 0;
}
