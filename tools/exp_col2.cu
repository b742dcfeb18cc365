// Experiment: two-level column pass, cluster (3 phases in 1 launch) vs phase-split (3 launches).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2412_12308_b200/csrc/col2.cuh"
#include "experimental/col2_phase.cuh"
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
template <int PH, int OP, int NT, int MINB> float run_phase(Col2Args<double> g, OpTables<double> tab, long nitems) {
    using I = Col2Items<double2, PH == PH_B ? 64 : 64, NT, 8>;
    size_t smem = I::SLOTS * I::SLOT_ELEMS * 16;
    auto k = col2_phase_kernel<double, 64, 64, PH, OP, NT, MINB, 8>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem);
    long grid = (nitems + I::SLOTS - 1) / I::SLOTS;
    long gmax = (long)occ * 148 * 4; if (grid > gmax) grid = gmax;
    for (int i = 0; i < 2; ++i) k<<<grid, NT, smem>>>(g, tab, nitems);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int i = 0; i < 10; ++i) k<<<grid, NT, smem>>>(g, tab, nitems); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("  phase %d op %d NT %d MINB %d occ %d grid %ld: %7.1f us  %6.0f GB/s %s\n", PH, OP, NT, MINB, occ, grid, ms * 1e3, (OP == C2_WAVE ? 4.0 : 2.0) * 4096.0 * 4096 * 16 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    return ms;
}
int main() {
    const long n = 4096;
    double2 *U, *V; cudaMalloc(&U, n * n * 16); cudaMalloc(&V, n * n * 16); cudaMemset(U, 0, n * n * 16); cudaMemset(V, 0, n * n * 16);
    std::vector<double2> tp; stage_tw(64, 8, tp); double2* dtp = up(tp);
    std::vector<double2> tn(n); for (long m = 0; m < n; ++m) { long double a = 2.0L * 3.14159265358979323846264338327950288L * m / n; tn[m] = {(double)cosl(a), (double)sinl(a)}; } double2* dtn = up(tn);
    std::vector<double> k2(n); for (long a = 0; a < n; ++a) { long f = 2 * a <= n ? a : a - n; k2[a] = (2 * M_PI * f) * (2 * M_PI * f); } double* dk2 = up(k2);
    std::vector<double> q((n / 2 + 1) * (n / 2 + 1), 0.5); double* dq = up(q);
    OpTables<double> tab{}; tab.kx2 = dk2; tab.ky2 = dk2; tab.ex = dk2; tab.ey = dk2; tab.wC = dq; tab.wS1 = dq; tab.wS2 = dq; tab.qpitch = n / 2 + 1; tab.nfold = n; tab.scale = 1.0 / (n * n);
    Col2Args<double> g{U, V, U, n, n * n, n / 8, dtp, dtp, dtn};
    long nb = n / 8;
    printf("poisson, phase split:\n");
    float t = 0;
    t += run_phase<PH_A_FWD, C2_POISSON, 256, 2>(g, tab, nb * 64);
    t += run_phase<PH_B, C2_POISSON, 256, 2>(g, tab, nb * 64);
    t += run_phase<PH_A_INV, C2_POISSON, 256, 2>(g, tab, nb * 64);
    printf("  total %.1f us\n", t * 1e3);
    t = 0;
    t += run_phase<PH_A_FWD, C2_POISSON, 128, 4>(g, tab, nb * 64);
    t += run_phase<PH_B, C2_POISSON, 128, 4>(g, tab, nb * 64);
    t += run_phase<PH_A_INV, C2_POISSON, 128, 4>(g, tab, nb * 64);
    printf("  total %.1f us\n", t * 1e3);
    t = 0;
    t += run_phase<PH_A_FWD, C2_POISSON, 256, 3>(g, tab, nb * 64);
    t += run_phase<PH_B, C2_POISSON, 256, 3>(g, tab, nb * 64);
    t += run_phase<PH_A_INV, C2_POISSON, 256, 3>(g, tab, nb * 64);
    printf("  total %.1f us\n", t * 1e3);
    printf("wave, phase split:\n");
    t = 0;
    t += run_phase<PH_A_FWD, C2_WAVE, 256, 2>(g, tab, nb * 128);
    t += run_phase<PH_B, C2_WAVE, 256, 2>(g, tab, nb * 64);
    t += run_phase<PH_A_INV, C2_WAVE, 256, 2>(g, tab, nb * 128);
    printf("  total %.1f us\n", t * 1e3);
    return 0;
}
