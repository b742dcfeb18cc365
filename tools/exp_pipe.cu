// Experiment harness: variants of pipe_kernel on a 4096^2 complex128 field.
#include <cstdio>
#include <cstring>
static const char* g_filter = nullptr;
#include <cmath>
#include <vector>
#include "../paper_2412_12308_b200/csrc/pipe.cuh"
using namespace fftpde;

static void twiddles(int n, std::vector<double2>& tw) {
    int E = n < 16 ? n : 16; tw.clear();
    auto put = [&](long M, long q) { long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)(q % M) / (long double)M; tw.push_back({(double)cosl(a), (double)sinl(a)}); };
    long ns = 1;
    while (ns * E < n) { if (ns > 1) for (long m = 0; m < E; ++m) for (long k = 0; k < ns; ++k) put(ns * E, m * k); ns *= E; }
    if (ns > 1) for (long m = 0; m < n / ns; ++m) for (long j = 0; j < ns; ++j) put(n, m * j);
}

template <typename K> float run(K k, int threads, size_t smem, const double2* in, double2* out, PipeArgs a, const double2* tw, OpTables<double> tab, const char* name, double bytes) {
    if (g_filter && !strstr(name, g_filter)) return 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
    int grid = occ * 148; if (grid > a.ntiles) grid = a.ntiles;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<grid, threads, smem>>>(in, out, a, tw, tab);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) k<<<grid, threads, smem>>>(in, out, a, tw, tab);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    cudaError_t err = cudaGetLastError();
    printf("%-40s occ %d grid %5d : %8.1f us  %6.0f GB/s  %s\n", name, occ, grid, ms * 1e3, bytes / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
    return ms;
}

template <int NN, int WW, bool COLS, int NB, int MB, bool TR>
void var32(const float2* in, float2* out, const float2* tw, OpTables<float> tab, long nlines, long batch, const char* name, int op = PIPE_POISSON) {
    if (!COLS) op = PIPE_FWD;
    if (g_filter && !strstr(name, g_filter)) return;
    using L = PipeSmem<float2, NN, WW, COLS, NB>;
    auto k = (op == PIPE_FWD) ? pipe_kernel<float, NN, WW, COLS, PIPE_FWD, NB, MB, TR> : (COLS ? pipe_kernel<float, NN, WW, COLS, PIPE_POISSON, NB, MB, TR> : pipe_kernel<float, NN, WW, COLS, PIPE_FWD, NB, MB, TR>);
    PipeArgs a = COLS ? PipeArgs{nlines, 1, NN, (long)NN * nlines, batch * (nlines / WW), nlines / WW, op}
                      : PipeArgs{NN, NN, 1, (long)NN * NN, batch * (NN / WW), NN / WW, PIPE_FWD};
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int threads = WW * Shape<NN>::TPT;
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    long grid = occ * 148; if (grid > a.ntiles) grid = a.ntiles;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<grid, threads, L::BYTES>>>(in, out, a, tw, tab);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) k<<<grid, threads, L::BYTES>>>(in, out, a, tw, tab);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    double bytes = 2.0 * 8 * NN * NN * batch;
    cudaError_t err = cudaGetLastError();
    printf("c64 %-44s W=%2d occ %d : %8.1f us  %6.0f GB/s %s\n", name, WW, occ, ms * 1e3, bytes / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
}

#define ROWV(NB, MB, TR) { using L = PipeSmem<double2, N, 1, false, NB>; auto k = pipe_kernel<double, N, 1, false, PIPE_FWD, NB, MB, TR>; \
    PipeArgs a{n, n, 1, (long)n * n, n, n, PIPE_FWD}; run(k, 256, L::BYTES, in, out, a, dtw, tab1, "rows nbuf=" #NB " minb=" #MB " twreg=" #TR, bytes); }
#define COLV(W, NB, MB, TR) { using L = PipeSmem<double2, N, W, true, NB>; auto k = pipe_kernel<double, N, W, true, PIPE_POISSON, NB, MB, TR>; \
    PipeArgs a{n, 1, n, (long)n * n, n / W, n / W, PIPE_POISSON}; run(k, 256 * W, L::BYTES, out, out, a, dtw, tab, "cols W=" #W " nbuf=" #NB " minb=" #MB " twreg=" #TR, bytes); }

int main(int argc, char** argv) {
    if (argc > 1) g_filter = argv[1];
    constexpr int N = 4096; const long n = N;
    double2 *in, *out; cudaMalloc(&in, n * n * 16); cudaMalloc(&out, n * n * 16);
    cudaMemset(in, 0, n * n * 16);
    std::vector<double2> tw; twiddles(N, tw);
    double2* dtw; cudaMalloc(&dtw, tw.size() * 16); cudaMemcpy(dtw, tw.data(), tw.size() * 16, cudaMemcpyHostToDevice);
    std::vector<double> k2(n); for (long a = 0; a < n; ++a) { long f = 2 * a <= n ? a : a - n; k2[a] = (2 * M_PI * f) * (2 * M_PI * f); }
    double* dk2; cudaMalloc(&dk2, n * 8); cudaMemcpy(dk2, k2.data(), n * 8, cudaMemcpyHostToDevice);
    OpTables<double> tab{}; tab.kx2 = dk2; tab.ky2 = dk2; tab.ex = dk2; tab.ey = dk2; tab.scale = 1.0 / (n * n);
    OpTables<double> tab1{}; tab1.scale = 1.0;
    double bytes = 2.0 * n * n * 16;
    ROWV(2, 1, true) ROWV(3, 1, true) ROWV(3, 1, false) ROWV(1, 2, false)
    COLV(1, 2, 1, true) COLV(1, 3, 1, true) COLV(1, 3, 1, false) COLV(1, 1, 2, false)
    COLV(2, 1, 1, false)
    { using L = PipeSmem<double2, N, 2, true, 1>; auto k = pipe_kernel<double, N, 2, true, PIPE_FWD, 1, 1, false>;
      PipeArgs a{n, 1, n, (long)n * n, n / 2, n / 2, PIPE_FWD}; run(k, 512, L::BYTES, out, out, a, dtw, tab, "cols W=2 FWD only", bytes); }
    {
        std::vector<double2> t64; twiddles(512, t64);
        std::vector<float2> t32(t64.size()); for (size_t i = 0; i < t64.size(); ++i) t32[i] = {(float)t64[i].x, (float)t64[i].y};
        float2* dt32; cudaMalloc(&dt32, t32.size() * 8); cudaMemcpy(dt32, t32.data(), t32.size() * 8, cudaMemcpyHostToDevice);
        std::vector<float> k2f(512); for (int a = 0; a < 512; ++a) { int f = 2 * a <= 512 ? a : a - 512; k2f[a] = (float)((2 * M_PI * f) * (2 * M_PI * f)); }
        float* dk2f; cudaMalloc(&dk2f, 512 * 4); cudaMemcpy(dk2f, k2f.data(), 512 * 4, cudaMemcpyHostToDevice);
        OpTables<float> tf{}; tf.kx2 = dk2f; tf.ky2 = dk2f; tf.scale = 1.0f / (512 * 512);
        OpTables<float> tf1{}; tf1.scale = 1.0f;
        float2* a32 = (float2*)in; float2* b32 = (float2*)out;   // 256 grids of 512^2 c64 = 512 MiB
        var32<512, 8, false, 1, 2, false>(a32, b32, dt32, tf1, 512, 256, "rows nbuf1 minb2");
        var32<512, 8, false, 3, 1, true>(a32, b32, dt32, tf1, 512, 256, "rows nbuf3 twreg");
        var32<512, 8, false, 4, 1, true>(a32, b32, dt32, tf1, 512, 256, "rows nbuf4 twreg");
        var32<512, 4, false, 4, 2, false>(a32, b32, dt32, tf1, 512, 256, "rows nbuf4 minb2");
        var32<512, 16, true, 1, 2, false>(b32, b32, dt32, tf, 512, 256, "cols FWD nbuf1 minb2", PIPE_FWD);
        var32<512, 16, true, 3, 1, false>(b32, b32, dt32, tf, 512, 256, "cols FWD nbuf3", PIPE_FWD);
        var32<512, 16, true, 1, 2, false>(b32, b32, dt32, tf, 512, 256, "cols nbuf1 minb2");
        var32<512, 16, true, 3, 1, false>(b32, b32, dt32, tf, 512, 256, "cols nbuf3");
        var32<512, 8, true, 3, 1, false>(b32, b32, dt32, tf, 512, 256, "cols nbuf3");
        var32<512, 8, true, 4, 1, false>(b32, b32, dt32, tf, 512, 256, "cols nbuf4");
        var32<512, 8, true, 3, 2, false>(b32, b32, dt32, tf, 512, 256, "cols nbuf3 minb2");
        var32<512, 4, true, 4, 2, false>(b32, b32, dt32, tf, 512, 256, "cols nbuf4 minb2");
    }
    return 0;
}
