// Experiment harness: line_kernel variants (E, W, MINB) vs pipe_kernel on the
// pass shapes of C2 (1024^2 c128), C3 (4096^2 c128 rows), C4 (512^2 x 256 c64).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I include tools/exp_line.cu -o tools/exp_line
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_2412_12308_b200/csrc/line.cuh"
#include "../paper_2412_12308_b200/csrc/pipe.cuh"
#include "experimental/rr.cuh"
#include "experimental/tpipe.cuh"
#include "experimental/wave_line.cuh"
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

// ---- line_kernel variant
template <typename T, int N, int E, int W, bool COLS, int OP, int MINB>
static void line_var(const void *in, void *out, void *out2, long nx, long ny, long batch, const void *tw,
                     const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s line E=%d W=%d minb=%d", tag, E, W, MINB);
    if (g_filter && !strstr(name, g_filter)) return;
    using L = LineSmem<C, N, E, W, COLS>;
    auto k = line_kernel<T, N, E, W, COLS, OP, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = W * (N / E);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    LineArgs a;
    if (COLS) a = LineArgs{nx, 1, nx, nx * ny, (nx + W - 1) / W, out2};
    else a = LineArgs{ny, nx, 1, nx * ny, (ny + W - 1) / W, out2};
    const long grid = batch * a.groups;
    const double fields = OP == LN_MID ? 3.0 : 2.0;
    const double bytes = fields * (double)nx * ny * batch * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((const C *)in, (C *)out, a, (const C *)tw, tab, PeerOut{}); },
           name, bytes, occ, grid);
}

template <typename T, int N, int E, int W, int MINB>
static void wave_var(void *U, void *V, long nx, long ny, const void *tw, const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s wave E=%d W=%d minb=%d", tag, E, W, MINB);
    if (g_filter && !strstr(name, g_filter)) return;
    using L = WaveLineSmem<C, N, E, W>;
    auto k = wave_line_kernel<T, N, E, W, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = W * (N / E);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    LineArgs a{nx, 1, nx, nx * ny, (nx + W - 1) / W, nullptr};
    const long grid = a.groups;
    const double bytes = 4.0 * nx * ny * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((C *)U, (C *)V, a, (const C *)tw, tab); }, name, bytes,
           occ, grid);
}

// ---- rr_kernel variant
template <typename T, int N, int W, bool COLS, int OP, int MINB>
static void rr_var(const void *in, void *out, void *out2, long nx, long ny, long batch, const void *tw,
                   const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s RR W=%d minb=%d", tag, W, MINB);
    if (g_filter && !strstr(name, g_filter)) return;
    using L = RRSmem<C, N, W, COLS>;
    auto k = rr_kernel<T, N, W, COLS, OP, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = W * (N / 16);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    LineArgs a;
    if (COLS) a = LineArgs{nx, 1, nx, nx * ny, (nx + W - 1) / W, out2};
    else a = LineArgs{ny, nx, 1, nx * ny, (ny + W - 1) / W, out2};
    const long ntiles = batch * a.groups;
    long grid = (long)occ * 148;
    if (grid > ntiles) grid = ntiles;
    const double fields = OP == LN_MID ? 3.0 : 2.0;
    const double bytes = fields * (double)nx * ny * batch * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((const C *)in, (C *)out, a, ntiles, (const C *)tw, tab); },
           name, bytes, occ, grid);
}

// ---- tpipe_kernel variant (transposed spectrum side)
template <typename T, int N, int W, int OP, int NBUF, bool TWREG>
static void tpipe_var(const void *in, void *out, void *out2, long nx, long ny, long batch, const void *tw, const char *tag)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s TPIPE op=%d W=%d nbuf=%d", tag, OP, W, NBUF);
    if (g_filter && !strstr(name, g_filter)) return;
    using L = PipeSmem<C, N, W, true, NBUF>;
    auto k = tpipe_kernel<T, N, W, OP, NBUF, TWREG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = W * Shape<N>::TPT;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    TPipeArgs a{ny, nx, ny, nx * ny, nx * ny, 0, (ny + W - 1) / W, out2};
    a.ntiles = batch * a.groups;
    long grid = (long)occ * 148;
    if (grid > a.ntiles) grid = a.ntiles;
    const double fields = OP == TP_MID_T ? 3.0 : 2.0;
    const double bytes = fields * (double)nx * ny * batch * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((const C *)in, (C *)out, a, (const C *)tw); }, name,
           bytes, occ, grid);
}

// ---- pipe_kernel reference (current library configuration)
template <typename T, int N, int W, bool COLS, int OP, int NBUF, bool TWREG, bool BULK = false, int MINB = 1>
static void pipe_ref(const void *in, void *out, void *out2, long nx, long ny, long batch, const void *tw,
                     const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s PIPE%s W=%d nbuf=%d minb=%d twreg=%d", tag, BULK ? " BULK" : "", W, NBUF, MINB, (int)TWREG);
    if (g_filter && !strstr(name, g_filter)) return;
    using L0 = PipeSmem<C, N, W, COLS, NBUF>;
    constexpr size_t SMB = L0::BYTES + (BULK ? 8 * NBUF * W : 0);
    auto k = pipe_kernel<T, N, W, COLS, OP, NBUF, MINB, TWREG, BULK>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMB);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = W * Shape<N>::TPT;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, SMB);
    PipeArgs a;
    if (COLS) a = PipeArgs{nx, 1, nx, nx * ny, 0, (nx + W - 1) / W, OP, out2};
    else a = PipeArgs{ny, nx, 1, nx * ny, 0, (ny + W - 1) / W, OP, out2};
    a.ntiles = batch * a.groups;
    long grid = (long)occ * 148;
    if (grid > a.ntiles) grid = a.ntiles;
    const double fields = OP == PIPE_MID ? 3.0 : 2.0;
    const double bytes = fields * (double)nx * ny * batch * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, SMB, g_stream>>>((const C *)in, (C *)out, a, (const C *)tw, tab, PeerOut{}); }, name,
           bytes, occ, grid);
}

int main(int argc, char **argv)
{
    if (argc > 1) g_filter = argv[1];
    if (argc > 2) g_reps = atoi(argv[2]);
    const size_t big = (size_t)1 << 30;   // 1 GiB per buffer
    void *A, *B, *Cb;
    cudaMalloc(&A, big); cudaMalloc(&B, big); cudaMalloc(&Cb, big);
    cudaMemset(A, 0, big); cudaMemset(B, 0, big); cudaMemset(Cb, 0, big);

    // ---------------- C2 shapes: 1024 x 1024 c128 (L2-resident), and 1024-long lines on 256 MiB
    {
        using D = double;
        OpTables<D> tab = make_tab<D>(1024, 1024);
        OpTables<D> tabw = make_tab<D>(16384, 1024);
        void *t16 = upload_tw<double2>(1024, 16), *t8 = upload_tw<double2>(1024, 8), *t4 = upload_tw<double2>(1024, 4);
        pipe_ref<D, 1024, 4, false, PIPE_MID, 2, true>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        line_var<D, 1024, 16, 2, false, LN_MID, 1>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        line_var<D, 1024, 16, 2, false, LN_MID, 2>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        line_var<D, 1024, 8, 2, false, LN_MID, 2>(A, B, Cb, 1024, 1024, 1, t8, tab, "c2 rowsMID");
        line_var<D, 1024, 8, 2, false, LN_MID, 3>(A, B, Cb, 1024, 1024, 1, t8, tab, "c2 rowsMID");
        line_var<D, 1024, 8, 1, false, LN_MID, 4>(A, B, Cb, 1024, 1024, 1, t8, tab, "c2 rowsMID");
        line_var<D, 1024, 8, 4, false, LN_MID, 1>(A, B, Cb, 1024, 1024, 1, t8, tab, "c2 rowsMID");
        line_var<D, 1024, 4, 1, false, LN_MID, 4>(A, B, Cb, 1024, 1024, 1, t4, tab, "c2 rowsMID");
        line_var<D, 1024, 16, 1, false, LN_MID, 7>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        line_var<D, 1024, 16, 1, false, LN_MID, 4>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        line_var<D, 1024, 8, 1, false, LN_MID, 7>(A, B, Cb, 1024, 1024, 1, t8, tab, "c2 rowsMID");
        line_var<D, 1024, 16, 1, true, LN_DIFFUSE, 7>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        line_var<D, 1024, 16, 1, true, LN_DIFFUSE, 4>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 1, true, LN_DIFFUSE, 7>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 16, 2, true, LN_DIFFUSE, 4>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 2, true, LN_DIFFUSE, 4>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 4, 1, false, LN_MID, 6>(A, B, Cb, 1024, 1024, 1, t4, tab, "c2 rowsMID");
        pipe_ref<D, 1024, 4, true, PIPE_DIFFUSE, 2, true>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        pipe_ref<D, 1024, 2, true, PIPE_DIFFUSE, 2, true>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        pipe_ref<D, 1024, 2, true, PIPE_DIFFUSE, 3, true>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        pipe_ref<D, 1024, 1, true, PIPE_DIFFUSE, 3, true>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        pipe_ref<D, 1024, 2, false, PIPE_MID, 2, true>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        tpipe_var<D, 1024, 4, TP_MID_T, 2, true>(A, B, Cb, 1024, 1024, 1, t16, "c2 T");
        tpipe_var<D, 1024, 2, TP_MID_T, 2, true>(A, B, Cb, 1024, 1024, 1, t16, "c2 T");
        tpipe_var<D, 1024, 2, TP_MID_T, 3, true>(A, B, Cb, 1024, 1024, 1, t16, "c2 T");
        tpipe_var<D, 1024, 4, TP_FWD_T, 2, true>(A, B, nullptr, 1024, 1024, 1, t16, "c2 T");
        tpipe_var<D, 1024, 4, TP_INV_T, 2, true>(A, B, nullptr, 1024, 1024, 1, t16, "c2 T");
        pipe_ref<D, 1024, 4, false, PIPE_DIFFUSE, 2, true>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 TrowsDIF");
        pipe_ref<D, 1024, 2, false, PIPE_DIFFUSE, 2, true>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 TrowsDIF");
        line_var<D, 1024, 16, 1, false, LN_DIFFUSE, 7>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 TrowsDIF");
        line_var<D, 1024, 16, 2, false, LN_DIFFUSE, 2>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 TrowsDIF");
        pipe_ref<D, 1024, 2, false, PIPE_MID, 3, true>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        pipe_ref<D, 1024, 1, false, PIPE_MID, 3, true>(A, B, Cb, 1024, 1024, 1, t16, tab, "c2 rowsMID");
        line_var<D, 1024, 16, 2, true, LN_DIFFUSE, 1>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        line_var<D, 1024, 16, 2, true, LN_DIFFUSE, 2>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        line_var<D, 1024, 16, 4, true, LN_DIFFUSE, 1>(B, B, nullptr, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 2, true, LN_DIFFUSE, 2>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 2, true, LN_DIFFUSE, 3>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 4, true, LN_DIFFUSE, 1>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 4, true, LN_DIFFUSE, 2>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 8, 8, true, LN_DIFFUSE, 1>(B, B, nullptr, 1024, 1024, 1, t8, tab, "c2 colsDIF");
        line_var<D, 1024, 4, 2, true, LN_DIFFUSE, 3>(B, B, nullptr, 1024, 1024, 1, t4, tab, "c2 colsDIF");
        line_var<D, 1024, 4, 4, true, LN_DIFFUSE, 2>(B, B, nullptr, 1024, 1024, 1, t4, tab, "c2 colsDIF");
        // HBM-resident: 16384 x 1024 (256 MiB)
        pipe_ref<D, 1024, 4, false, PIPE_MID, 2, true>(A, B, Cb, 1024, 16384, 1, t16, tab, "hbm1024 rowsMID");
        line_var<D, 1024, 8, 2, false, LN_MID, 2>(A, B, Cb, 1024, 16384, 1, t8, tab, "hbm1024 rowsMID");
        line_var<D, 1024, 8, 2, false, LN_MID, 3>(A, B, Cb, 1024, 16384, 1, t8, tab, "hbm1024 rowsMID");
        line_var<D, 1024, 16, 2, false, LN_MID, 2>(A, B, Cb, 1024, 16384, 1, t16, tab, "hbm1024 rowsMID");
        line_var<D, 1024, 4, 1, false, LN_MID, 6>(A, B, Cb, 1024, 16384, 1, t4, tab, "hbm1024 rowsMID");
        pipe_ref<D, 1024, 4, true, PIPE_DIFFUSE, 2, true>(B, B, nullptr, 16384, 1024, 1, t16, tabw, "hbm1024 colsDIF");
        line_var<D, 1024, 8, 4, true, LN_DIFFUSE, 2>(B, B, nullptr, 16384, 1024, 1, t8, tabw, "hbm1024 colsDIF");
        line_var<D, 1024, 8, 8, true, LN_DIFFUSE, 1>(B, B, nullptr, 16384, 1024, 1, t8, tabw, "hbm1024 colsDIF");
        line_var<D, 1024, 16, 4, true, LN_DIFFUSE, 1>(B, B, nullptr, 16384, 1024, 1, t16, tabw, "hbm1024 colsDIF");
        line_var<D, 1024, 16, 8, true, LN_DIFFUSE, 1>(B, B, nullptr, 16384, 1024, 1, t16, tabw, "hbm1024 colsDIF");
        line_var<D, 1024, 4, 4, true, LN_DIFFUSE, 2>(B, B, nullptr, 16384, 1024, 1, t4, tabw, "hbm1024 colsDIF");
        wave_var<D, 1024, 8, 4, 1>(A, B, 1024, 1024, t8, tab, "c2size");
        wave_var<D, 1024, 8, 2, 2>(A, B, 1024, 1024, t8, tab, "c2size");
        wave_var<D, 1024, 16, 4, 1>(A, B, 1024, 1024, t16, tab, "c2size");
    }
    // ---------------- C3 rows: 4096 x 4096 c128
    {
        using D = double;
        OpTables<D> tab = make_tab<D>(4096, 4096);
        void *t16 = upload_tw<double2>(4096, 16), *t8 = upload_tw<double2>(4096, 8);
        void *t16_2048 = upload_tw<double2>(2048, 16);
        OpTables<D> tab2048 = make_tab<D>(8192, 2048);
        pipe_ref<D, 4096, 1, false, PIPE_MID, 2, true>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        line_var<D, 4096, 16, 1, false, LN_MID, 1>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        line_var<D, 4096, 16, 1, false, LN_MID, 2>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        line_var<D, 4096, 16, 1, false, LN_MID, 3>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        {   // radix 32: one 128-thread CTA per row (round 2)
            void *t32 = upload_tw<double2>(4096, 32);
            line_var<D, 4096, 32, 1, false, LN_MID, 1>(A, B, Cb, 4096, 4096, 1, t32, tab, "c3 rowsMID");
            line_var<D, 4096, 32, 1, false, LN_MID, 2>(A, B, Cb, 4096, 4096, 1, t32, tab, "c3 rowsMID");
        }
        line_var<D, 4096, 8, 1, false, LN_MID, 1>(A, B, Cb, 4096, 4096, 1, t8, tab, "c3 rowsMID");
        line_var<D, 4096, 8, 1, false, LN_MID, 2>(A, B, Cb, 4096, 4096, 1, t8, tab, "c3 rowsMID");
        line_var<D, 4096, 8, 1, false, LN_MID, 3>(A, B, Cb, 4096, 4096, 1, t8, tab, "c3 rowsMID");
        rr_var<D, 4096, 2, false, LN_MID, 1>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        rr_var<D, 4096, 1, false, LN_MID, 2>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        rr_var<D, 4096, 1, false, LN_MID, 1>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        pipe_ref<D, 4096, 1, false, PIPE_FWD, 2, true>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        rr_var<D, 4096, 2, false, LN_FWD, 1>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        rr_var<D, 4096, 1, false, LN_FWD, 2>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        rr_var<D, 4096, 2, true, LN_POISSON, 1>(B, B, nullptr, 4096, 4096, 1, t16, tab, "c3 colsPOI");
        rr_var<D, 4096, 2, true, LN_FWD, 1>(B, B, nullptr, 4096, 4096, 1, t16, tab, "c3 colsFWD");
        rr_var<D, 2048, 4, true, LN_POISSON, 1>(B, B, nullptr, 8192, 2048, 1, t16_2048, tab2048, "c2048 colsPOI");
        rr_var<D, 2048, 2, true, LN_POISSON, 2>(B, B, nullptr, 8192, 2048, 1, t16_2048, tab2048, "c2048 colsPOI");
        pipe_ref<D, 4096, 1, false, PIPE_MID, 2, true, true>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        pipe_ref<D, 4096, 1, false, PIPE_FWD, 2, true, true>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        pipe_ref<D, 4096, 1, false, PIPE_MID, 1, false, true, 2>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        pipe_ref<D, 4096, 1, false, PIPE_MID, 2, false, true, 1>(A, B, Cb, 4096, 4096, 1, t16, tab, "c3 rowsMID");
        pipe_ref<D, 4096, 1, false, PIPE_FWD, 1, false, true, 2>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        pipe_ref<D, 2048, 2, false, PIPE_MID, 2, true, false>(A, B, Cb, 2048, 8192, 1, t16_2048, tab2048, "c2048 rowsMID");
        pipe_ref<D, 2048, 2, false, PIPE_MID, 2, true, true>(A, B, Cb, 2048, 8192, 1, t16_2048, tab2048, "c2048 rowsMID");
        // transposed-spectrum design for C3: W = 2 rows per tile -> 32-byte segments on the T side
        tpipe_var<D, 4096, 2, TP_MID_T, 1, false>(A, B, Cb, 4096, 4096, 1, t16, "c3 T");
        tpipe_var<D, 4096, 1, TP_MID_T, 2, false>(A, B, Cb, 4096, 4096, 1, t16, "c3 T");
        tpipe_var<D, 4096, 2, TP_FWD_T, 1, false>(A, B, nullptr, 4096, 4096, 1, t16, "c3 T");
        pipe_ref<D, 4096, 2, false, PIPE_DIFFUSE, 1, false>(B, B, nullptr, 4096, 4096, 1, t16, tab, "c3 TrowsDIF");
        pipe_ref<D, 4096, 1, false, PIPE_DIFFUSE, 2, false>(B, B, nullptr, 4096, 4096, 1, t16, tab, "c3 TrowsDIF");
        pipe_ref<D, 4096, 1, false, PIPE_DIFFUSE, 2, true>(B, B, nullptr, 4096, 4096, 1, t16, tab, "c3 TrowsDIF");
        line_var<D, 4096, 16, 1, false, LN_DIFFUSE, 2>(B, B, nullptr, 4096, 4096, 1, t16, tab, "c3 TrowsDIF");
        line_var<D, 4096, 16, 1, false, LN_FWD, 2>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        line_var<D, 4096, 16, 1, false, LN_FWD, 3>(A, B, nullptr, 4096, 4096, 1, t16, tab, "c3 rowsFWD");
        line_var<D, 4096, 8, 1, false, LN_FWD, 2>(A, B, nullptr, 4096, 4096, 1, t8, tab, "c3 rowsFWD");
        line_var<D, 4096, 8, 1, false, LN_FWD, 3>(A, B, nullptr, 4096, 4096, 1, t8, tab, "c3 rowsFWD");
    }
    // ---------------- C4: 256 x 512 x 512 c64
    {
        using F = float;
        OpTables<F> tab = make_tab<F>(512, 512);
        void *t16 = upload_tw<float2>(512, 16), *t8 = upload_tw<float2>(512, 8);
        pipe_ref<F, 512, 8, false, PIPE_FWD, 2, true>(A, B, nullptr, 512, 512, 256, t16, tab, "c4 rowsFWD");
        line_var<F, 512, 16, 4, false, LN_FWD, 2>(A, B, nullptr, 512, 512, 256, t16, tab, "c4 rowsFWD");
        line_var<F, 512, 16, 8, false, LN_FWD, 1>(A, B, nullptr, 512, 512, 256, t16, tab, "c4 rowsFWD");
        line_var<F, 512, 16, 8, false, LN_FWD, 2>(A, B, nullptr, 512, 512, 256, t16, tab, "c4 rowsFWD");
        line_var<F, 512, 8, 4, false, LN_FWD, 2>(A, B, nullptr, 512, 512, 256, t8, tab, "c4 rowsFWD");
        line_var<F, 512, 8, 4, false, LN_FWD, 3>(A, B, nullptr, 512, 512, 256, t8, tab, "c4 rowsFWD");
        line_var<F, 512, 8, 8, false, LN_FWD, 2>(A, B, nullptr, 512, 512, 256, t8, tab, "c4 rowsFWD");
        pipe_ref<F, 512, 16, true, PIPE_POISSON, 2, false>(B, B, nullptr, 512, 512, 256, t16, tab, "c4 colsPOI");
        line_var<F, 512, 16, 16, true, LN_POISSON, 1>(B, B, nullptr, 512, 512, 256, t16, tab, "c4 colsPOI");
        line_var<F, 512, 16, 16, true, LN_POISSON, 2>(B, B, nullptr, 512, 512, 256, t16, tab, "c4 colsPOI");
        line_var<F, 512, 16, 8, true, LN_POISSON, 2>(B, B, nullptr, 512, 512, 256, t16, tab, "c4 colsPOI");
        line_var<F, 512, 16, 8, true, LN_POISSON, 3>(B, B, nullptr, 512, 512, 256, t16, tab, "c4 colsPOI");
        line_var<F, 512, 8, 16, true, LN_POISSON, 1>(B, B, nullptr, 512, 512, 256, t8, tab, "c4 colsPOI");
        line_var<F, 512, 8, 16, true, LN_POISSON, 2>(B, B, nullptr, 512, 512, 256, t8, tab, "c4 colsPOI");
        line_var<F, 512, 8, 8, true, LN_POISSON, 2>(B, B, nullptr, 512, 512, 256, t8, tab, "c4 colsPOI");
        line_var<F, 512, 8, 8, true, LN_POISSON, 3>(B, B, nullptr, 512, 512, 256, t8, tab, "c4 colsPOI");
        line_var<F, 512, 8, 4, true, LN_POISSON, 4>(B, B, nullptr, 512, 512, 256, t8, tab, "c4 colsPOI");
    }
    printf("done\n");
    return 0;
}
