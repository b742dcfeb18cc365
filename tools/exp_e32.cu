// Experiment harness: radix-32 (one warp per 1024-point line) line passes vs the
// radix-16 passes on the C2 shape (1024^2 c128).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I include tools/exp_e32.cu -o tools/exp_e32
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_2412_12308_b200/csrc/line.cuh"
#include "../paper_2412_12308_b200/csrc/pipe.cuh"
#include "experimental/rr.cuh"
#include "../paper_2412_12308_b200/csrc/tmacols.cuh"
#include <cudaTypedefs.h>
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
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((const C *)in, (C *)out, a, (const C *)tw, tab); },
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

// ---- pipe_kernel reference (current library configuration)
template <typename T, int N, int W, bool COLS, int OP, int NBUF, bool TWREG>
static void pipe_ref(const void *in, void *out, void *out2, long nx, long ny, long batch, const void *tw,
                     const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s PIPE W=%d nbuf=%d", tag, W, NBUF);
    if (g_filter && !strstr(name, g_filter)) return;
    using L = PipeSmem<C, N, W, COLS, NBUF>;
    auto k = pipe_kernel<T, N, W, COLS, OP, NBUF, 1, TWREG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = W * Shape<N>::TPT;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    PipeArgs a;
    if (COLS) a = PipeArgs{nx, 1, nx, nx * ny, 0, (nx + W - 1) / W, OP, out2};
    else a = PipeArgs{ny, nx, 1, nx * ny, 0, (ny + W - 1) / W, OP, out2};
    a.ntiles = batch * a.groups;
    long grid = (long)occ * 148;
    if (grid > a.ntiles) grid = a.ntiles;
    const double fields = OP == PIPE_MID ? 3.0 : 2.0;
    const double bytes = fields * (double)nx * ny * batch * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((const C *)in, (C *)out, a, (const C *)tw, tab); }, name,
           bytes, occ, grid);
}


template <typename T, int N, int E, int W, bool COLS, int OP, int MINB>
static void run_line(const void *in, void *out, void *out2, long nx, long ny, const void *tw, const OpTables<T> &tab)
{
    using C = typename cplx_t<T>::type;
    using L = LineSmem<C, N, E, W, COLS>;
    auto k = line_kernel<T, N, E, W, COLS, OP, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    LineArgs a{COLS ? nx : ny, COLS ? 1 : nx, COLS ? nx : 1, nx * ny, ((COLS ? nx : ny) + W - 1) / W, out2};
    k<<<(unsigned)a.groups, W * (N / E), L::BYTES>>>((const C *)in, (C *)out, a, (const C *)tw, tab);
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

template <typename T> static CUtensorMap tmap(void *p, long nx, long ny, long batch, long stride, int W, int boxr)
{
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&g_encode, cudaEnableDefault, &q);
    }
    CUtensorMap m;
    const size_t esz = 2 * sizeof(T);
    cuuint64_t dims[3] = {(cuuint64_t)(2 * nx), (cuuint64_t)ny, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)(nx * esz), (cuuint64_t)(stride * esz)};
    cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)boxr, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(&m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p,
                          dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

template <typename T, int N, int W, int OP, int MINB, int EX = 16>
static void tma_var(void *buf, long nx, long ny, long batch, const void *tw, const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    using L = TmaColSmem<C, N, W, EX>;
    char name[160];
    snprintf(name, sizeof name, "%s TMA E=%d W=%d minb=%d", tag, EX, W, MINB);
    if (g_filter && !strstr(name, g_filter)) return;
    auto k = tma_cols_kernel<T, N, W, OP, MINB, EX>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    const int threads = W * Shape<N, EX>::TPT;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    CUtensorMap m = tmap<T>(buf, nx, ny, batch, nx * ny, W, L::BOXR);
    TmaColArgs a{nx, (nx + W - 1) / W, 0};
    a.ntiles = batch * a.groups;
    long grid = (long)occ * 148;
    if (grid > a.ntiles) grid = a.ntiles;
    const double bytes = 2.0 * nx * ny * batch * sizeof(C);
    timeit([&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>(m, m, a, (const C *)tw, tab); }, name, bytes, occ,
           grid);
}


static double maxdiff(const double2 *A, const double2 *B, size_t n)
{
    std::vector<double2> a(n), b(n);
    cudaMemcpy(a.data(), A, n * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), B, n * 16, cudaMemcpyDeviceToHost);
    double m = 0, s = 0;
    for (size_t i = 0; i < n; ++i) {
        m = fmax(m, fabs(a[i].x - b[i].x) + fabs(a[i].y - b[i].y));
        s = fmax(s, fabs(b[i].x) + fabs(b[i].y));
    }
    return m / s;
}

int main(int argc, char **argv)
{
    if (argc > 1 && argv[1][0]) g_filter = argv[1];
    if (argc > 2) g_reps = atoi(argv[2]);
    using D = double;
    const long n = 1024;
    const size_t cnt = (size_t)n * n;
    double2 *X, *Y, *Z, *P;
    cudaMalloc(&X, cnt * 16); cudaMalloc(&Y, cnt * 16); cudaMalloc(&Z, cnt * 16); cudaMalloc(&P, cnt * 16);
    std::vector<double2> h(cnt);
    for (size_t i = 0; i < cnt; ++i) h[i] = {sin(0.37 * i) + 0.1 * cos(1.3 * i * i), cos(0.11 * i)};
    cudaMemcpy(X, h.data(), cnt * 16, cudaMemcpyHostToDevice);
    OpTables<D> tab = make_tab<D>(n, n);
    void *t16 = upload_tw<double2>(n, 16), *t32 = upload_tw<double2>(n, 32);
    // correctness: E=32 vs E=16 (same definition), forward rows, MID rows, columns with the operator
    run_line<D, 1024, 16, 1, false, LN_FWD, 1>(X, Y, nullptr, n, n, t16, tab);
    run_line<D, 1024, 32, 1, false, LN_FWD, 1>(X, Z, nullptr, n, n, t32, tab);
    cudaDeviceSynchronize();
    printf("rows FWD  E32 vs E16 rel max diff %.3e %s\n", maxdiff(Z, Y, cnt), cudaGetErrorString(cudaGetLastError()));
    run_line<D, 1024, 16, 1, false, LN_MID, 1>(X, Y, P, n, n, t16, tab);
    run_line<D, 1024, 32, 1, false, LN_MID, 1>(X, Z, P, n, n, t32, tab);
    cudaDeviceSynchronize();
    printf("rows MID  E32 vs E16 rel max diff %.3e\n", maxdiff(Z, Y, cnt));
    cudaMemcpy(Y, h.data(), cnt * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(Z, h.data(), cnt * 16, cudaMemcpyHostToDevice);
    run_line<D, 1024, 16, 4, true, LN_DIFFUSE, 1>(Y, Y, nullptr, n, n, t16, tab);
    run_line<D, 1024, 32, 4, true, LN_DIFFUSE, 1>(Z, Z, nullptr, n, n, t32, tab);
    cudaDeviceSynchronize();
    printf("cols DIF  E32 vs E16 rel max diff %.3e %s\n", maxdiff(Z, Y, cnt), cudaGetErrorString(cudaGetLastError()));
    // timing (graph-timed)
    pipe_ref<D, 1024, 4, false, PIPE_MID, 2, true>(X, Y, P, n, n, 1, t16, tab, "c2 rowsMID");
    line_var<D, 1024, 16, 1, false, LN_MID, 7>(X, Y, P, n, n, 1, t16, tab, "c2 rowsMID");
    line_var<D, 1024, 32, 1, false, LN_MID, 8>(X, Y, P, n, n, 1, t32, tab, "c2 rowsMID");
    line_var<D, 1024, 32, 1, false, LN_MID, 4>(X, Y, P, n, n, 1, t32, tab, "c2 rowsMID");
    line_var<D, 1024, 32, 2, false, LN_MID, 4>(X, Y, P, n, n, 1, t32, tab, "c2 rowsMID");
    line_var<D, 1024, 32, 4, false, LN_MID, 2>(X, Y, P, n, n, 1, t32, tab, "c2 rowsMID");
    line_var<D, 1024, 32, 8, false, LN_MID, 1>(X, Y, P, n, n, 1, t32, tab, "c2 rowsMID");
    line_var<D, 1024, 32, 4, true, LN_DIFFUSE, 2>(Y, Y, nullptr, n, n, 1, t32, tab, "c2 colsDIF");
    line_var<D, 1024, 32, 8, true, LN_DIFFUSE, 1>(Y, Y, nullptr, n, n, 1, t32, tab, "c2 colsDIF");
    line_var<D, 1024, 32, 1, false, LN_DIFFUSE, 4>(Y, Y, nullptr, n, n, 1, t32, tab, "c2 rowsDIF");
    line_var<D, 1024, 32, 2, false, LN_DIFFUSE, 4>(Y, Y, nullptr, n, n, 1, t32, tab, "c2 rowsDIF");
    line_var<D, 1024, 32, 2, true, LN_DIFFUSE, 4>(Y, Y, nullptr, n, n, 1, t32, tab, "c2 colsDIF");
    line_var<D, 1024, 32, 1, false, LN_DIFFUSE, 8>(Y, Y, nullptr, n, n, 1, t32, tab, "c2 TrowsDIF");
    line_var<D, 1024, 16, 1, false, LN_DIFFUSE, 7>(Y, Y, nullptr, n, n, 1, t16, tab, "c2 TrowsDIF");
    {   // TMA columns, radix 16 vs 32 (+ correctness of the radix-32 TMA pass vs the radix-16 line pass)
        cudaMemcpy(Y, h.data(), cnt * 16, cudaMemcpyHostToDevice);
        cudaMemcpy(Z, h.data(), cnt * 16, cudaMemcpyHostToDevice);
        run_line<D, 1024, 16, 4, true, LN_DIFFUSE, 1>(Y, Y, nullptr, n, n, t16, tab);
        using L = TmaColSmem<double2, 1024, 4, 32>;
        auto k = tma_cols_kernel<D, 1024, 4, PIPE_DIFFUSE, 1, 32>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
        CUtensorMap m = tmap<D>(Z, n, n, 1, n * n, 4, L::BOXR);
        TmaColArgs a{n, n / 4, n / 4};
        k<<<148, 4 * 32, L::BYTES>>>(m, m, a, (const double2 *)t32, tab);
        cudaDeviceSynchronize();
        printf("cols DIF TMA E32 vs line E16 rel max diff %.3e %s\n", maxdiff(Z, Y, cnt), cudaGetErrorString(cudaGetLastError()));
        tma_var<D, 1024, 4, PIPE_DIFFUSE, 1, 16>(Y, n, n, 1, t16, tab, "c2 colsDIF");
        tma_var<D, 1024, 4, PIPE_DIFFUSE, 1, 32>(Y, n, n, 1, t32, tab, "c2 colsDIF");
        tma_var<D, 1024, 4, PIPE_DIFFUSE, 2, 32>(Y, n, n, 1, t32, tab, "c2 colsDIF");
    }
    {   // C3 rows (4096 c128, 256 MiB per field)
        OpTables<D> tab4 = make_tab<D>(4096, 4096);
        void *t16_4 = upload_tw<double2>(4096, 16), *t32_4 = upload_tw<double2>(4096, 32);
        double2 *A4, *B4, *C4;
        cudaMalloc(&A4, (size_t)4096 * 4096 * 16); cudaMalloc(&B4, (size_t)4096 * 4096 * 16); cudaMalloc(&C4, (size_t)4096 * 4096 * 16);
        cudaMemset(A4, 0, (size_t)4096 * 4096 * 16);
        pipe_ref<D, 4096, 1, false, PIPE_MID, 2, true>(A4, B4, C4, 4096, 4096, 1, t16_4, tab4, "c3 rowsMID");
        line_var<D, 4096, 32, 1, false, LN_MID, 1>(A4, B4, C4, 4096, 4096, 1, t32_4, tab4, "c3 rowsMID");
        line_var<D, 4096, 32, 1, false, LN_MID, 2>(A4, B4, C4, 4096, 4096, 1, t32_4, tab4, "c3 rowsMID");
        pipe_ref<D, 4096, 1, false, PIPE_FWD, 2, true>(A4, B4, nullptr, 4096, 4096, 1, t16_4, tab4, "c3 rowsFWD");
        line_var<D, 4096, 32, 1, false, LN_FWD, 2>(A4, B4, nullptr, 4096, 4096, 1, t32_4, tab4, "c3 rowsFWD");
        cudaFree(A4); cudaFree(B4); cudaFree(C4);
    }
    {   // C4 (256 x 512^2 c64)
        using F = float;
        OpTables<F> tab5 = make_tab<F>(512, 512);
        void *f16 = upload_tw<float2>(512, 16), *f8 = upload_tw<float2>(512, 8), *f32 = upload_tw<float2>(512, 32);
        float2 *A5, *B5;
        cudaMalloc(&A5, (size_t)256 * 512 * 512 * 8); cudaMalloc(&B5, (size_t)256 * 512 * 512 * 8);
        cudaMemset(A5, 0, (size_t)256 * 512 * 512 * 8);
        line_var<F, 512, 16, 4, false, LN_FWD, 2>(A5, B5, nullptr, 512, 512, 256, f16, tab5, "c4 rowsFWD");
        line_var<F, 512, 32, 4, false, LN_FWD, 2>(A5, B5, nullptr, 512, 512, 256, f32, tab5, "c4 rowsFWD");
        line_var<F, 512, 32, 8, false, LN_FWD, 2>(A5, B5, nullptr, 512, 512, 256, f32, tab5, "c4 rowsFWD");
        line_var<F, 512, 32, 8, false, LN_FWD, 4>(A5, B5, nullptr, 512, 512, 256, f32, tab5, "c4 rowsFWD");
        line_var<F, 512, 8, 8, true, LN_POISSON, 3>(B5, B5, nullptr, 512, 512, 256, f8, tab5, "c4 colsPOI");
        line_var<F, 512, 32, 8, true, LN_POISSON, 2>(B5, B5, nullptr, 512, 512, 256, f32, tab5, "c4 colsPOI");
        line_var<F, 512, 32, 8, true, LN_POISSON, 4>(B5, B5, nullptr, 512, 512, 256, f32, tab5, "c4 colsPOI");
        line_var<F, 512, 32, 16, true, LN_POISSON, 2>(B5, B5, nullptr, 512, 512, 256, f32, tab5, "c4 colsPOI");
        tma_var<F, 512, 8, PIPE_POISSON, 2, 32>(B5, 512, 512, 256, f32, tab5, "c4 colsPOI");
        tma_var<F, 512, 8, PIPE_POISSON, 3, 32>(B5, 512, 512, 256, f32, tab5, "c4 colsPOI");
    }
    printf("done\n");
    return 0;
}
