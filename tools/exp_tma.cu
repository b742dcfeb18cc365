// Experiment harness: TMA column pass (tmacols.cuh) vs pipe_kernel columns on the
// C2 (1024^2 c128), C4 (256 x 512^2 c64) and an HBM-resident 1024-row shape.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I include tools/exp_tma.cu -o tools/exp_tma -lcuda
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_2412_12308_b200/csrc/line.cuh"
#include "../paper_2412_12308_b200/csrc/pipe.cuh"
#include "../paper_2412_12308_b200/csrc/tmacols.cuh"
#include <cudaTypedefs.h>
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

template <typename T, int N, int W, int OP, int MINB>
static void tma_var(void *buf, long nx, long ny, long batch, const void *tw, const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    using L = TmaColSmem<C, N, W>;
    char name[160];
    snprintf(name, sizeof name, "%s TMA W=%d minb=%d", tag, W, MINB);
    if (g_filter && !strstr(name, g_filter)) return;
    auto k = tma_cols_kernel<T, N, W, OP, MINB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    const int threads = W * Shape<N>::TPT;
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

template <typename T, int N, int W, int OP, int NBUF, bool TWREG>
static void pipe_cols(void *buf, long nx, long ny, long batch, const void *tw, const OpTables<T> &tab, const char *tag,
                      bool time = true)
{
    using C = typename cplx_t<T>::type;
    char name[160];
    snprintf(name, sizeof name, "%s PIPE W=%d nbuf=%d", tag, W, NBUF);
    if (time && g_filter && !strstr(name, g_filter)) return;
    using L = PipeSmem<C, N, W, true, NBUF>;
    auto k = pipe_kernel<T, N, W, true, OP, NBUF, 1, TWREG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    const int threads = W * Shape<N>::TPT;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, L::BYTES);
    PipeArgs a{nx, 1, nx, nx * ny, 0, (nx + W - 1) / W, OP, nullptr};
    a.ntiles = batch * a.groups;
    long grid = (long)occ * 148;
    if (grid > a.ntiles) grid = a.ntiles;
    const double bytes = 2.0 * nx * ny * batch * sizeof(C);
    auto go = [&] { k<<<(unsigned)grid, threads, L::BYTES, g_stream>>>((const C *)buf, (C *)buf, a, (const C *)tw, tab); };
    if (time) timeit(go, name, bytes, occ, grid);
    else go();
}

// correctness: one application of each pass on identical random data, max |diff|
template <typename T, int N, int W, int OP, int NBUF, bool TWREG>
static void check(long nx, long ny, long batch, const void *tw, const OpTables<T> &tab, const char *tag)
{
    using C = typename cplx_t<T>::type;
    using L = TmaColSmem<C, N, W>;
    const size_t n = (size_t)nx * ny * batch;
    std::vector<C> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = C{(T)((i * 2654435761u) % 1000) / 1000, (T)((i * 40503u) % 997) / 997};
    C *A, *B;
    cudaMalloc(&A, n * sizeof(C)); cudaMalloc(&B, n * sizeof(C));
    cudaMemcpy(A, h.data(), n * sizeof(C), cudaMemcpyHostToDevice);
    cudaMemcpy(B, h.data(), n * sizeof(C), cudaMemcpyHostToDevice);
    pipe_cols<T, N, W, OP, NBUF, TWREG>(A, nx, ny, batch, tw, tab, tag, false);
    auto k = tma_cols_kernel<T, N, W, OP, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES);
    CUtensorMap m = tmap<T>(B, nx, ny, batch, nx * ny, W, L::BOXR);
    TmaColArgs a{nx, (nx + W - 1) / W, 0};
    a.ntiles = batch * a.groups;
    k<<<148, W * Shape<N>::TPT, L::BYTES>>>(m, m, a, (const C *)tw, tab);
    cudaError_t err = cudaDeviceSynchronize();
    std::vector<C> ha(n), hb(n);
    cudaMemcpy(ha.data(), A, n * sizeof(C), cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), B, n * sizeof(C), cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (size_t i = 0; i < n; ++i) {
        md = fmax(md, fabs((double)ha[i].x - hb[i].x) + fabs((double)ha[i].y - hb[i].y));
        mx = fmax(mx, fabs((double)ha[i].x) + fabs((double)ha[i].y));
    }
    printf("%s check: max|pipe - tma| = %.3e (max |x| %.3e) %s\n", tag, md, mx, err ? cudaGetErrorString(err) : "ok");
    cudaFree(A); cudaFree(B);
}

int main(int argc, char **argv)
{
    if (argc > 1 && argv[1][0]) g_filter = argv[1];
    if (argc > 2) g_reps = atoi(argv[2]);
    void *A;
    cudaMalloc(&A, (size_t)1 << 30);
    cudaMemset(A, 0, (size_t)1 << 30);
    {
        using D = double;
        OpTables<D> tab = make_tab<D>(1024, 1024);
        void *t16 = upload_tw<double2>(1024, 16);
        check<D, 1024, 4, PIPE_DIFFUSE, 2, true>(1024, 1024, 1, t16, tab, "c2 colsDIF");
        check<D, 1024, 4, PIPE_POISSON, 2, true>(1024, 1024, 1, t16, tab, "c2 colsPOI");
        check<D, 1024, 4, PIPE_FWD, 2, true>(1024, 1024, 1, t16, tab, "c2 colsFWD");
        pipe_cols<D, 1024, 4, PIPE_DIFFUSE, 2, true>(A, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        pipe_cols<D, 1024, 2, PIPE_DIFFUSE, 2, true>(A, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        tma_var<D, 1024, 4, PIPE_DIFFUSE, 1>(A, 1024, 1024, 1, t16, tab, "c2 colsDIF");
        OpTables<D> tabw = make_tab<D>(16384, 1024);
        pipe_cols<D, 1024, 4, PIPE_DIFFUSE, 2, true>(A, 16384, 1024, 1, t16, tabw, "hbm1024 colsDIF");
        tma_var<D, 1024, 4, PIPE_DIFFUSE, 1>(A, 16384, 1024, 1, t16, tabw, "hbm1024 colsDIF");
        OpTables<D> tab512 = make_tab<D>(512, 512);
        void *t16_512 = upload_tw<double2>(512, 16);
        check<D, 512, 4, PIPE_POISSON, 2, true>(512, 512, 4, t16_512, tab512, "c128 512x512x4 colsPOI");
        OpTables<D> tab2k = make_tab<D>(2048, 2048);
        void *t16_2k = upload_tw<double2>(2048, 16);
        pipe_cols<D, 2048, 4, PIPE_DIFFUSE, 1, true>(A, 2048, 2048, 1, t16_2k, tab2k, "c2048 colsDIF");
        tma_var<D, 2048, 4, PIPE_DIFFUSE, 1>(A, 2048, 2048, 1, t16_2k, tab2k, "c2048 colsDIF");
    }
    {
        using F = float;
        OpTables<F> tab = make_tab<F>(512, 512);
        void *t16 = upload_tw<float2>(512, 16);
        check<F, 512, 8, PIPE_POISSON, 2, false>(512, 512, 256, t16, tab, "c4 colsPOI");
        pipe_cols<F, 512, 16, PIPE_POISSON, 2, false>(A, 512, 512, 256, t16, tab, "c4 colsPOI");
        pipe_cols<F, 512, 8, PIPE_POISSON, 2, false>(A, 512, 512, 256, t16, tab, "c4 colsPOI");
        tma_var<F, 512, 8, PIPE_POISSON, 1>(A, 512, 512, 256, t16, tab, "c4 colsPOI");
        tma_var<F, 512, 8, PIPE_POISSON, 2>(A, 512, 512, 256, t16, tab, "c4 colsPOI");
    }
    printf("done\n");
    return 0;
}
