// dispatch.cuh -- launch configurations and length dispatch of the pass kernels.
// Included by the per-dtype instantiation units (passes_c128.cu, passes_c64.cu).
#pragma once
#include <atomic>
#include "kernels.cuh"

namespace fftpde {

#define FFTPDE_LEN_CASES(X) \
    X(1) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

// Opt a kernel into > 48 KiB dynamic shared memory once per device.
template <typename K> struct SmemOptIn {
    std::atomic<uint64_t> done{0};
    cudaError_t operator()(K kernel, size_t bytes)
    {
        if (bytes <= 48 * 1024) return cudaSuccess;
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        const uint64_t bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_relaxed) & bit) return cudaSuccess;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e == cudaSuccess) done.fetch_or(bit);
        return e;
    }
};

// ---- launch shapes ---------------------------------------------------------
// rows: ROWS rows per CTA so a CTA has >= 256 threads
template <int N> struct RowCfg {
    static constexpr int TPT = Shape<N>::TPT;
    static constexpr int ROWS = TPT >= 256 ? 1 : 256 / TPT;
};
// columns: W adjacent columns per CTA (c128: 256 threads; c64: up to 512 threads
// so that a row segment is >= 64 B)
template <typename T, int N> struct ColCfg {
    static constexpr int TPT = Shape<N>::TPT;
    static constexpr int TARGET = sizeof(T) == 8 ? 256 : 512;
    static constexpr int W = TPT >= TARGET ? 1 : TARGET / TPT;
};

template <typename T, int N>
cudaError_t rows_n(const void *in, void *out, int64_t ny, int64_t stride, int64_t batch,
                   int conj, const void *tw, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    constexpr int ROWS = RowCfg<N>::ROWS;
    constexpr int THREADS = ROWS * Shape<N>::TPT;
    const size_t smem = (size_t)ROWS * Shape<N>::PADDED * sizeof(C);
    auto k = row_fft_kernel<T, N, ROWS>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, smem);
    if (e != cudaSuccess) return e;
    const int64_t total = batch * ny;
    const int64_t grid = (total + ROWS - 1) / ROWS;
    k<<<(unsigned)grid, THREADS, smem, st>>>((const C *)in, (C *)out, ny, stride, total, conj,
                                             (const C *)tw);
    return cudaGetLastError();
}

template <typename T, int N>
cudaError_t cols_n(const void *in, void *out, int64_t nx, int64_t stride, int64_t batch, int op,
                   const void *tw, const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    constexpr int W = ColCfg<T, N>::W;
    constexpr int THREADS = W * Shape<N>::TPT;
    const size_t smem = ColSmem<C, N, W>::BYTES;
    auto k = col_fused_kernel<T, N, W>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((nx + W - 1) / W), (unsigned)batch);
    k<<<grid, THREADS, smem, st>>>((const C *)in, (C *)out, nx, stride, op, (const C *)tw, tab);
    return cudaGetLastError();
}

template <typename T, int N>
cudaError_t wave_cols_n(void *U, void *V, int64_t nx, int64_t stride, int64_t batch,
                        const void *tw, const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    constexpr int W = Shape<N>::TPT >= 256 ? 1 : 256 / Shape<N>::TPT;
    constexpr int THREADS = W * Shape<N>::TPT;
    const size_t smem = WaveSmem<C, N, W>::BYTES;
    auto k = col_wave_kernel<T, N, W>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((nx + W - 1) / W), (unsigned)batch);
    k<<<grid, THREADS, smem, st>>>((C *)U, (C *)V, nx, stride, (const C *)tw, tab);
    return cudaGetLastError();
}

template <typename T, int N>
cudaError_t small_n(const void *in, void *out, int64_t stride, int64_t batch, int op,
                    const void *twx, const void *twy, const OpTables<T> &tab, cudaStream_t st)
{
    using C = typename cplx_t<T>::type;
    using L = SmallLayout<C, N, N>;
    auto k = small_solve_kernel<T, N, N>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, L::BYTES);
    if (e != cudaSuccess) return e;
    k<<<(unsigned)batch, L::THREADS, L::BYTES, st>>>((const C *)in, (C *)out, stride, op,
                                                      (const C *)twx, (const C *)twy, tab);
    return cudaGetLastError();
}

// ---- length dispatch -------------------------------------------------------
template <typename T>
cudaError_t launch_rows(int64_t n, const void *in, void *out, int64_t ny, int64_t stride,
                        int64_t batch, int conj, const void *tw, cudaStream_t st)
{
    switch (n) {
#define X(L) case L: return rows_n<T, L>(in, out, ny, stride, batch, conj, tw, st);
        FFTPDE_LEN_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

template <typename T>
cudaError_t launch_cols(int64_t ny, const void *in, void *out, int64_t nx, int64_t stride,
                        int64_t batch, int op, const void *tw, const OpTables<T> &tab,
                        cudaStream_t st)
{
    switch (ny) {
#define X(L) case L: return cols_n<T, L>(in, out, nx, stride, batch, op, tw, tab, st);
        FFTPDE_LEN_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

template <typename T>
cudaError_t launch_wave_cols(int64_t ny, void *U, void *V, int64_t nx, int64_t stride,
                             int64_t batch, const void *tw, const OpTables<T> &tab,
                             cudaStream_t st)
{
    switch (ny) {
#define X(L) case L: return wave_cols_n<T, L>(U, V, nx, stride, batch, tw, tab, st);
        FFTPDE_LEN_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
    }
}

template <typename T> bool small_supported(int64_t nx, int64_t ny)
{
    return nx == ny && (nx == 16 || nx == 32 || nx == 64);
}

template <typename T>
cudaError_t launch_small(int64_t nx, int64_t ny, const void *in, void *out, int64_t stride,
                         int64_t batch, int op, const void *twx, const void *twy,
                         const OpTables<T> &tab, cudaStream_t st)
{
    if (nx != ny) return cudaErrorInvalidValue;
    switch (nx) {
    case 16: return small_n<T, 16>(in, out, stride, batch, op, twx, twy, tab, st);
    case 32: return small_n<T, 32>(in, out, stride, batch, op, twx, twy, tab, st);
    case 64: return small_n<T, 64>(in, out, stride, batch, op, twx, twy, tab, st);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace fftpde
