// wavet.cu -- launchers of the transposed-spectrum wave passes (wavet.cuh).
#include "dispatch.cuh"
#include "wavet.cuh"

namespace fftpde {

bool wave_t_supported(int64_t nx, int64_t ny)
{
    const bool ok = (nx == 2048 || nx == 4096) && (ny == 2048 || ny == 4096) && tma_encoder() != nullptr;
    // opt-in (FFTPDE_WAVET=1): measured slower on C3 (488.8 vs 463.5 ms per 500 steps: column
    // pass 0.44 vs 0.56 ms, but the cluster-pair row pass 0.268 vs 0.184 ms per launch)
    static const bool on = [] { const char *e = std::getenv("FFTPDE_WAVET"); return e && e[0] == '1'; }();
    return ok && on;
}

template <int NX, int OP>
static cudaError_t rows_t(const CUtensorMap &m, const void *phys_in, void *phys_out, int64_t ny, const void *tw,
                          cudaStream_t st)
{
    using G = WaveTRowGeom<NX>;
    auto k = wavet_rows_kernel<NX, OP>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, G::BYTES);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ny, 1, 1);                   // a cluster pair per row pair
    cfg.blockDim = dim3(G::TPT, 1, 1);
    cfg.dynamicSmemBytes = G::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, m, (const double2 *)phys_in, (double2 *)phys_out, ny, (const double2 *)tw);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int NX>
static cudaError_t rows_t_nx(int op, void *T, const void *phys_in, void *phys_out, int64_t ny, const void *tw,
                             cudaStream_t st)
{
    CUtensorMap m;
    // T = [NX][ny] complex128 (y fastest): box {2 complex (a row pair), 256 kx}
    if (!tma_map<double>(m, T, ny, NX, 1, NX * ny, 2, WaveTRowGeom<NX>::BOXK, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
        return cudaErrorNotSupported;
    switch (op) {
    case WT_FWD: return rows_t<NX, WT_FWD>(m, phys_in, phys_out, ny, tw, st);
    case WT_MID: return rows_t<NX, WT_MID>(m, phys_in, phys_out, ny, tw, st);
    case WT_INV: return rows_t<NX, WT_INV>(m, phys_in, phys_out, ny, tw, st);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_wave_t_rows(int op, void *T, const void *phys_in, void *phys_out, int64_t nx, int64_t ny,
                               const void *twx32, cudaStream_t st)
{
    if (ny % 2) return cudaErrorInvalidValue;
    switch (nx) {
    case 2048: return rows_t_nx<2048>(op, T, phys_in, phys_out, ny, twx32, st);
    case 4096: return rows_t_nx<4096>(op, T, phys_in, phys_out, ny, twx32, st);
    default: return cudaErrorInvalidValue;
    }
}

template <int NY>
static cudaError_t cols_t(void *TU, void *TV, int64_t nx, const void *tw, const OpTables<double> &tab,
                          cudaStream_t st)
{
    using G = WaveTColGeom<NY>;
    auto k = wavet_cols_kernel<NY>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, G::BYTES);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * nx), 1, 1);             // a cluster pair (U, V) per column kx
    cfg.blockDim = dim3(G::TPT, 1, 1);
    cfg.dynamicSmemBytes = G::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, (double2 *)TU, (double2 *)TV, (const double2 *)tw, tab);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_wave_t_cols(void *TU, void *TV, int64_t nx, int64_t ny, const void *twy32,
                               const OpTables<double> &tab, cudaStream_t st)
{
    switch (ny) {
    case 2048: return cols_t<2048>(TU, TV, nx, twy32, tab, st);
    case 4096: return cols_t<4096>(TU, TV, nx, twy32, tab, st);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace fftpde
