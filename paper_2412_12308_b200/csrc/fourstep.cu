// fourstep.cu -- launcher of the four-step AA pass (fourstep.cuh).
#include <cuda.h>
#include "fourstep.cuh"
#include "dispatch.cuh"

namespace fftpde {

bool fourstep_supported(int64_t nx, int64_t ny, int64_t batch, int elem_bytes)
{
    return elem_bytes == 16 && nx == FsGeom::N && ny == FsGeom::N && batch == 1;
}

// The field as the 4D tensor {2 n1 (doubles), n2, m1, m2} of a [y = m1 + P m2][x = n1 + P n2]
// grid; boxes of {2 W doubles, Q, 1, Q}: one tile per box.
static bool fs_map(CUtensorMap &m, const void *p)
{
    using G = FsGeom;
    auto enc = tma_encoder();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)(2 * G::P), (cuuint64_t)G::Q, (cuuint64_t)G::P, (cuuint64_t)G::Q};
    cuuint64_t strides[3] = {(cuuint64_t)G::P * 16, (cuuint64_t)G::N * 16, (cuuint64_t)G::P * G::N * 16};
    cuuint32_t box[4] = {(cuuint32_t)(2 * G::W), (cuuint32_t)G::Q, 1, (cuuint32_t)G::Q};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void *>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int OP>
static cudaError_t aa_n(const CUtensorMap &mi, const CUtensorMap &mo, const CUtensorMap &mp, const void *tw,
                        cudaStream_t st)
{
    using G = FsGeom;
    auto k = aa_kernel<OP>;
    static SmemOptIn<decltype(k)> opt;
    cudaError_t e = opt(k, G::BYTES);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)(G::P * G::NCHUNK));
    e = launch_pdl(k, grid, dim3(G::NT), G::BYTES, st, mi, mo, mp, (const double2 *)tw);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_aa(int op, const void *in, void *out, void *phys, const void *tw, cudaStream_t st)
{
    CUtensorMap mi, mo, mp;
    if (!fs_map(mi, in)) return cudaErrorNotSupported;
    if (out == in) mo = mi;
    else if (!fs_map(mo, out)) return cudaErrorNotSupported;
    if (!phys) mp = mo;
    else if (!fs_map(mp, phys)) return cudaErrorNotSupported;
    switch (op) {
    case FS_FWD: return aa_n<FS_FWD>(mi, mo, mp, tw, st);
    case FS_INV: return aa_n<FS_INV>(mi, mo, mp, tw, st);
    case FS_MID: return aa_n<FS_MID>(mi, mo, mp, tw, st);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace fftpde
