// passes_c64.cu -- instantiation unit of the pass launchers for c64 (float).
#include "dispatch.cuh"

namespace fftpde {
template cudaError_t launch_rows<float>(int64_t, const void *, void *, void *, int64_t, int64_t, int64_t, int,
                                     const ColTw &, cudaStream_t, RowMul, PeerOut);
template cudaError_t launch_cols<float>(int64_t, const void *, void *, int64_t, int64_t, int64_t, int,
                                     const ColTw &, const OpTables<float> &, cudaStream_t, PeerOut);
template cudaError_t launch_wave_cols<float>(int64_t, void *, void *, int64_t, int64_t, int64_t,
                                          const ColTw &, const OpTables<float> &, cudaStream_t);
template cudaError_t launch_rows2<float>(int64_t, const void *, void *, void *, int64_t, int64_t, int64_t, int,
                                      const ColTw &, cudaStream_t, RowMul, PeerOut);
template bool small_supported<float>(int64_t, int64_t);
template cudaError_t launch_small<float>(int64_t, int64_t, const void *, void *, int64_t, int64_t, int,
                                     const void *, const void *, const OpTables<float> &, cudaStream_t);
} // namespace fftpde
