// passes_c128.cu -- instantiation unit of the pass launchers for c128 (double).
#include "dispatch.cuh"

namespace fftpde {
template cudaError_t launch_rows<double>(int64_t, const void *, void *, void *, int64_t, int64_t, int64_t, int,
                                     const ColTw &, cudaStream_t, RowMul, PeerOut);
template cudaError_t launch_cols<double>(int64_t, const void *, void *, int64_t, int64_t, int64_t, int,
                                     const ColTw &, const OpTables<double> &, cudaStream_t, PeerOut);
template cudaError_t launch_wave_cols<double>(int64_t, void *, void *, int64_t, int64_t, int64_t,
                                          const ColTw &, const OpTables<double> &, cudaStream_t);
template cudaError_t launch_rows2<double>(int64_t, const void *, void *, void *, int64_t, int64_t, int64_t, int,
                                      const ColTw &, cudaStream_t, RowMul, PeerOut);
template bool small_supported<double>(int64_t, int64_t);
template cudaError_t launch_small<double>(int64_t, int64_t, const void *, void *, int64_t, int64_t, int,
                                     const void *, const void *, const OpTables<double> &, cudaStream_t);
} // namespace fftpde
