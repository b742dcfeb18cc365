// pack.cu -- block transpose for the sharded (slab-decomposed) path:
//   direction 0: [nrows][nblocks][bw] -> [nblocks][nrows][bw]   (row slab -> per-peer send blocks)
//   direction 1: [nblocks][nrows][bw] -> [nrows][nblocks][bw]   (received blocks -> row slab)
// Pure data movement, 16-byte vector copies; bw is a multiple of the vector.
#include <cuda_runtime.h>
#include <stdint.h>
#include "launch.h"

namespace fftpde {

__global__ void pack_blocks_kernel(const int4 *__restrict__ in, int4 *__restrict__ out, int64_t nrows,
                                   int64_t nblocks, int64_t bwv, int direction)
{
    const int64_t total = nrows * nblocks * bwv;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        // i enumerates the destination in order
        const int64_t v = i % bwv;
        const int64_t rest = i / bwv;
        int64_t src;
        if (direction == 0) {          // dst [blk][row][v] <- src [row][blk][v]
            const int64_t row = rest % nrows, blk = rest / nrows;
            src = (row * nblocks + blk) * bwv + v;
        } else {                       // dst [row][blk][v] <- src [blk][row][v]
            const int64_t blk = rest % nblocks, row = rest / nblocks;
            src = (blk * nrows + row) * bwv + v;
        }
        out[i] = in[src];
    }
}

cudaError_t launch_pack(const void *in, void *out, int64_t nrows, int64_t nblocks, int64_t bw_bytes,
                        int direction, cudaStream_t st)
{
    const int64_t bwv = bw_bytes / 16;
    const int64_t total = nrows * nblocks * bwv;
    if (total == 0) return cudaSuccess;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    pack_blocks_kernel<<<(unsigned)grid, 256, 0, st>>>((const int4 *)in, (int4 *)out, nrows, nblocks, bwv,
                                                        direction);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Slab exchange as direct stores into the peers' buffers:
// the transpose of the slab decomposition done by one kernel per rank with
// NVLink peer stores (P2P-mapped pointers), instead of a pack pass plus an
// all-to-all.  Reads are local and coalesced; every destination run is a
// contiguous bw-element segment of a peer's buffer.
//   direction 0: src = this rank's row slab [R][P*bw]; element (k, q*bw + c)
//                -> peers[q][(rank*R + k)*bw + c]        (the peer's column slab [P*R][bw])
//   direction 1: src = this rank's column slab [P*R][bw]; element (s*R + k, c)
//                -> peers[s][k*(P*bw) + rank*bw + c]      (the peer's row slab [R][P*bw])
__global__ void peer_transpose_kernel(const int4 *__restrict__ src, PeerPtrs peers, int P, int rank, int64_t R,
                                      int64_t bwv, int direction)
{
    const int64_t total = R * P * bwv;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i % bwv;           // 16-byte vector within a bw segment
        const int64_t seg = i / bwv;         // segment index in src order
        int4 *dst;
        if (direction == 0) {                // src [R][P][bwv]: seg = k*P + q
            const int64_t k = seg / P, q = seg - k * P;
            dst = (int4 *)peers.p[q] + ((int64_t)rank * R + k) * bwv + v;
        } else {                             // src [P][R][bwv]: seg = s*R + k
            const int64_t s = seg / R, k = seg - s * R;
            dst = (int4 *)peers.p[s] + (k * P + rank) * bwv + v;
        }
        *dst = src[i];
    }
}

cudaError_t launch_peer_transpose(const void *src, const PeerPtrs &peers, int P, int rank, int64_t R,
                                  int64_t bw_bytes, int direction, cudaStream_t st)
{
    const int64_t bwv = bw_bytes / 16;
    const int64_t total = R * P * bwv;
    if (total == 0) return cudaSuccess;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    peer_transpose_kernel<<<(unsigned)grid, 256, 0, st>>>((const int4 *)src, peers, P, rank, R, bwv, direction);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The row slab <-> distributed four-step layout permutation (R28), 16-byte elements:
//   A = [T][P][M][Q][P][M]  (m2_l, r, m1_l, n2, q, n1_l): a rank's row slab, rows
//        y = m1 + 1024 m2 with m1 = r M + m1_l, x = n1 + 1024 n2 with n1 = q M + n1_l
//   B = [P][P][T][M][Q][M]  (r, q, m2_l, m1_l, n2, n1_l): block r is the part of the
//        slab Y-part rank r owns, ordered as it needs it
// direction 0: A -> B, direction 1: B -> A.  Runs of M contiguous elements on both sides.
__global__ void fs_perm_kernel(const int4 *__restrict__ in, int4 *__restrict__ out, int64_t T, int64_t P, int64_t M,
                               int64_t Q, int direction)
{
    const int64_t total = T * P * M * Q * P * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = i % M;
        int64_t s = i / M;
        int64_t r, q, m2, m1, n2;
        if (direction == 0) {              // i walks B
            n2 = s % Q; s /= Q;
            m1 = s % M; s /= M;
            m2 = s % T; s /= T;
            q = s % P; r = s / P;
            out[i] = in[((((m2 * P + r) * M + m1) * Q + n2) * P + q) * M + e];
        } else {                           // i walks A
            q = s % P; s /= P;
            n2 = s % Q; s /= Q;
            m1 = s % M; s /= M;
            r = s % P; m2 = s / P;
            out[i] = in[((((r * P + q) * T + m2) * M + m1) * Q + n2) * M + e];
        }
    }
}

cudaError_t launch_fs_perm(const void *in, void *out, int P, int direction, cudaStream_t st)
{
    const int64_t M = 1024 / P, T = 32 / P, Q = 32;
    const int64_t total = T * P * M * Q * P * M;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    fs_perm_kernel<<<(unsigned)grid, 256, 0, st>>>((const int4 *)in, (int4 *)out, T, P, M, Q, direction);
    return cudaGetLastError();
}

} // namespace fftpde
