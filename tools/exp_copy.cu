// Access-pattern experiment: copy 512 MiB in (a) contiguous rows, (b) column tiles of
// W x 8 B x 512 rows (c64 512^2 grids), (c) column tiles of 2 x 16 B x 4096 rows.
#include <cstdio>
#include <cstdint>
template <int SEG_BYTES, int ROWS_PER_TILE, int THREADS>
__global__ void tile_copy(const int4* __restrict__ in, int4* __restrict__ out, long row_bytes, long grid_bytes, long tiles_per_grid, long ntiles) {
    // tile = (grid g, col group c): copies ROWS_PER_TILE rows x SEG_BYTES at column offset c*SEG_BYTES
    constexpr int V = SEG_BYTES / 16;                  // int4 per row segment
    for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        long g = tile / tiles_per_grid, c = tile % tiles_per_grid;
        const char* src = (const char*)in + g * grid_bytes + c * SEG_BYTES;
        char* dst = (char*)out + g * grid_bytes + c * SEG_BYTES;
        for (int i = threadIdx.x; i < ROWS_PER_TILE * V; i += THREADS) {
            int r = i / V, v = i % V;
            ((int4*)(dst + r * row_bytes))[v] = ((const int4*)(src + r * row_bytes))[v];
        }
    }
}
template <typename K> void run(K k, int threads, const int4* in, int4* out, long row_bytes, long grid_bytes, long tpg, long ntiles, const char* name) {
    int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, 0);
    int grid = occ * 148;
    for (int i = 0; i < 2; ++i) k<<<grid, threads>>>(in, out, row_bytes, grid_bytes, tpg, ntiles);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int i = 0; i < 10; ++i) k<<<grid, threads>>>(in, out, row_bytes, grid_bytes, tpg, ntiles); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-50s occ %2d: %7.1f us %6.0f GB/s\n", name, occ, ms * 1e3, 2.0 * (512 << 20) / (ms * 1e-3) / 1e9);
}
int main() {
    int4 *in, *out; size_t bytes = 512ul << 20; cudaMalloc(&in, bytes); cudaMalloc(&out, bytes); cudaMemset(in, 1, bytes);
    // c64 512^2 grids: row 4096 B, grid 2 MiB, 256 grids
    run(tile_copy<4096, 8, 256>, 256, in, out, 4096, 2 << 20, 64, 256 * 64, "rows: 8 x 4096 B contiguous");
    run(tile_copy<128, 512, 512>, 512, in, out, 4096, 2 << 20, 32, 256 * 32, "c64 col tile W=16 (128 B x 512 rows)");
    run(tile_copy<64, 512, 256>, 256, in, out, 4096, 2 << 20, 64, 256 * 64, "c64 col tile W=8 (64 B x 512 rows)");
    run(tile_copy<256, 512, 512>, 512, in, out, 4096, 2 << 20, 16, 256 * 16, "c64 col tile W=32 (256 B x 512 rows)");
    // c128 4096^2: row 64 KiB, 1 grid of 256 MiB, x2 -> use 2 grids
    run(tile_copy<32, 4096, 512>, 512, in, out, 65536, 256 << 20, 2048, 2 * 2048, "c128 col tile W=2 (32 B x 4096 rows)");
    run(tile_copy<16, 4096, 256>, 256, in, out, 65536, 256 << 20, 4096, 2 * 4096, "c128 col tile W=1 (16 B x 4096 rows)");
    run(tile_copy<128, 4096, 512>, 512, in, out, 65536, 256 << 20, 512, 2 * 512, "c128 col tile W=8 (128 B x 4096 rows)");
    return 0;
}
