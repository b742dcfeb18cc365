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
__global__ void fill_random(unsigned* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)i * 2654435761u + 12345u; x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15; p[i] = x;
    }
}
// 2-level column access: tile = 8 columns (128 B) x 64 rows with row stride (stride_rows) rows
__global__ void strided_tile_copy(const int4* __restrict__ in, int4* __restrict__ out, long row_bytes, long stride_rows, long ntiles, long col_groups, long rows) {
    for (long tile = blockIdx.x * 8 + threadIdx.x / 32; tile < ntiles; tile += gridDim.x * 8) {
        long cg = tile % col_groups, r0 = tile / col_groups;     // r0 = n1 (phase A) or k1 block
        long base_row = stride_rows == 64 ? (r0 % 64) : (r0 * 64);
        int lane = threadIdx.x % 32;
        for (int i = lane; i < 64 * 8; i += 32) {
            int rr = i / 8, v = i % 8;
            long row = stride_rows == 64 ? base_row + 64 * rr : base_row + rr;
            const int4* s = (const int4*)((const char*)in + row * row_bytes + cg * 128) + v;
            int4* d = (int4*)((char*)out + row * row_bytes + cg * 128) + v;
            *d = *s;
        }
    }
}
int main() {
    int4 *in, *out; size_t bytes = 512ul << 20; cudaMalloc(&in, bytes); cudaMalloc(&out, bytes);
    fill_random<<<1024, 256>>>((unsigned*)in, bytes / 4); fill_random<<<1024, 256>>>((unsigned*)out, bytes / 4);
    // c64 512^2 grids: row 4096 B, grid 2 MiB, 256 grids
    run(tile_copy<4096, 8, 256>, 256, in, out, 4096, 2 << 20, 64, 256 * 64, "rows: 8 x 4096 B contiguous");
    run(tile_copy<128, 512, 512>, 512, in, out, 4096, 2 << 20, 32, 256 * 32, "c64 col tile W=16 (128 B x 512 rows)");
    run(tile_copy<64, 512, 256>, 256, in, out, 4096, 2 << 20, 64, 256 * 64, "c64 col tile W=8 (64 B x 512 rows)");
    run(tile_copy<256, 512, 512>, 512, in, out, 4096, 2 << 20, 16, 256 * 16, "c64 col tile W=32 (256 B x 512 rows)");
    // c128 4096^2: row 64 KiB, 1 grid of 256 MiB, x2 -> use 2 grids
    run(tile_copy<32, 4096, 512>, 512, in, out, 65536, 256 << 20, 2048, 2 * 2048, "c128 col tile W=2 (32 B x 4096 rows)");
    run(tile_copy<16, 4096, 256>, 256, in, out, 65536, 256 << 20, 4096, 2 * 4096, "c128 col tile W=1 (16 B x 4096 rows)");
    run(tile_copy<128, 4096, 512>, 512, in, out, 65536, 256 << 20, 512, 2 * 512, "c128 col tile W=8 (128 B x 4096 rows)");
    // 2-level on a 4096 x 4096 c128 field (first 256 MiB): phase A (stride 64 rows) and phase B (consecutive)
    {
        long row_bytes = 65536, col_groups = 512, ntiles = 64 * col_groups;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int ph = 0; ph < 2; ++ph) {
            long stride = ph == 0 ? 64 : 1;
            int grid = 148 * 8;
            for (int i = 0; i < 2; ++i) strided_tile_copy<<<grid, 256>>>(in, out, row_bytes, stride, ntiles, col_groups, 4096);
            cudaEventRecord(a); for (int i = 0; i < 10; ++i) strided_tile_copy<<<grid, 256>>>(in, out, row_bytes, stride, ntiles, col_groups, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
            printf("2-level %s tile 8 cols x 64 rows           : %7.1f us %6.0f GB/s\n", ph == 0 ? "A (stride 64 rows)" : "B (64 consec rows)", ms * 1e3, 2.0 * (256 << 20) / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
