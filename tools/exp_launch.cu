// Kernel-boundary cost on B200: back-to-back launches of kernels that spin for
// a set time (stream and CUDA graph), vs an in-kernel grid barrier.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(long long ns)
{
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    long long t = t0;
    while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
}

__device__ unsigned int g_bar_count;
__device__ volatile unsigned int g_bar_gen;

__device__ __forceinline__ void grid_barrier(unsigned int nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int gen = g_bar_gen;
        __threadfence();
        if (atomicAdd(&g_bar_count, 1) == nblocks - 1) {
            g_bar_count = 0;
            __threadfence();
            g_bar_gen = gen + 1;
        } else {
            while (g_bar_gen == gen) { }
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void spin_barrier(long long ns, int iters)
{
    for (int i = 0; i < iters; ++i) {
        long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        t = t0;
        while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        grid_barrier(gridDim.x);
    }
}

int main()
{
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int reps = 200;
    for (long long ns : {0LL, 1000LL, 2000LL, 3000LL, 5000LL, 10000LL, 14000LL}) {
        for (int grid : {148, 296, 592}) {
            for (int i = 0; i < 10; ++i) spin<<<grid, 256, 0, s>>>(ns);
            cudaEventRecord(a, s);
            for (int i = 0; i < reps; ++i) spin<<<grid, 256, 0, s>>>(ns);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            // graph of the same launches
            cudaGraph_t g; cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < reps; ++i) spin<<<grid, 256, 0, s>>>(ns);
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(a, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float gms; cudaEventElapsedTime(&gms, a, b);
            printf("spin %6lld ns grid %4d: stream %7.3f us/launch, graph %7.3f us/launch\n", ns, grid, ms * 1e3 / reps,
                   gms * 1e3 / reps);
            cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
        }
    }
    for (long long ns : {0LL, 1000LL, 5000LL}) {
        for (int grid : {148, 296}) {
            spin_barrier<<<grid, 256, 0, s>>>(ns, 10);
            cudaEventRecord(a, s);
            spin_barrier<<<grid, 256, 0, s>>>(ns, reps);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("grid barrier: spin %6lld ns grid %4d: %7.3f us/iteration %s\n", ns, grid, ms * 1e3 / reps,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
