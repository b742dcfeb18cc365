// FP64 / FP32 ALU roof on the box (SURVEY §8(d) "measure the sustained FP64
// clock and DFMA/DADD rate first").
//
// Each thread runs ILP independent dependency chains of one instruction kind
// for ITERS iterations; the grid is several waves of 148 x (resident CTAs), so
// the pipe, not latency, is the limit.  Reported: instructions per SM per clock
// (at the clock nvidia-smi reports during the run, sampled by the caller) and
// GFLOP/s (FMA = 2 flops, ADD/MUL = 1).  A second, seconds-long DFMA run gives
// the sustained rate under the power cap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

enum Kind { FMA = 0, ADD = 1, MUL = 2 };

template <typename T, int KIND, int ILP>
__global__ void __launch_bounds__(256) alu_kernel(T *out, int iters, T a, T b)
{
    T x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = (T)(threadIdx.x + i) * (T)1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if constexpr (KIND == FMA) x[i] = x[i] * a + b;
            else if constexpr (KIND == ADD) x[i] = x[i] + a;
            else x[i] = x[i] * a;
        }
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == (T)12345.678) out[0] = s;   // never true; keeps the chains live
}

template <typename T, int KIND, int ILP>
double run(const char *name, int iters, int reps, int *sms_out)
{
    int dev = 0, sms = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, alu_kernel<T, KIND, ILP>, 256, 0);
    const int grid = sms * occ * 4;
    T *out;
    cudaMalloc(&out, sizeof(T));
    const T a = (T)0.999999, b = (T)1e-7;
    alu_kernel<T, KIND, ILP><<<grid, 256>>>(out, iters / 10, a, b);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) alu_kernel<T, KIND, ILP><<<grid, 256>>>(out, iters, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = (double)grid * 256 * ILP * (double)iters * reps;
    const double flops = inst * (KIND == FMA ? 2 : 1);
    const double s = ms * 1e-3;
    printf("{\"kind\": \"%s\", \"grid\": %d, \"occ\": %d, \"ms\": %.3f, \"ginst_per_s\": %.1f, "
           "\"gflops\": %.1f, \"inst_per_sm_per_ns\": %.3f}\n",
           name, grid, occ, ms, inst / s * 1e-9, flops / s * 1e-9, inst / s * 1e-9 / sms);
    fflush(stdout);
    cudaFree(out);
    *sms_out = sms;
    return ms / reps;   // ms per launch
}

int main(int argc, char **argv)
{
    const double sustain_s = argc > 1 ? atof(argv[1]) : 5.0;
    int sms = 0;
    run<double, FMA, 8>("dfma", 4096, 5, &sms);
    run<double, ADD, 8>("dadd", 4096, 5, &sms);
    run<double, MUL, 8>("dmul", 4096, 5, &sms);
    run<float, FMA, 8>("ffma", 16384, 5, &sms);
    run<float, ADD, 8>("fadd", 16384, 5, &sms);
    // sustained: repeat the DFMA kernel for ~sustain_s seconds
    {
        const double per_launch_s = run<double, FMA, 8>("dfma_probe", 4096, 1, &sms) * 1e-3;
        int reps = (int)(sustain_s / (per_launch_s > 0 ? per_launch_s : 1e-3));
        if (reps < 10) reps = 10;
        if (reps > 200000) reps = 200000;
        run<double, FMA, 8>("dfma_sustained", 4096, reps, &sms);
    }
    return 0;
}
