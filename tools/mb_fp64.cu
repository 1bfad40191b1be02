// FP64 FMA throughput microbenchmark (dev tool): whole GPU and one SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_fma(double* out, int iters, double s)
{
    double a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] = fma(a[c], s, 1e-9);
    double r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += a[c];
    if (r == 12345.0) out[0] = r;
}
int main()
{
    double* o;
    cudaMalloc(&o, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int cfg = 0; cfg < 3; ++cfg) {
        const int blocks = cfg == 0 ? 148 * 8 : (cfg == 1 ? 1 : 1), threads = cfg == 2 ? 1024 : 256;
        k_fma<<<blocks, threads>>>(o, iters, 0.999999);
        cudaEventRecord(a);
        k_fma<<<blocks, threads>>>(o, iters, 0.999999);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double fl = 2.0 * 8 * iters * (double)blocks * threads;
        printf("blocks %d threads %d: %.3f ms, %.2f TFLOP/s fp64 (%.1f DFMA/clk/SM at 1.965 GHz over %d SMs)\n", blocks,
               threads, ms, fl / ms / 1e9, fl / 2 / (ms * 1e-3) / 1.965e9 / (blocks >= 148 ? 148 : 1), blocks >= 148 ? 148 : 1);
    }
    return 0;
}
