// FP64 tensor-core (DMMA) peak microbenchmark: mma.sync.m8n8k4.f64 in independent
// accumulator chains per warp, whole GPU (148 SMs x 4 CTAs x 8 warps) and one SM.
// Prints a JSON line (the measured FP64 tensor peak that bench.py quotes k_gemm_dmma
// against).  build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_dmma mb_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
__global__ void k_dmma(double* out, int iters)
{
    double d0[CH], d1[CH];
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
    for (int c = 0; c < CH; ++c) d0[c] = d1[c] = c;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d0[c]), "+d"(d1[c])
                         : "d"(a), "d"(b));
    double r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r += d0[c] + d1[c];
    if (r == 12345.0) out[0] = r;
}
__global__ void k_dfma(double* out, int iters)
{
    double a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] = fma(a[c], 0.999999, 1e-9);
    double r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += a[c];
    if (r == 12345.0) out[0] = r;
}
int main()
{
    double* o;
    cudaMalloc(&o, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    double best_gpu = 0, best_sm = 0, best_fma = 0;
    for (int rep = 0; rep < 5; ++rep) {
        for (int cfg = 0; cfg < 3; ++cfg) {
            const int blocks = cfg == 1 ? 1 : nsm * 4, threads = 256;
            float ms = 0;
            if (cfg < 2) {
                k_dmma<<<blocks, threads>>>(o, iters);
                cudaEventRecord(e0);
                k_dmma<<<blocks, threads>>>(o, iters);
                cudaEventRecord(e1);
            } else {
                k_dfma<<<blocks, threads>>>(o, iters);
                cudaEventRecord(e0);
                k_dfma<<<blocks, threads>>>(o, iters);
                cudaEventRecord(e1);
            }
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double warps = blocks * (threads / 32.0);
            const double fl = cfg < 2 ? 2.0 * 8 * 8 * 4 * CH * (double)iters * warps : 2.0 * 8 * iters * (double)blocks * threads;
            const double tf = fl / (ms * 1e-3) / 1e12;
            if (cfg == 0 && tf > best_gpu) best_gpu = tf;
            if (cfg == 1 && tf > best_sm) best_sm = tf;
            if (cfg == 2 && tf > best_fma) best_fma = tf;
        }
    }
    printf("{\"fp64_dmma_tflops\": %.3f, \"fp64_dmma_tflops_one_sm\": %.4f, \"fp64_dfma_tflops\": %.3f, \"sms\": %d, "
           "\"how\": \"mma.sync.m8n8k4.f64, %d independent accumulator chains per warp, %d CTAs x 8 warps, best of 5; "
           "DFMA: 8 chains per thread\"}\n", best_gpu, best_sm, best_fma, nsm, CH, nsm * 4);
    return 0;
}
