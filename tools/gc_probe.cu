// microtest: green context stream + primary-context memory/events from the runtime API
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
__global__ void k_fill(double* p, int n, double v) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) p[i] = v + i; }
__global__ void k_smid(int* out) { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); if (threadIdx.x == 0) out[blockIdx.x] = s; }
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s failed: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)
int main() {
    RK(cudaSetDevice(0)); RK(cudaFree(0));
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs %u\n", all.sm.smCount);
    CUdevResource grp[1], rem; unsigned ng = 1;
    CK(cuDevSmResourceSplitByCount(grp, &ng, &all, &rem, 0, 112));
    printf("group %u SMs, remaining %u\n", grp[0].sm.smCount, rem.sm.smCount);
    CUdevResourceDesc d1, d2; CK(cuDevResourceGenerateDesc(&d1, &grp[0], 1)); CK(cuDevResourceGenerateDesc(&d2, &rem, 1));
    CUgreenCtx g1, g2; CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CK(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s1, s2; CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0)); CK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, -1));
    double* p; RK(cudaMalloc(&p, 1 << 20));
    int* sm1; int* sm2; RK(cudaMalloc(&sm1, 4096 * 4)); RK(cudaMalloc(&sm2, 4096 * 4));
    cudaStream_t sp; RK(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
    cudaEvent_t e; RK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    k_fill<<<256, 256, 0, sp>>>(p, 65536, 1.0);
    RK(cudaEventRecord(e, sp));
    RK(cudaStreamWaitEvent((cudaStream_t)s1, e, 0));
    k_fill<<<256, 256, 0, (cudaStream_t)s1>>>(p, 65536, 2.0);
    RK(cudaGetLastError());
    RK(cudaEventRecord(e, (cudaStream_t)s1));
    RK(cudaStreamWaitEvent(sp, e, 0));
    k_smid<<<4096, 32, 0, (cudaStream_t)s1>>>(sm1);
    k_smid<<<4096, 32, 0, (cudaStream_t)s2>>>(sm2);
    RK(cudaGetLastError());
    RK(cudaDeviceSynchronize());
    double h[4]; RK(cudaMemcpy(h, p, 32, cudaMemcpyDeviceToHost));
    printf("p[0..3] = %g %g %g %g (expect 2,3,4,5)\n", h[0], h[1], h[2], h[3]);
    int a[4096], b[4096]; RK(cudaMemcpy(a, sm1, sizeof(a), cudaMemcpyDeviceToHost)); RK(cudaMemcpy(b, sm2, sizeof(b), cudaMemcpyDeviceToHost));
    int m1[256] = {}, m2[256] = {};
    for (int i = 0; i < 4096; ++i) { m1[a[i] & 255] = 1; m2[b[i] & 255] = 1; }
    int c1 = 0, c2 = 0, both = 0; for (int i = 0; i < 256; ++i) { c1 += m1[i]; c2 += m2[i]; both += m1[i] && m2[i]; }
    printf("distinct SMs: green1 %d, green2 %d, overlap %d\n", c1, c2, both);
    // timing of a launch on a green stream vs primary
    cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
    cudaEventRecord(t0, (cudaStream_t)s1); for (int i = 0; i < 100; ++i) k_fill<<<1, 32, 0, (cudaStream_t)s1>>>(p, 32, 0.0); cudaEventRecord(t1, (cudaStream_t)s1);
    RK(cudaEventSynchronize(t1)); float ms; cudaEventElapsedTime(&ms, t0, t1); printf("100 tiny launches on green stream: %.1f us each\n", ms * 10);
    printf("OK\n");
    return 0;
}
