// Cost of cooperative-groups grid barriers (dev tool).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_sync(int n, double* out)
{
    cg::grid_group g = cg::this_grid();
    double s = 0;
    for (int i = 0; i < n; ++i) {
        s += threadIdx.x * 1e-9;
        g.sync();
    }
    if (s < -1) out[0] = s;
}
// flag-based barrier: one atomic per CTA + spin (sense reversal)
__device__ unsigned int g_count = 0, g_gen = 0;
__global__ void k_flag(int n, double* out)
{
    double s = 0;
    unsigned int gen = 0;
    for (int i = 0; i < n; ++i) {
        s += threadIdx.x * 1e-9;
        __syncthreads();
        if (threadIdx.x == 0) {
            gen = *(volatile unsigned int*)&g_gen;
            __threadfence();
            if (atomicAdd(&g_count, 1) == gridDim.x - 1) {
                g_count = 0;
                __threadfence();
                atomicAdd(&g_gen, 1);
            } else {
                while (*(volatile unsigned int*)&g_gen == gen) {}
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (s < -1) out[0] = s;
}
int main()
{
    double* o;
    cudaMalloc(&o, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int thr : {256, 512}) {
        int n = 1000;
        void* args[] = {&n, &o};
        cudaLaunchCooperativeKernel((void*)k_sync, 148, thr, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_sync, 148, thr, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cg grid.sync, 148 x %d: %.2f us per barrier\n", thr, 1e3 * ms / n);
        cudaLaunchCooperativeKernel((void*)k_flag, 148, thr, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_flag, 148, thr, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("flag barrier,  148 x %d: %.2f us per barrier (%s)\n", thr, 1e3 * ms / n, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
