// microbenchmark: shared-memory leaf triangular inverse (dev tool)
#include <cstdio>
#include <cuda_runtime.h>
template <int TRN>
__global__ void __launch_bounds__(1024) k_trsm(const double* __restrict__ D, int m, long long ld, double* X,
                                              long long ldx, int ncols, int mode)
{
    extern __shared__ double T[];
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) T[t] = D[(long long)(t / m) * ld + (t % m)];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool fwd = (mode != 1);
    for (int col = blockIdx.x * nw + w; col < ncols; col += gridDim.x * nw) {
        double* x = X + (long long)col * ldx;
        double r[TRN];
#pragma unroll
        for (int t = 0; t < TRN; ++t) r[t] = (t * 32 + lane < m) ? x[t * 32 + lane] : 0.0;
        for (int s = 0; s < m; ++s) {
            const int i = fwd ? s : m - 1 - s;
            const int ti = i >> 5, li = i & 31;
            double xi = 0.0;
#pragma unroll
            for (int t = 0; t < TRN; ++t) if (t == ti) xi = r[t];
            xi = __shfl_sync(0xffffffffu, xi, li);
            if (mode != 0) xi /= T[i * m + i];
            if (lane == li) {
#pragma unroll
                for (int t = 0; t < TRN; ++t) if (t == ti) r[t] = xi;
            }
#pragma unroll
            for (int t = 0; t < TRN; ++t) {
                const int row = t * 32 + lane;
                if (row < m && (fwd ? row > i : row < i)) {
                    const double l = (mode == 2) ? T[row * m + i] : T[i * m + row];
                    r[t] = fma(-l, xi, r[t]);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < TRN; ++t) if (t * 32 + lane < m) x[t * 32 + lane] = r[t];
    }
}
int main() {
    const int m = 128;
    double *D, *X;
    cudaMalloc(&D, m * m * 8); cudaMalloc(&X, m * m * 8);
    double* h = new double[m * m];
    for (int i = 0; i < m * m; ++i) h[i] = (i % (m + 1) == 0) ? 2.0 : 0.001;
    cudaMemcpy(D, h, m * m * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(X, h, m * m * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_trsm<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, m * m * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode)
      for (int threads : {256, 512, 1024}) {
        int g = (m + threads / 32 - 1) / (threads / 32);
        k_trsm<4><<<g, threads, m * m * 8>>>(D, m, m, X, m, m, mode);
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) k_trsm<4><<<g, threads, m * m * 8>>>(D, m, m, X, m, m, mode);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("mode %d threads %d grid %d: %.2f us  (%s)\n", mode, threads, g, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
      }
    return 0;
}
