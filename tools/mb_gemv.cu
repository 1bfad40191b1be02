// GEMV variants on the c4-sized dense operator (8192 x 8192 fp64, 537 MB) (dev tool).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ double2 ld_stream(const double2* p)
{
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <int U>
__global__ void __launch_bounds__(256) k_gemv(const double* A, long long lda, long long rows, const double* x, double* y)
{
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const double2* a2 = reinterpret_cast<const double2*>(A + row * lda);
    const long long n2 = lda >> 1;
    double acc0 = 0, acc1 = 0;
    long long k = lane;
    for (; k + 32 * (U - 1) < n2; k += 32 * U) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = ld_stream(a2 + k + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double2 xv = __ldg(reinterpret_cast<const double2*>(x) + k + 32 * u);
            acc0 = fma(a[u].x, xv.x, acc0);
            acc1 = fma(a[u].y, xv.y, acc1);
        }
    }
    for (; k < n2; k += 32) {
        double2 a = ld_stream(a2 + k);
        const double2 xv = __ldg(reinterpret_cast<const double2*>(x) + k);
        acc0 = fma(a.x, xv.x, acc0);
        acc0 = fma(a.y, xv.y, acc0);
    }
    double v = acc0 + acc1;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) y[row] = v;
}
__global__ void k_read(const double2* A, long long n2, double* out)
{
    double s = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
        double2 v = ld_stream(A + i);
        s += v.x + v.y;
    }
    if (s == 1234.5) out[0] = s;
}

// ---- bulk-copy (TMA engine) GEMV: 8 consumer warps (one row each of an 8-row
// block), 1 producer warp, NST-stage ring of (8 rows x CW cols) + x chunk
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
template <int NST, int CW>
__global__ void __launch_bounds__(288) k_gemv_tma(const double* A, long long lda, long long rows, long long n,
                                                  const double* x, double* y)
{
    extern __shared__ __align__(128) double sm[];
    double* ring = sm;                         // NST x (8 x CW)
    double* xs = sm + NST * 8 * CW;            // NST x CW
    __shared__ __align__(8) unsigned long long full[NST], empty[NST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nblk = (rows + 7) / 8;
    const int nch = (int)((n + CW - 1) / CW);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {   // producer
        if (lane == 0) {
            int s = 0;
            unsigned ph = 0;
            for (long long rb = blockIdx.x; rb < nblk; rb += gridDim.x)
                for (int c = 0; c < nch; ++c) {
                    mbar_wait(&empty[s], ph ^ 1);
                    const long long c0 = (long long)c * CW;
                    const int cw = (int)min((long long)CW, n - c0);
                    const int nr = (int)min(8LL, rows - rb * 8);
                    mbar_expect_tx(&full[s], (unsigned)((nr + 1) * cw * 8));
                    for (int r = 0; r < nr; ++r)
                        bulk_g2s(ring + (s * 8 + r) * CW, A + (rb * 8 + r) * lda + c0, cw * 8, &full[s]);
                    bulk_g2s(xs + s * CW, x + c0, cw * 8, &full[s]);
                    if (++s == NST) { s = 0; ph ^= 1; }
                }
        }
        return;
    }
    int s = 0;
    unsigned ph = 0;
    for (long long rb = blockIdx.x; rb < nblk; rb += gridDim.x) {
        double acc0 = 0, acc1 = 0;
        const long long row = rb * 8 + warp;
        for (int c = 0; c < nch; ++c) {
            mbar_wait(&full[s], ph);
            const long long c0 = (long long)c * CW;
            const int cw = (int)min((long long)CW, n - c0);
            if (row < rows) {
                const double2* a2 = reinterpret_cast<const double2*>(ring + (s * 8 + warp) * CW);
                const double2* x2 = reinterpret_cast<const double2*>(xs + s * CW);
#pragma unroll
                for (int u = 0; u < CW / 64; ++u) {
                    const int k = lane + 32 * u;
                    if (2 * k < cw) {
                        const double2 a = a2[k], xv = x2[k];
                        acc0 = fma(a.x, xv.x, acc0);
                        acc1 = fma(a.y, xv.y, acc1);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == NST) { s = 0; ph ^= 1; }
        }
        double v = acc0 + acc1;
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0 && row < rows) y[row] = v;
    }
}

int main()
{
    const long long n = 8192, rows = 8192, lda = 8192;
    std::vector<double> hA(1 << 20), hx(n);
    double *A, *x, *y, *o;
    CK(cudaMalloc(&A, sizeof(double) * rows * lda));
    CK(cudaMalloc(&x, sizeof(double) * n));
    CK(cudaMalloc(&y, sizeof(double) * rows));
    CK(cudaMalloc(&o, 8));
    for (int i = 0; i < (1 << 20); ++i) hA[i] = ((i * 2654435761u) % 1000) / 1000.0 - 0.5;
    for (long long r = 0; r < rows * lda; r += (1 << 20)) CK(cudaMemcpy(A + r, hA.data(), sizeof(double) * (1 << 20), cudaMemcpyHostToDevice));
    for (int i = 0; i < n; ++i) hx[i] = (i % 7) * 0.1 - 0.3;
    CK(cudaMemcpy(x, hx.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    std::vector<double> yref(rows), yt(rows);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = 8.0 * rows * lda;
    auto timeit = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s %8.2f us  %7.1f GB/s\n", name, 1e3 * ms / 20, bytes / (ms / 20 * 1e-3) / 1e9);
    };
    timeit("pure read (148x2048 thr)", [&] { k_read<<<148 * 8, 256>>>((const double2*)A, rows * lda / 2, o); });
    timeit("pure read (148x8x4 CTAs)", [&] { k_read<<<148 * 32, 256>>>((const double2*)A, rows * lda / 2, o); });
    timeit("gemv warp/row unroll 4 (current)", [&] { k_gemv<4><<<rows / 8, 256>>>(A, lda, rows, x, y); });
    CK(cudaMemcpy(yref.data(), y, sizeof(double) * rows, cudaMemcpyDeviceToHost));
    timeit("gemv warp/row unroll 8", [&] { k_gemv<8><<<rows / 8, 256>>>(A, lda, rows, x, y); });
    timeit("gemv warp/row unroll 16", [&] { k_gemv<16><<<rows / 8, 256>>>(A, lda, rows, x, y); });
    auto variant = [&](auto nst_c, auto cw_c) {
        constexpr int NSTv = decltype(nst_c)::value, CWv = decltype(cw_c)::value;
        const int smem = (NSTv * 8 * CWv + NSTv * CWv) * 8;
        CK(cudaFuncSetAttribute(k_gemv_tma<NSTv, CWv>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        char nm[64];
        snprintf(nm, 64, "bulk ring NST %d CW %d (%d KB)", NSTv, CWv, smem / 1024);
        timeit(nm, [&] { k_gemv_tma<NSTv, CWv><<<148, 288, smem>>>(A, lda, rows, n, x, y); });
        CK(cudaMemcpy(yt.data(), y, sizeof(double) * rows, cudaMemcpyDeviceToHost));
        double md = 0;
        for (int i = 0; i < rows; ++i) md = fmax(md, fabs(yt[i] - yref[i]) / (1e-30 + fabs(yref[i])));
        if (md > 1e-12) printf("   MISMATCH %.2e\n", md);
    };
    variant(std::integral_constant<int, 4>{}, std::integral_constant<int, 512>{});
    variant(std::integral_constant<int, 6>{}, std::integral_constant<int, 512>{});
    variant(std::integral_constant<int, 3>{}, std::integral_constant<int, 1024>{});
    variant(std::integral_constant<int, 8>{}, std::integral_constant<int, 256>{});
    variant(std::integral_constant<int, 12>{}, std::integral_constant<int, 128>{});
    return 0;
}
