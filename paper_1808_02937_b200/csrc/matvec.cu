// stiffness_matvec, dense path: y = A x with the dense fp64 row shard
// (O(N_d^2) per Krylov iteration).  HBM-bound GEMV: one warp per
// row, 128-bit streaming loads of A (L1 no-allocate), x from L1/L2, fixed-order
// warp-shuffle reduction (deterministic, no atomics).  Multi-RHS blocks reuse
// each A row for up to 4 right-hand sides per pass.
//
// Also: paper <-> element-interleaved permutations and the NCCL all-gather of
// row shards (world > 1).
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "fde_internal.h"

// ------------------------------------------------------------- permutation
__device__ inline long long paper_of_internal(long long r, int N, int P)
{
    int e = (int)(r / P), q = (int)(r - (long long)e * P);
    if (q < P - 1) return (long long)e * (P - 1) + q;
    return (long long)N * (P - 1) + e;
}

__global__ void k_perm_p2i(int N, int P, long long n, const double* src, long long lds, double* dst, long long ldd)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= ldd) return;
    dst[c * ldd + r] = (r < n) ? src[c * lds + paper_of_internal(r, N, P)] : 0.0;
}

__global__ void k_perm_i2p(int N, int P, long long n, const double* src, long long lds, double* dst, long long ldd)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= n) return;
    dst[c * ldd + paper_of_internal(r, N, P)] = src[c * lds + r];
}

void perm_paper_to_internal(fde_ctx* h, int N, int P, const double* src, int64_t lds, double* dst, int64_t ldd,
                            int nrhs)
{
    const long long n = (long long)N * P - 1;
    dim3 g((unsigned)ceil_div(ldd, 256), (unsigned)nrhs);
    k_perm_p2i<<<g, 256, 0, h->stream>>>(N, P, n, src, lds, dst, ldd);
    FDE_CHECK_LAUNCH();
}

void perm_internal_to_paper(fde_ctx* h, int N, int P, const double* src, int64_t lds, double* dst, int64_t ldd,
                            int nrhs)
{
    const long long n = (long long)N * P - 1;
    dim3 g((unsigned)ceil_div(n, 256), (unsigned)nrhs);
    k_perm_i2p<<<g, 256, 0, h->stream>>>(N, P, n, src, lds, dst, ldd);
    FDE_CHECK_LAUNCH();
}

// ------------------------------------------------------------------- GEMV
__device__ __forceinline__ double2 ld_stream(const double2* p)
{
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

#define GEMV_WARPS 8
#define GEMV_UNROLL 4

// y[row + c*ldy] = sum_k A[row*lda + k] x[k + c*ldx], c < NR ; lda % 2 == 0, x padded with zeros to lda
template <int NR>
__global__ void __launch_bounds__(32 * GEMV_WARPS) k_gemv(const double* __restrict__ A, long long lda,
                                                         long long rows, const double* __restrict__ x,
                                                         long long ldx, double* __restrict__ y, long long ldy)
{
    const int lane = threadIdx.x & 31;
    const long long row = (long long)blockIdx.x * GEMV_WARPS + (threadIdx.x >> 5);
    if (row >= rows) return;
    const double2* a2 = reinterpret_cast<const double2*>(A + row * lda);
    const long long n2 = lda >> 1;
    double acc[NR][2];
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[c][0] = acc[c][1] = 0.0;
    long long k = lane;
    for (; k + 32 * (GEMV_UNROLL - 1) < n2; k += 32 * GEMV_UNROLL) {
        double2 a[GEMV_UNROLL];
#pragma unroll
        for (int u = 0; u < GEMV_UNROLL; ++u) a[u] = ld_stream(a2 + k + 32 * u);
#pragma unroll
        for (int u = 0; u < GEMV_UNROLL; ++u) {
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                const double2 xv = __ldg(reinterpret_cast<const double2*>(x + c * ldx) + k + 32 * u);
                acc[c][u & 1] = fma(a[u].x, xv.x, acc[c][u & 1]);
                acc[c][u & 1] = fma(a[u].y, xv.y, acc[c][u & 1]);
            }
        }
    }
    for (; k < n2; k += 32) {
        double2 a = ld_stream(a2 + k);
#pragma unroll
        for (int c = 0; c < NR; ++c) {
            const double2 xv = __ldg(reinterpret_cast<const double2*>(x + c * ldx) + k);
            acc[c][0] = fma(a.x, xv.x, acc[c][0]);
            acc[c][0] = fma(a.y, xv.y, acc[c][0]);
        }
    }
#pragma unroll
    for (int c = 0; c < NR; ++c) {
        double v = acc[c][0] + acc[c][1];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) y[row + c * ldy] = v;
    }
}

// ---- bulk-copy GEMV (the TMA engine streams A): one CTA per SM, 8 consumer warps
// (one row each of an 8-row block) and 1 producer warp that issues 1D
// cp.async.bulk copies of (8 rows x CW columns) of A plus the matching x chunks
// into a GV_NST-stage shared-memory ring, signalled through mbarriers.  Every
// lane sums the same elements in the same order as k_gemv (bit-identical).
// Measured on c4's 537 MB operator: 6.48 TB/s (tools/mb_gemv.cu; pure-read
// ceiling 7.06 TB/s, warp-per-row k_gemv 5.33 TB/s).
#define GV_NST 3
__device__ __forceinline__ unsigned gv_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void gv_mbar_init(unsigned long long* b, unsigned cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(gv_smem(b)), "r"(cnt));
}
__device__ __forceinline__ void gv_expect_tx(unsigned long long* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gv_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gv_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gv_smem(b)) : "memory");
}
__device__ __forceinline__ void gv_wait(unsigned long long* b, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n GV_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra GV_WAIT_%=;\n}\n" ::"r"(gv_smem(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void gv_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(gv_smem(dst)), "l"(src), "r"(bytes), "r"(gv_smem(bar)) : "memory");
}
template <int NR, int CW>
constexpr int gv_smem_bytes() { return GV_NST * (8 + NR) * CW * (int)sizeof(double); }

template <int NR, int CW>
__global__ void __launch_bounds__(288) k_gemv_bulk(const double* __restrict__ A, long long lda, long long rows,
                                                   const double* __restrict__ x, long long ldx, double* __restrict__ y,
                                                   long long ldy)
{
    extern __shared__ __align__(128) double gsm_v[];
    double* ring = gsm_v;                       // [stage][8 rows][CW]
    double* xs = gsm_v + GV_NST * 8 * CW;       // [stage][NR][CW]
    __shared__ __align__(8) unsigned long long full[GV_NST], empty[GV_NST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long nblk = (rows + 7) / 8, n = lda;
    const int nch = (int)((n + CW - 1) / CW);
    if (threadIdx.x == 0) {
        for (int s = 0; s < GV_NST; ++s) {
            gv_mbar_init(&full[s], 1);
            gv_mbar_init(&empty[s], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {   // producer
        if (lane == 0) {
            int s = 0;
            unsigned ph = 0;
            for (long long rb = blockIdx.x; rb < nblk; rb += gridDim.x)
                for (int c = 0; c < nch; ++c) {
                    gv_wait(&empty[s], ph ^ 1);
                    const long long c0 = (long long)c * CW;
                    const int cw = (int)min((long long)CW, n - c0);
                    const int nr = (int)min(8LL, rows - rb * 8);
                    gv_expect_tx(&full[s], (unsigned)((nr + NR) * cw * 8));
                    for (int r = 0; r < nr; ++r)
                        gv_bulk(ring + (s * 8 + r) * CW, A + (rb * 8 + r) * lda + c0, cw * 8, &full[s]);
                    for (int q = 0; q < NR; ++q) gv_bulk(xs + (s * NR + q) * CW, x + q * ldx + c0, cw * 8, &full[s]);
                    if (++s == GV_NST) { s = 0; ph ^= 1; }
                }
        }
        return;
    }
    int s = 0;
    unsigned ph = 0;
    for (long long rb = blockIdx.x; rb < nblk; rb += gridDim.x) {
        double acc[NR][2];
#pragma unroll
        for (int q = 0; q < NR; ++q) acc[q][0] = acc[q][1] = 0.0;
        const long long row = rb * 8 + warp;
        for (int c = 0; c < nch; ++c) {
            gv_wait(&full[s], ph);
            const int cw = (int)min((long long)CW, n - (long long)c * CW);
            if (row < rows) {
                const double2* a2 = reinterpret_cast<const double2*>(ring + (s * 8 + warp) * CW);
#pragma unroll
                for (int u = 0; u < CW / 64; ++u) {
                    const int k = lane + 32 * u;
                    if (2 * k < cw) {
                        const double2 a = a2[k];
#pragma unroll
                        for (int q = 0; q < NR; ++q) {
                            const double2 xv = reinterpret_cast<const double2*>(xs + (s * NR + q) * CW)[k];
                            acc[q][u & 1] = fma(a.x, xv.x, acc[q][u & 1]);
                            acc[q][u & 1] = fma(a.y, xv.y, acc[q][u & 1]);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) gv_arrive(&empty[s]);
            if (++s == GV_NST) { s = 0; ph ^= 1; }
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) {
            double v = acc[q][0] + acc[q][1];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0 && row < rows) y[row + q * ldy] = v;
        }
    }
}

template <int NR, int CW>
static void gemv_bulk_launch(cudaStream_t s, const double* A, long long lda, long long rows, const double* x,
                             long long ldx, double* y, long long ldy)
{
    // the shared-memory opt-in and the SM count are per device
    static int smem_set[64] = {}, nsm_dev[64] = {};
    constexpr int smem = gv_smem_bytes<NR, CW>();
    int dev = 0;
    FDE_CUDA(cudaGetDevice(&dev));
    const int d = dev & 63;
    if (!smem_set[d]) {
        FDE_CUDA(cudaFuncSetAttribute(k_gemv_bulk<NR, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        smem_set[d] = 1;
    }
    if (!nsm_dev[d]) FDE_CUDA(cudaDeviceGetAttribute(&nsm_dev[d], cudaDevAttrMultiProcessorCount, dev));
    const int nsm = nsm_dev[d];
    const long long nblk = (rows + 7) / 8;
    k_gemv_bulk<NR, CW><<<(unsigned)std::min<long long>(nsm, nblk), 288, smem, s>>>(A, lda, rows, x, ldx, y, ldy);
    FDE_CHECK_LAUNCH();
}

void dense_gemv_raw(cudaStream_t s, const double* A, long long lda, long long rows, const double* x, long long ldx,
                    double* y, long long ldy, int nrhs)
{
    // bulk copies need 16-byte aligned rows / x columns (lda, ldx even, aligned bases)
    const bool bulk = (lda % 2 == 0) && (ldx % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)x % 16 == 0) &&
                      rows > 0 && getenv("FDE_GEMV_WARP") == nullptr;
    if (bulk) {
        int c = 0;
        while (c < nrhs) {
            const int r = nrhs - c;
            if (r == 1) gemv_bulk_launch<1, 1024>(s, A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            else if (r == 2) gemv_bulk_launch<2, 512>(s, A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            else if (r == 3) gemv_bulk_launch<3, 512>(s, A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            else gemv_bulk_launch<4, 512>(s, A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            c += std::min(r, 4);
        }
        return;
    }

    const unsigned blocks = (unsigned)ceil_div(rows, GEMV_WARPS);
    int c = 0;
    while (c < nrhs) {
        int r = nrhs - c;
        if (r >= 4) {
            k_gemv<4><<<blocks, 32 * GEMV_WARPS, 0, s>>>(A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            c += 4;
        } else if (r == 3) {
            k_gemv<3><<<blocks, 32 * GEMV_WARPS, 0, s>>>(A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            c += 3;
        } else if (r == 2) {
            k_gemv<2><<<blocks, 32 * GEMV_WARPS, 0, s>>>(A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            c += 2;
        } else {
            k_gemv<1><<<blocks, 32 * GEMV_WARPS, 0, s>>>(A, lda, rows, x + c * ldx, ldx, y + c * ldy, ldy);
            c += 1;
        }
        FDE_CHECK_LAUNCH();
    }
}

void dense_gemm_dmma(fde_ctx* h, const double* A, long long lda, long long rows, long long ncol, const double* X,
                     long long ldx, double* Y, long long ldy, int nrhs);

// y = A x on the shard: GEMV (HBM-bound) for up to 4 RHS per pass, the DMMA
// GEMM (FP64 tensor cores, one pass over A) from 8 RHS on
void dense_gemv(fde_ctx* h, fde_op* op, const double* x, int64_t ldx, double* y, int64_t ldy, int nrhs)
{
    if (op->r1 <= op->r0) return;   // an empty shard (more ranks than elements): no local rows
    if (nrhs >= 8 && (op->lda % 2) == 0 && (ldx % 2) == 0)
        dense_gemm_dmma(h, op->A.p, op->lda, op->r1 - op->r0, op->lda, x, ldx, y, ldy, nrhs);
    else
        dense_gemv_raw(h->stream, op->A.p, op->lda, op->r1 - op->r0, x, ldx, y, ldy, nrhs);
}

// ------------------------------------------------------------------ NCCL
// NCCL is resolved at run time (dlopen) so that the library uses the
// libnccl.so.2 already loaded by the host process (torch) when there is one.
typedef struct { char internal[128]; } nccl_uid_t;
typedef int (*nccl_getuid_fn)(nccl_uid_t*);
typedef int (*nccl_init_fn)(void**, int, nccl_uid_t, int);
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*nccl_destroy_fn)(void*);
typedef const char* (*nccl_errstr_fn)(int);

struct NcclApi {
    void* lib = nullptr;
    nccl_getuid_fn getuid = nullptr;
    nccl_init_fn init = nullptr;
    nccl_allgather_fn allgather = nullptr;
    nccl_destroy_fn destroy = nullptr;
    nccl_errstr_fn errstr = nullptr;
};

static NcclApi& nccl_api()
{
    static NcclApi api;
    if (!api.lib) {
        void* l = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!l) l = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!l) l = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!l) fde_fail(FDE_ENCCL, "cannot dlopen libnccl.so.2");
        api.lib = l;
        api.getuid = (nccl_getuid_fn)dlsym(l, "ncclGetUniqueId");
        api.init = (nccl_init_fn)dlsym(l, "ncclCommInitRank");
        api.allgather = (nccl_allgather_fn)dlsym(l, "ncclAllGather");
        api.destroy = (nccl_destroy_fn)dlsym(l, "ncclCommDestroy");
        api.errstr = (nccl_errstr_fn)dlsym(l, "ncclGetErrorString");
        if (!api.getuid || !api.init || !api.allgather || !api.destroy)
            fde_fail(FDE_ENCCL, "libnccl.so.2 lacks required symbols");
    }
    return api;
}

void comm_unique_id(void* out128)
{
    nccl_uid_t id;
    int r = nccl_api().getuid(&id);
    if (r != 0) fde_fail(FDE_ENCCL, "ncclGetUniqueId failed");
    memcpy(out128, &id, 128);
}

void comm_init(fde_ctx* h, const void* uid128)
{
    nccl_uid_t id;
    memcpy(&id, uid128, 128);
    void* comm = nullptr;
    int r = nccl_api().init(&comm, h->world, id, h->rank);
    if (r != 0) fde_fail(FDE_ENCCL, std::string("ncclCommInitRank failed: ") + (nccl_api().errstr ? nccl_api().errstr(r) : ""));
    h->nccl = comm;
}

void comm_destroy(fde_ctx* h)
{
    if (h->nccl) nccl_api().destroy(h->nccl);
    h->nccl = nullptr;
}

// gathered buffer holds world blocks of rows_max rows per RHS column -> compact
__global__ void k_compact_gather(const double* gath, long long rows_max, int world, const int64_t* rstart,
                                 long long n, double* full, long long ldfull, int nrhs)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= n) return;
    // find owning rank (world <= 64, linear scan)
    int g = 0;
    while (g + 1 < world && rstart[g + 1] <= r) ++g;
    const long long loc = r - rstart[g];
    full[c * ldfull + r] = gath[((long long)g * nrhs + c) * rows_max + loc];
}

// gathered: world blocks of nrhs columns of rows_max rows (the all-gather
// layout) -> full: n rows per column (internal order), ldfull
void comm_compact_gathered(fde_ctx* h, fde_op* op, const double* gathered, double* full, int64_t ldfull, int nrhs)
{
    if (h->g_rstart.n < (size_t)op->world) h->g_rstart.alloc(op->world);
    h->g_rstart.upload(op->rank_r0.data(), op->world, h->stream);
    dim3 g((unsigned)ceil_div(op->n, 256), (unsigned)nrhs);
    k_compact_gather<<<g, 256, 0, h->stream>>>(gathered, op->rows_max, op->world, h->g_rstart.p, op->n, full, ldfull,
                                                nrhs);
    FDE_CHECK_LAUNCH();
}

// local: (r1-r0) rows per column with ld = rows_max ; full: n rows with ldfull
void comm_allgather_rows(fde_ctx* h, fde_op* op, const double* local, double* full, int64_t ldfull, int nrhs)
{
    if (!h->nccl)
        fde_fail(FDE_ENCCL, h->virt ? "virtual rank handle: no communicator for the row all-gather"
                                    : "world > 1 without an NCCL communicator");
    const size_t chunk = (size_t)op->rows_max * nrhs;
    if (h->g_recv.n < chunk * h->world) h->g_recv.alloc(chunk * h->world);
    int r = nccl_api().allgather(local, h->g_recv.p, chunk, /*ncclFloat64*/ 8, h->nccl, h->stream);
    if (r != 0) fde_fail(FDE_ENCCL, "ncclAllGather failed");
    comm_compact_gathered(h, op, h->g_recv.p, full, ldfull, nrhs);
}

// --------------------------------------------------- operator application
// x: internal order (padded, ld ldx >= lda); y: internal order, full n rows.
void op_apply_internal(fde_ctx* h, fde_op* op, const double* x, int64_t ldx, double* y, int64_t ldy, int nrhs,
                       int path)
{
    if (path == FDE_PATH_AUTO) path = (op->flags & FDE_OP_DENSE) ? FDE_PATH_DENSE : FDE_PATH_TOEPLITZ;
    if (path == FDE_PATH_TOEPLITZ) {
        if (!(op->flags & FDE_OP_TOEPLITZ)) fde_fail(FDE_EUNSUPPORTED_MESH, "operator has no Toeplitz form");
        const int pi = prof_begin(h, PROF_FFT, 0.0);
        toeplitz_matvec(h, op, x, ldx, y, ldy, nrhs);
        prof_end(h, pi);
        return;
    }
    if (!(op->flags & FDE_OP_DENSE)) fde_fail(FDE_EINVAL_PARAM, "operator has no dense form");
    const double passes = (nrhs >= 8) ? 1.0 : (double)((nrhs + 3) / 4);
    const double gemv_bytes = 8.0 * (double)(op->r1 - op->r0) * (double)op->n * passes +
                              8.0 * (double)op->n * nrhs + 8.0 * (double)(op->r1 - op->r0) * nrhs;
    if (h->world == 1) {
        const int pi = prof_begin(h, PROF_GEMV, gemv_bytes);
        dense_gemv(h, op, x, ldx, y, ldy, nrhs);
        prof_end(h, pi);
        return;
    }
    if (!h->nccl)
        fde_fail(FDE_ENCCL, "virtual rank handle: the full operator application needs the row all-gather");
    const size_t need = (size_t)op->rows_max * nrhs;
    if (h->mv_loc.n < need) h->mv_loc.alloc(need);
    const int pi = prof_begin(h, PROF_GEMV, gemv_bytes);
    dense_gemv(h, op, x, ldx, h->mv_loc.p, op->rows_max, nrhs);
    prof_end(h, pi);
    comm_allgather_rows(h, op, h->mv_loc.p, y, ldy, nrhs);
}

// ------------------------------------------------- dense exports (tests)
__device__ inline long long paper_idx(long long r, int N, int P) { return paper_of_internal(r, N, P); }

// out (paper order, row-major ldo) <- A (internal order, row-major lda), world == 1
__global__ void k_dense_to_paper(const double* A, long long lda, long long n, int N, int P, double* out, long long ldo)
{
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long r = blockIdx.y;
    if (c >= n) return;
    out[paper_idx(r, N, P) * ldo + paper_idx(c, N, P)] = A[r * lda + c];
}

void dense_to_paper(fde_ctx* h, fde_op* op, double* out, int64_t ldo)
{
    dim3 g((unsigned)ceil_div(op->n, 256), (unsigned)op->n);
    k_dense_to_paper<<<g, 256, 0, h->stream>>>(op->A.p, op->lda, op->n, op->N, op->P, out, ldo);
    FDE_CHECK_LAUNCH();
}

// out col-major (paper order, ldo) <- in col-major (internal order, ldi)
__global__ void k_idense_to_paper(const double* in, long long ldi, long long n, int N, int P, double* out,
                                  long long ldo)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long c = blockIdx.y;
    if (r >= n) return;
    out[paper_idx(c, N, P) * ldo + paper_idx(r, N, P)] = in[c * ldi + r];
}

void internal_dense_to_paper(fde_ctx* h, int N, int P, const double* in, int64_t ldi, double* out, int64_t ldo)
{
    const long long n = (long long)N * P - 1;
    dim3 g((unsigned)ceil_div(n, 256), (unsigned)n);
    k_idense_to_paper<<<g, 256, 0, h->stream>>>(in, ldi, n, N, P, out, ldo);
    FDE_CHECK_LAUNCH();
}

void bnd_to_paper(fde_ctx* h, fde_op* op, double* out)
{
    perm_internal_to_paper(h, op->N, op->P, op->bnd.p, op->n, out, op->n, 2);
}


// ------------------------------------------------------------ profiling
long long g_fde_launches = 0;

static cudaEvent_t prof_event(fde_ctx* h)
{
    if (!h->ev_pool.empty()) {
        cudaEvent_t e = h->ev_pool.back();
        h->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    FDE_CUDA(cudaEventCreate(&e));
    return e;
}

int prof_begin(fde_ctx* h, int cls, double bytes)
{
    if (!h->profiling) return -1;
    ProfRec r;
    r.a = prof_event(h);
    r.b = prof_event(h);
    r.cls = cls;
    r.bytes = bytes;
    FDE_CUDA(cudaEventRecord(r.a, h->stream));
    h->prof.push_back(r);
    return (int)h->prof.size() - 1;
}

void prof_end(fde_ctx* h, int idx)
{
    if (idx < 0) return;
    FDE_CUDA(cudaEventRecord(h->prof[idx].b, h->stream));
}

// totals per class: out[3*c + 0] = launches, [1] = total ms, [2] = total bytes
void prof_collect(fde_ctx* h, double* out, int reset)
{
    for (int c = 0; c < PROF_NCLASS; ++c) out[3 * c] = out[3 * c + 1] = out[3 * c + 2] = 0.0;
    FDE_CUDA(cudaStreamSynchronize(h->stream));
    for (auto& r : h->prof) {
        float ms = 0;
        FDE_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        out[3 * r.cls] += 1;
        out[3 * r.cls + 1] += ms;
        out[3 * r.cls + 2] += r.bytes;
    }
    if (reset) {
        for (auto& r : h->prof) {
            h->ev_pool.push_back(r.a);
            h->ev_pool.push_back(r.b);
        }
        h->prof.clear();
    }
}

// ------------------------------------------------- multi-RHS DMMA GEMM
// Y[rows x k] = A[rows x n] X[n x k] for k >= 8 right-hand sides (config 5: 64):
// FP64 tensor cores through mma.sync.m8n8k4.f64 (DMMA; tcgen05 has no f64 kind).
// CTA tile 64 rows x 64 RHS x 32 (K), 8 warps of 16 x 32, 3-stage cp.async
// pipeline; A is streamed once from HBM, X (L2-resident) once per row tile.
// Split-K over gridDim.z: with 2 CTAs per SM, c5's 512 row tiles are 1.73 waves
// (the last one 73 % full: 13.5 % of the time lost to the tail); S = 4 K-slices
// make 2048 work units = 6.92 waves.  Each slice writes its partial product to a
// workspace and k_sum_splits adds the S partials in a fixed order (deterministic).
#define DG_BM 64
#define DG_BN 64
#define DG_BK 32
#define DG_LD 36      // padded smem row (doubles)
#define DG_STAGES 3

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) k_gemm_dmma(const double* __restrict__ A, long long lda, long long rows,
                                                  long long ncol, const double* __restrict__ X, long long ldx, int nrhs,
                                                  double* __restrict__ Y, long long ldy)
{
    extern __shared__ __align__(16) double dsm[];
    double* As = dsm;                                    // [stage][64][DG_LD]
    double* Xs = dsm + DG_STAGES * DG_BM * DG_LD;        // [stage][64 rhs][DG_LD]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long m0 = (long long)blockIdx.x * DG_BM;
    const int n0 = blockIdx.y * DG_BN;
    const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int nkt = (int)((ncol + DG_BK - 1) / DG_BK);
    const int kbeg = (int)((long long)nkt * blockIdx.z / gridDim.z), kend = (int)((long long)nkt * (blockIdx.z + 1) / gridDim.z);
    const int nk = kend - kbeg;
    if (gridDim.z > 1) Y += (long long)blockIdx.z * nrhs * ldy;   // this slice's partial (workspace, ld ldy = rows)
    auto load_stage = [&](int st, int kt0) {
        const int kt = kbeg + kt0;
        const long long k0 = (long long)kt * DG_BK;
        double* as = As + st * DG_BM * DG_LD;
        double* xs = Xs + st * DG_BN * DG_LD;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int id = tid + c * 256;                // 1024 16-byte chunks per operand
            const int r = id >> 4, kk = (id & 15) * 2;
            const long long gr = m0 + r, gk = k0 + kk;
            const bool pa = (gr < rows) && (gk < ncol);
            cp_async16(as + r * DG_LD + kk, A + (pa ? gr * lda + gk : 0), pa);
            const int rhs = n0 + r;
            const bool px = (rhs < nrhs) && (gk < ncol);
            cp_async16(xs + r * DG_LD + kk, X + (px ? (long long)rhs * ldx + gk : 0), px);
        }
    };
#pragma unroll
    for (int s = 0; s < DG_STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<DG_STAGES - 2>();
        __syncthreads();
        const int nxt = kt + DG_STAGES - 1;
        if (nxt < nk) load_stage(nxt % DG_STAGES, nxt);
        cp_async_commit();
        const double* as = As + (kt % DG_STAGES) * DG_BM * DG_LD;
        const double* xs = Xs + (kt % DG_STAGES) * DG_BN * DG_LD;
#pragma unroll
        for (int kk = 0; kk < DG_BK; kk += 4) {
            double a[2], b[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) a[i] = as[(wm + i * 8 + (lane >> 2)) * DG_LD + kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = xs[(wn + j * 8 + (lane >> 2)) * DG_LD + kk + (lane & 3)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long r = m0 + wm + i * 8 + (lane >> 2);
            const int c = n0 + wn + j * 8 + (lane & 3) * 2;
            if (r < rows) {
                if (c < nrhs) Y[(long long)c * ldy + r] = acc[i][j][0];
                if (c + 1 < nrhs) Y[(long long)(c + 1) * ldy + r] = acc[i][j][1];
            }
        }
}

// ---- the same contraction with TMA staging (cp.async.bulk.tensor) and mbarriers:
// one producer warp streams 64 x 16 tiles of A and X (128-byte rows, SWIZZLE_128B,
// out-of-range rows / columns zero-filled by the TMA unit) into a 6-stage ring; the
// eight DMMA warps wait on the stage's full barrier and release it on its empty
// barrier -- no CTA barrier and no per-thread copy instructions in the K loop.
// Fragment reads undo the swizzle: element (r, c) of a tile sits at double
// r*16 + (((c>>1) ^ (r&7)) << 1) + (c&1) (16-byte chunk XOR row mod 8: conflict free).
#define DT_BK 16                  // doubles per swizzled 128-byte tile row
#define DT_SUB 2                  // sub-tiles per stage (K = 32 per stage)
#define DT_ST 3
#define DT_TILE (DG_BM * DT_BK * DT_SUB)   // doubles per operand stage (16 KB)
#define DT_SMEM (2 * DT_ST * DT_TILE * 8 + 2 * DT_ST * 8 + 1024)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count)
{
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b)
{
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];\n" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity));
}
__device__ __forceinline__ void tma_load_2d(double* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ int dt_swz(int r, int c) { return r * DT_BK + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1); }

__global__ void __launch_bounds__(288) k_gemm_dmma_tma(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmX, long long rows,
                                                       long long ncol, int nrhs, double* __restrict__ Y, long long ldy)
{
    extern __shared__ unsigned char dt_raw[];
    double* As = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(dt_raw) + 1023) & ~(uintptr_t)1023);
    double* Xs = As + DT_ST * DT_TILE;
    uint64_t* full = reinterpret_cast<uint64_t*>(Xs + DT_ST * DT_TILE);
    uint64_t* empty = full + DT_ST;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m0 = blockIdx.x * DG_BM, n0 = blockIdx.y * DG_BN;
    const int nkt = (int)((ncol + DT_BK * DT_SUB - 1) / (DT_BK * DT_SUB));
    const int kbeg = (int)((long long)nkt * blockIdx.z / gridDim.z), kend = (int)((long long)nkt * (blockIdx.z + 1) / gridDim.z);
    const int nk = kend - kbeg;
    if (gridDim.z > 1) Y += (long long)blockIdx.z * nrhs * ldy;
    if (tid == 0) {
        for (int s = 0; s < DT_ST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {   // producer
        if (lane == 0) {
            for (int it = 0; it < nk; ++it) {
                const int s = it % DT_ST;
                if (it >= DT_ST) mbar_wait(empty + s, ((it / DT_ST) & 1) ^ 1);
                mbar_expect_tx(full + s, 2 * DT_TILE * 8);
                const int k0 = (kbeg + it) * DT_BK * DT_SUB;
#pragma unroll
                for (int u = 0; u < DT_SUB; ++u) {
                    tma_load_2d(As + s * DT_TILE + u * DG_BM * DT_BK, &tmA, k0 + u * DT_BK, m0, full + s);
                    tma_load_2d(Xs + s * DT_TILE + u * DG_BM * DT_BK, &tmX, k0 + u * DT_BK, n0, full + s);
                }
            }
        }
        return;
    }
    const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int it = 0; it < nk; ++it) {
        const int s = it % DT_ST;
        mbar_wait(full + s, (it / DT_ST) & 1);
        const double* as = As + s * DT_TILE;
        const double* xs = Xs + s * DT_TILE;
#pragma unroll
        for (int kk = 0; kk < DT_BK * DT_SUB; kk += 4) {
            const int c = (kk % DT_BK) + (lane & 3), so = (kk / DT_BK) * DG_BM * DT_BK;
            double a[2], b[4];
#pragma unroll
            for (int i = 0; i < 2; ++i) a[i] = as[so + dt_swz(wm + i * 8 + (lane >> 2), c)];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = xs[so + dt_swz(wn + j * 8 + (lane >> 2), c)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long r = m0 + wm + i * 8 + (lane >> 2);
            const int c = n0 + wn + j * 8 + (lane & 3) * 2;
            if (r < rows) {
                if (c < nrhs) Y[(long long)c * ldy + r] = acc[i][j][0];
                if (c + 1 < nrhs) Y[(long long)(c + 1) * ldy + r] = acc[i][j][1];
            }
        }
}

// row-major [d1][d0] double matrix (stride ld elements) -> 2-D tensor map with
// 64 x 16 boxes, SWIZZLE_128B; false if the layout does not qualify (stride or base
// not 16-byte aligned) or the driver entry point is missing
typedef CUresult (*tmap_encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool make_tmap(CUtensorMap* tm, const double* base, long long d0, long long d1, long long ld)
{
    static tmap_encode_fn enc = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = (tmap_encode_fn)fn;
        (void)cudaGetLastError();
    }
    if (!enc || (ld % 2) != 0 || (reinterpret_cast<uintptr_t>(base) % 16) != 0 || d0 < 1 || d1 < 1) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    const cuuint32_t box[2] = {DT_BK, DG_BM};
    const cuuint32_t es[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__global__ void k_sum_splits(const double* W, int S, long long rows, int nrhs, double* Y, long long ldy)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= rows) return;
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += W[((long long)z * nrhs + c) * rows + r];
    Y[(long long)c * ldy + r] = s;
}

void dense_gemm_dmma(fde_ctx* h, const double* A, long long lda, long long rows, long long ncol, const double* X,
                     long long ldx, double* Y, long long ldy, int nrhs)
{
    cudaStream_t s = h->stream;
    const size_t smem = (size_t)DG_STAGES * (DG_BM + DG_BN) * DG_LD * sizeof(double);
    static int smem_set_dev[64] = {};
    static int occ_dev[64] = {};
    const int dv = h->device & 63;
    if (!smem_set_dev[dv]) {   // (per device)
        FDE_CUDA(cudaFuncSetAttribute(k_gemm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        FDE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gemm_dmma, 256, smem));
        occ_dev[dv] = std::max(1, occ);
        smem_set_dev[dv] = 1;
    }
    const long long tiles = ceil_div(rows, DG_BM) * ceil_div(nrhs, DG_BN);
    const long long slots = (long long)occ_dev[dv] * h->num_sms;
    const int nkt = (int)ceil_div(ncol, DG_BK);
    // K slices: the fewest (<= 8, >= 16 K-tiles each) whose work units fill the
    // last wave to >= 95 % (FDE_GEMM_SPLITK: fixed count)
    int S = 1;
    if (const char* e = getenv("FDE_GEMM_SPLITK")) {
        S = std::max(1, std::min(8, atoi(e)));
    } else {
        for (int c = 1; c <= 8 && nkt / c >= 16; ++c) {
            const long long u = tiles * c, waves = ceil_div(u, slots);
            if ((double)u / (double)(waves * slots) >= 0.95) { S = c; break; }
        }
    }
    if (nkt / S < 1) S = 1;
    dim3 g((unsigned)ceil_div(rows, DG_BM), (unsigned)ceil_div(nrhs, DG_BN), (unsigned)S);
    // TMA + mbarrier pipeline (opt-in FDE_GEMM_TMA=1, when both operands qualify)
    const bool tma_on = getenv("FDE_GEMM_TMA") && atoi(getenv("FDE_GEMM_TMA")) == 1;
    CUtensorMap tmA, tmX;
    const bool tma = tma_on && make_tmap(&tmA, A, ncol, rows, lda) && make_tmap(&tmX, X, ncol, nrhs, ldx);
    static int tma_smem_set[64] = {};
    if (tma && !tma_smem_set[dv]) {
        FDE_CUDA(cudaFuncSetAttribute(k_gemm_dmma_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, DT_SMEM));
        tma_smem_set[dv] = 1;
    }
    double* out = Y;
    long long ldo = ldy;
    if (S > 1) {
        const size_t need = (size_t)S * nrhs * rows;
        if (h->gemm_ws.n < need) h->gemm_ws.alloc(need);
        out = h->gemm_ws.p;
        ldo = rows;
    }
    if (tma) k_gemm_dmma_tma<<<g, 288, DT_SMEM, s>>>(tmA, tmX, rows, ncol, nrhs, out, ldo);
    else k_gemm_dmma<<<g, 256, smem, s>>>(A, lda, rows, ncol, X, ldx, nrhs, out, ldo);
    FDE_CHECK_LAUNCH();
    if (S == 1) return;
    k_sum_splits<<<dim3((unsigned)ceil_div(rows, 256), (unsigned)nrhs), 256, 0, s>>>(h->gemm_ws.p, S, rows, nrhs, Y, ldy);
    FDE_CHECK_LAUNCH();
}
