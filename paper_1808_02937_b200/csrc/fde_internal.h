// Internal declarations of libfde (B200 hot path of arXiv 1808.02937).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <vector>

#include "../../include/fde.h"

// ---------------------------------------------------------------- errors
struct FdeError {
    int code;
    std::string msg;
};

#define FDE_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess) {                                                              \
            char _b[512];                                                                     \
            snprintf(_b, sizeof(_b), "%s:%d %s: %s", __FILE__, __LINE__, #call,               \
                     cudaGetErrorString(_e));                                                 \
            throw FdeError{FDE_ECUDA, _b};                                                    \
        }                                                                                     \
    } while (0)

// every kernel launch site calls FDE_CHECK_LAUNCH(): it also counts launches
// (fde_launch_count, reported by bench.py as gpu_launches)
extern long long g_fde_launches;
#define FDE_CHECK_LAUNCH()                        \
    do {                                          \
        __atomic_add_fetch(&g_fde_launches, 1, __ATOMIC_RELAXED); \
        FDE_CUDA(cudaGetLastError());             \
    } while (0)

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl right
// behind another kernel of the same stream may start (its CTAs scheduled, its
// descriptor prologue run) while that kernel drains; it calls pdl_wait() before
// touching anything the previous kernel writes.  Every kernel that can be such a
// predecessor calls pdl_trigger() first (both are no-ops without the attribute).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
#endif
template <typename... KArgs, typename... Args>
inline void launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FDE_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

inline void fde_fail(int code, const std::string& m) { throw FdeError{code, m}; }

// ----------------------------------------------------------- device buffer
// All library buffers come from the device's stream-ordered memory pool on the
// stream of the API call in progress (fde_set_alloc_stream); the pool keeps
// freed memory (release threshold = max), so a cold solve does not pay for
// cudaMalloc/cudaFree page mapping and implicit device synchronisation.
cudaStream_t fde_alloc_stream();
void fde_set_alloc_stream(cudaStream_t s);
// Host -> device uploads staged through a page-locked ring of the calling handle
// (set by API_BEGIN): a copy from pageable memory may wait for the stream's
// pending work, which serialised the host's next steps behind the device.
// Returns false (caller copies directly) when no handle / ring is available.
bool fde_ring_upload(void* dst, const void* src, size_t bytes, cudaStream_t s);
struct fde_ctx;
void krylov_ws_free(fde_ctx* h);

// Device-time of an asynchronous library call: events recorded on its stream at
// start and end; the elapsed time is read (and waited for) only when asked.
struct LazyTimer {
    cudaEvent_t b = nullptr, e = nullptr;
    double ms = -1.0;
    LazyTimer() = default;
    LazyTimer(const LazyTimer&) = delete;
    LazyTimer& operator=(const LazyTimer&) = delete;
    void start(cudaStream_t s)
    {
        if (!b) cudaEventCreate(&b);
        if (!e) cudaEventCreate(&e);
        ms = -1.0;
        cudaEventRecord(b, s);
    }
    void stop(cudaStream_t s) { cudaEventRecord(e, s); }
    bool ready() { return ms >= 0.0 || !e || cudaEventQuery(e) == cudaSuccess; }
    double peek() { return ready() ? get() : -1.0; }   // -1: still running (does not wait)
    double get()
    {
        if (ms < 0.0 && e) {
            float f = 0.0f;
            if (cudaEventSynchronize(e) == cudaSuccess && cudaEventElapsedTime(&f, b, e) == cudaSuccess) ms = f;
        }
        return ms < 0.0 ? 0.0 : ms;
    }
    ~LazyTimer()
    {
        if (b) cudaEventDestroy(b);
        if (e) cudaEventDestroy(e);
    }
};

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        release();
        if (count == 0) return;
        s = fde_alloc_stream();
        cudaError_t e = cudaMallocAsync(&p, count * sizeof(T), s);
        if (e != cudaSuccess) {
            p = nullptr;
            throw FdeError{FDE_ENOMEM, std::string("cudaMallocAsync failed: ") + cudaGetErrorString(e)};
        }
        n = count;
    }
    void upload(const T* h, size_t count, cudaStream_t s) {
        if (count > n) alloc(count);
        if (count && !fde_ring_upload(p, h, count * sizeof(T), s))
            FDE_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void zero(cudaStream_t s) {
        if (n) FDE_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
};

// ------------------------------------------------------------------ context
// live kernel timing (CUDA events on the launching stream), enabled by fde_profile
enum { PROF_GEMV = 0, PROF_FFT = 1, PROF_PRECOND = 2, PROF_NCLASS = 3 };
struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    double bytes;
};

struct fde_ctx {
    int profiling = 0;
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int rank = 0, world = 1;
    void* nccl = nullptr;   // ncclComm_t
    bool virt = false;      // virtual rank (fde_create_virtual_rank): world > 1, no communicator
    // build stream: hmatrix_build and hlu_factor run on it, ordered only after the
    // operator's tables, so they overlap the dense assembly on the caller's stream
    cudaStream_t hb = nullptr;
    cudaEvent_t ev_hb = nullptr;
    std::string err;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int num_sms = 148;
    // auxiliary stream + events for work that overlaps the caller's stream
    // (created on first use; ordered by events, never by implicit synchronisation)
    int* pinned = nullptr;   // small page-locked read-back buffer (allocated once per handle)
    cudaStream_t aux = nullptr, aux2 = nullptr, aux3 = nullptr, aux4 = nullptr, aux5 = nullptr, aux6 = nullptr,
                 aux7 = nullptr, aux8 = nullptr;
    cudaEvent_t ev_aux[20] = {};
    // SM partition of the H-LU sweep (FDE_H2_GREEN = SMs of the bulk dense updates):
    // streams of two green contexts, made once per handle and partition size
    int green_n = 0;
    cudaStream_t g_bulk = nullptr;
    cudaStream_t g_chain[6] = {};
    void* stage = nullptr;   // page-locked staging of descriptor uploads (grow-only)
    size_t stage_bytes = 0;
    // upload ring (fde_ring_upload): two halves; a half is reused after the event
    // recorded behind its last copy completes
    void* kws = nullptr;     // Krylov workspace (krylov.cu), grow-only
    DBuf<double> kt_row, kt_col;   // pair-moment tables of the assembly (transient), grow-only
    // per-handle scratch of the operator application (several handles may run
    // concurrently on different streams / devices): the local GEMV shard, the
    // all-gather receive buffer and row starts, the Toeplitz spectra
    DBuf<double> mv_loc, g_recv;
    DBuf<double> gemm_ws;   // split-K partial products of the multi-RHS DMMA GEMM
    DBuf<int64_t> g_rstart;
    DBuf<double2> t_Dhat, t_What;
    DBuf<double> t_wv;
    char* ring = nullptr;
    size_t ring_off = 0;
    int ring_cur = 0;
    cudaEvent_t ring_ev[2] = {};
    bool ring_rec[2] = {};
};

// page-locked staging buffer of at least `bytes` (the previous contents are dropped;
// callers only grow it when no copy from it is pending)
inline void* ctx_stage(fde_ctx* h, size_t bytes)
{
    if (bytes > h->stage_bytes) {
        if (h->stage) {
            FDE_CUDA(cudaDeviceSynchronize());
            FDE_CUDA(cudaFreeHost(h->stage));
        }
        h->stage = nullptr;
        h->stage_bytes = 0;
        FDE_CUDA(cudaMallocHost(&h->stage, bytes + bytes / 4));
        h->stage_bytes = bytes + bytes / 4;
    }
    return h->stage;
}

inline int* ctx_pinned(fde_ctx* h)
{
    if (!h->pinned) FDE_CUDA(cudaMallocHost(&h->pinned, sizeof(int) * 16));
    return h->pinned;
}

inline cudaStream_t aux_stream(fde_ctx* h)
{
    if (!h->aux) {
        // priorities: the critical chains (aux: truncations, aux4: diagonal LUs,
        // aux5: the H-LU critical stream) are served before the bulk updates (aux2)
        int lo = 0, hi = 0;
        FDE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux2, cudaStreamNonBlocking, lo));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux3, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux4, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux5, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux6, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux7, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->aux8, cudaStreamNonBlocking, hi));
        for (auto& e : h->ev_aux) FDE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return h->aux;
}
inline cudaStream_t build_stream(fde_ctx* h)
{
    if (!h->hb) {
        int lo = 0, hi = 0;
        FDE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FDE_CUDA(cudaStreamCreateWithPriority(&h->hb, cudaStreamNonBlocking, hi));
        FDE_CUDA(cudaEventCreateWithFlags(&h->ev_hb, cudaEventDisableTiming));
    }
    return h->hb;
}
// make stream `waiter` wait for everything enqueued on `on` so far
inline void stream_after(fde_ctx* h, cudaStream_t waiter, cudaStream_t on)
{
    if (waiter == on) return;
    build_stream(h);
    FDE_CUDA(cudaEventRecord(h->ev_hb, on));
    FDE_CUDA(cudaStreamWaitEvent(waiter, h->ev_hb, 0));
}

inline cudaStream_t aux_stream2(fde_ctx* h)
{
    aux_stream(h);
    return h->aux2;
}
inline cudaStream_t aux_stream3(fde_ctx* h)
{
    aux_stream(h);
    return h->aux3;
}
inline cudaStream_t aux_stream4(fde_ctx* h)
{
    aux_stream(h);
    return h->aux4;
}
inline cudaStream_t aux_stream5(fde_ctx* h)
{
    aux_stream(h);
    return h->aux5;
}
inline cudaStream_t aux_stream6(fde_ctx* h)
{
    aux_stream(h);
    return h->aux6;
}
inline cudaStream_t aux_stream7(fde_ctx* h)
{
    aux_stream(h);
    return h->aux7;
}
inline cudaStream_t aux_stream8(fde_ctx* h)
{
    aux_stream(h);
    return h->aux8;
}

// ------------------------------------------------------- quadrature tables
// Host-side generation (long double), Sturm-sequence bisection for the nodes
// of the Jacobi matrix and Christoffel numbers for the weights.
namespace fdeq {
// Gauss-Legendre on [-1,1]
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w);
// Gauss-Jacobi for the weight (1-x)^a (1+x)^b on [-1,1]
void gauss_jacobi(int n, double a, double b, std::vector<double>& x, std::vector<double>& w);
}  // namespace fdeq

// Maximum points of one tensor-rule direction on the device.
#define FDE_QMAX 34   // (P + 2 points for the mass matrix at P = FDE_MAX_P = 32)
// Packed Gauss-Legendre rules for Q = 1..FDE_QMAX: offset(Q) = Q(Q-1)/2.
#define FDE_GL_TOTAL (FDE_QMAX * (FDE_QMAX + 1) / 2)

// ----------------------------------------------------------------- operator
struct AsmTables {
    // device copies
    DBuf<double> nodes;        // N+1
    DBuf<double> gjr_x, gjr_w; // Gauss-Jacobi (0, 2-alpha): radial Duffy / self outer
    DBuf<double> gji_x, gji_w; // Gauss-Jacobi (0, 1-alpha): self inner
    DBuf<double> kself;        // P*P reference self moment
    DBuf<double> mref;         // (P+1)^2 reference mass
    int qr = 0, qi = 0;
};

struct fde_op {
    LazyTimer tm;        // device time of the assembly (read lazily)
    fde_problem prob{};
    int N = 0, P = 0;
    int64_t n = 0;
    int flags = 0;
    bool uniform = false;
    bool geometric = false;         // one geometric progression h_{e+1} = q h_e (Toeplitz after scaling)
    double g0 = 0;                  // 1/Gamma(2-alpha)
    std::vector<double> nodes_h;
    AsmTables tab;
    // sharding (element ranges; rows in internal order)
    int e_lo = 0, e_hi = 0;         // owned elements [e_lo, e_hi)
    int64_t r0 = 0, r1 = 0;         // owned rows [r0, r1)
    int64_t rows_max = 0;           // max rows over ranks (allgather padding)
    std::vector<int64_t> rank_r0;   // row starts of every rank
    // dense shard
    int64_t lda = 0;
    DBuf<double> A;                 // (r1-r0) x lda row-major, internal order
    DBuf<double> bnd;               // 2 x n internal order: columns of hats 0 and N
    // Toeplitz
    int L = 0;                      // FFT length
    DBuf<double> sym;               // N x P*P lag moments K_{k,0}
    DBuf<double> spec;              // L x P x P complex (interleaved re,im): theta K^ + (1-theta) K^H
                                    // (geometric: theta K^, then (1-theta) K^H, two arrays)
    DBuf<double> wsc;               // geometric: column scales w_e = (h_e / h_0)^(1-alpha)
    DBuf<double> twid;              // L/2 complex twiddles
    // scratch
    DBuf<double> xw, yw, gw;        // internal-order work vectors
    size_t xw_cols = 0;
    double assemble_ms = 0;
    int world = 1;
    cudaEvent_t ev_side = nullptr;  // recorded on the build stream after an H-matrix build read this operator
    cudaEvent_t ev_tab = nullptr;   // recorded after the quadrature / node tables: the H-matrix build may start
    cudaEvent_t ev_k = nullptr;     // recorded after the pair-moment band (world 1): leaves can be expanded from it
    const double* kb_row = nullptr; // the band (the handle's kt_row / kt_col: valid until the next assembly)
    const double* kb_col = nullptr;
    ~fde_op()
    {
        if (ev_tab) cudaEventDestroy(ev_tab);
        if (ev_k) cudaEventDestroy(ev_k);
        if (ev_side) cudaEventDestroy(ev_side);
    }
};

// ------------------------------------------------------------- kernels API
// (implemented in assemble.cu / matvec.cu / toeplitz.cu)
struct PairList {
    // explicit element pairs (i >= j) and output slots
    DBuf<int> i, j;
    DBuf<long long> slot;
    int64_t count = 0;
};

void asm_prepare_tables(fde_ctx* h, fde_op* op);
// K blocks for rows i in [i0, i1) x j in [0, i] (packed lower triangle rows) -> out
void asm_k_triangle(fde_ctx* h, fde_op* op, int i0, int i1, double* out);
// K blocks K_{i,j} for i in [i0,i1) x j in [j0, j1), all with i > j, dense rect
void asm_k_rect(fde_ctx* h, fde_op* op, int i0, int i1, int j0, int j1, double* out);
// explicit list
void asm_k_list(fde_ctx* h, fde_op* op, const int* di, const int* dj, const long long* dslot,
                int64_t count, double* out);
// expand dense shard rows [r0,r1) from the band K storage
void asm_expand_dense(fde_ctx* h, fde_op* op, const double* Krow, const double* Kcol);
void asm_boundary_columns(fde_ctx* h, fde_op* op);
void asm_rhs(fde_ctx* h, fde_op* op, const fde_forcing* f, int nrhs, double* G_internal, int64_t ld);

// generic entry expansion from a K lookup described by a "KIndex" (see kindex.cuh)
struct KIndexDev;

// permutations
void perm_paper_to_internal(fde_ctx* h, int N, int P, const double* src, int64_t lds, double* dst,
                            int64_t ldd, int nrhs);
void perm_internal_to_paper(fde_ctx* h, int N, int P, const double* src, int64_t lds, double* dst,
                            int64_t ldd, int nrhs);

// dense matvec on the shard: y[r0..r1) = A x (internal order, padded lda)
void dense_gemv(fde_ctx* h, fde_op* op, const double* x, int64_t ldx, double* y, int64_t ldy, int nrhs);

// Toeplitz
void toeplitz_prepare(fde_ctx* h, fde_op* op);
void toeplitz_matvec(fde_ctx* h, fde_op* op, const double* x, int64_t ldx, double* y, int64_t ldy, int nrhs);

// full operator application in internal order (dense/fft + allgather)
void op_apply_internal(fde_ctx* h, fde_op* op, const double* x, int64_t ldx, double* y, int64_t ldy,
                       int nrhs, int path);

// communication
void comm_allgather_rows(fde_ctx* h, fde_op* op, const double* local, double* full, int64_t ldfull, int nrhs);
// the compaction step of comm_allgather_rows on an already gathered buffer
void comm_compact_gathered(fde_ctx* h, fde_op* op, const double* gathered, double* full, int64_t ldfull, int nrhs);

// profiling helpers (no-ops unless h->profiling)
int prof_begin(fde_ctx* h, int cls, double bytes);
void prof_end(fde_ctx* h, int idx);

// -------------------------------------------------------------- utilities
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
