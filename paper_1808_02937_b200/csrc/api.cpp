// C-ABI entry points of libfde (include/fde.h).  Host orchestration only:
// validation, sharding bookkeeping, buffer management and kernel launches.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>

#include "fde_internal.h"
#include "hlu.h"
#include "hmatrix.h"

void comm_unique_id(void* out128);
void comm_init(fde_ctx* h, const void* uid128);
void comm_destroy(fde_ctx* h);
void krylov_gmres(fde_ctx* h, fde_op* op, fde_lu* lu, const double* G, double* X, int nrhs, long long ldv,
                  const fde_solve_opts* o, fde_solve_report* rep);
void krylov_bicgstab(fde_ctx* h, fde_op* op, fde_lu* lu, const double* G, double* X, int nrhs, long long ldv,
                     const fde_solve_opts* o, fde_solve_report* rep);
void dense_to_paper(fde_ctx* h, fde_op* op, double* out, int64_t ldo);
void bnd_to_paper(fde_ctx* h, fde_op* op, double* out);
void internal_dense_to_paper(fde_ctx* h, int N, int P, const double* in, int64_t ldi, double* out, int64_t ldo);
void prof_collect(fde_ctx* h, double* out, int reset);
void hlu_trunc_stats(unsigned long long* out4);
void hlu_trunc_profile(unsigned long long* out32);
int hlu_debug_truncate(fde_ctx* h, const double* U, const double* V, long long m, long long n, int k, int nb,
                       double tol, int kc, double* Uo, double* Vo);

static thread_local std::string g_noctx_err;
static thread_local cudaStream_t g_alloc_stream = nullptr;
static thread_local fde_ctx* g_cur_ctx = nullptr;
cudaStream_t fde_alloc_stream() { return g_alloc_stream; }
void fde_set_alloc_stream(cudaStream_t s) { g_alloc_stream = s; }

#define FDE_RING_HALF ((size_t)16 << 20)
bool fde_ring_upload(void* dst, const void* src, size_t bytes, cudaStream_t s)
{
    fde_ctx* h = g_cur_ctx;
    if (!h || bytes == 0 || bytes > FDE_RING_HALF) return false;
    if (!h->ring) {
        if (cudaMallocHost((void**)&h->ring, 2 * FDE_RING_HALF) != cudaSuccess) {
            h->ring = nullptr;
            return false;
        }
        for (auto& e : h->ring_ev) FDE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (h->ring_off + bytes > FDE_RING_HALF) {   // next half (its last copies were long ago)
        h->ring_cur ^= 1;
        if (h->ring_rec[h->ring_cur]) FDE_CUDA(cudaEventSynchronize(h->ring_ev[h->ring_cur]));
        h->ring_off = 0;
    }
    char* p = h->ring + (size_t)h->ring_cur * FDE_RING_HALF + h->ring_off;
    memcpy(p, src, bytes);
    FDE_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s));
    FDE_CUDA(cudaEventRecord(h->ring_ev[h->ring_cur], s));
    h->ring_rec[h->ring_cur] = true;
    h->ring_off += (bytes + 255) & ~(size_t)255;
    return true;
}

#define API_BEGIN try { if (h) fde_set_alloc_stream(h->stream); g_cur_ctx = h;
#define API_END(h)                                                   \
    }                                                                \
    catch (FdeError & e) {                                           \
        if (h) (h)->err = e.msg; else g_noctx_err = e.msg;           \
        return e.code;                                               \
    }                                                                \
    catch (std::exception & e) {                                     \
        if (h) (h)->err = e.what(); else g_noctx_err = e.what();     \
        return FDE_ECUDA;                                            \
    }                                                                \
    return FDE_OK;

extern "C" {

static int create_ctx(fde_handle* out, int device, void* cuda_stream, const void* nccl_unique_id, int rank, int world,
                      bool virt)
{
    fde_ctx* h = nullptr;
    try {
        if (!out) fde_fail(FDE_EINVAL_PARAM, "fde_create: out is NULL");
        if (world < 1 || rank < 0 || rank >= world) fde_fail(FDE_EINVAL_PARAM, "fde_create: bad rank/world");
        if (world > 1 && !nccl_unique_id && !virt)
            fde_fail(FDE_EINVAL_PARAM, "fde_create: world > 1 needs an NCCL unique id");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fde_fail(FDE_ECUDA, "no CUDA device");
        h = new fde_ctx();
        h->device = device;
        h->rank = rank;
        h->world = world;
        h->virt = virt;
        FDE_CUDA(cudaSetDevice(device));
        // NULL is the legacy default stream (stream 0), as everywhere in CUDA;
        // work is always ordered on the caller's stream.
        h->stream = (cudaStream_t)cuda_stream;
        h->own_stream = false;
        FDE_CUDA(cudaEventCreate(&h->ev0));
        FDE_CUDA(cudaEventCreate(&h->ev1));
        FDE_CUDA(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device));
        {
            // keep freed stream-ordered allocations in the pool (the H-LU allocates
            // and frees many small temporaries; returning them to the OS at every
            // synchronisation costs tens of microseconds per allocation)
            cudaMemPool_t pool;
            FDE_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t thr = UINT64_MAX;
            FDE_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        if (world > 1 && !virt) comm_init(h, nccl_unique_id);
        *out = h;
    } catch (FdeError& e) {
        g_noctx_err = e.msg;
        delete h;
        return e.code;
    } catch (std::exception& e) {
        g_noctx_err = e.what();
        delete h;
        return FDE_ENOMEM;
    }
    return FDE_OK;
}

int fde_create(fde_handle* out, int device, void* cuda_stream, const void* nccl_unique_id, int rank, int world)
{
    return create_ctx(out, device, cuda_stream, nccl_unique_id, rank, world, false);
}

int fde_create_virtual_rank(fde_handle* out, int device, void* cuda_stream, int rank, int world)
{
    return create_ctx(out, device, cuda_stream, nullptr, rank, world, true);
}

void fde_destroy(fde_handle h)
{
    if (!h) return;
    comm_destroy(h);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->pinned) cudaFreeHost(h->pinned);
    if (h->stage) cudaFreeHost(h->stage);
    krylov_ws_free(h);
    if (h->ring) cudaFreeHost(h->ring);
    for (auto e : h->ring_ev)
        if (e) cudaEventDestroy(e);
    if (h->hb) {
        cudaStreamSynchronize(h->hb);
        cudaStreamDestroy(h->hb);
        cudaEventDestroy(h->ev_hb);
    }
    if (h->aux) {
        cudaStreamSynchronize(h->aux);
        cudaStreamSynchronize(h->aux2);
        cudaStreamSynchronize(h->aux3);
        cudaStreamSynchronize(h->aux4);
        cudaStreamDestroy(h->aux4);
        cudaStreamSynchronize(h->aux5);
        cudaStreamDestroy(h->aux5);
        cudaStreamSynchronize(h->aux6);
        cudaStreamDestroy(h->aux6);
        cudaStreamSynchronize(h->aux7);
        cudaStreamDestroy(h->aux7);
        cudaStreamSynchronize(h->aux8);
        cudaStreamDestroy(h->aux8);
        cudaStreamDestroy(h->aux);
        cudaStreamDestroy(h->aux2);
        cudaStreamDestroy(h->aux3);
        for (auto e : h->ev_aux) cudaEventDestroy(e);
    }
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

const char* fde_last_error(fde_handle h) { return h ? h->err.c_str() : g_noctx_err.c_str(); }

int fde_sync(fde_handle h)
{
    API_BEGIN
    FDE_CUDA(cudaStreamSynchronize(h->stream));
    API_END(h)
}

int fde_nccl_unique_id(void* out128)
{
    fde_ctx* h = nullptr;
    API_BEGIN
    comm_unique_id(out128);
    API_END(h)
}

int fde_profile(fde_handle h, int enable)
{
    API_BEGIN
    h->profiling = enable;
    API_END(h)
}

int fde_profile_collect(fde_handle h, double* out9, int reset)
{
    API_BEGIN
    prof_collect(h, out9, reset);
    API_END(h)
}

int fde_debug_trunc_stats(unsigned long long* out4)
{
    fde_ctx* h = nullptr;
    API_BEGIN
    hlu_trunc_stats(out4);
    API_END(h)
}

int fde_debug_trunc_profile(unsigned long long* out32)
{
    fde_ctx* h = nullptr;
    API_BEGIN
    hlu_trunc_profile(out32);
    API_END(h)
}

int fde_debug_truncate(fde_handle h, const double* U, const double* V, int64_t m, int64_t n, int k, int nb, double tol,
                       int kc, double* Uo, double* Vo, int* overflow)
{
    API_BEGIN
    if (!U || !V || !Uo || !Vo || !overflow) fde_fail(FDE_EINVAL_PARAM, "fde_debug_truncate: NULL pointer");
    *overflow = hlu_debug_truncate(h, U, V, m, n, k, nb, tol, kc, Uo, Vo);
    API_END(h)
}

int fde_debug_pool_bytes(int device, unsigned long long* reserved, unsigned long long* used)
{
    fde_ctx* h = nullptr;
    API_BEGIN
    cudaMemPool_t pool;
    FDE_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    unsigned long long r = 0, u = 0;
    FDE_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r));
    FDE_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u));
    *reserved = r;
    *used = u;
    API_END(h)
}

extern int g_hlu_mode;
extern int g_hlu2_stop;
int fde_debug_hlu_mode(int mode)
{
    fde_ctx* h = nullptr;
    API_BEGIN
    if (mode < 0) fde_fail(FDE_EINVAL_PARAM, "fde_debug_hlu_mode: mode must be 0, 1 or 2 + steps");
    g_hlu_mode = mode >= 2 ? 0 : mode;
    g_hlu2_stop = mode >= 2 ? mode - 2 : -1;
    API_END(h)
}

extern unsigned long long* g_apply_tl;
extern size_t g_apply_tl_n;
// debug: copy the last preconditioner-application timeline (FDE_APPLY_TIMELINE=1) to host
int fde_debug_apply_timeline(unsigned long long* out, long long cap)
{
    if (!g_apply_tl) return 0;
    const size_t n = std::min((size_t)cap, g_apply_tl_n);
    if (cudaDeviceSynchronize() != cudaSuccess) return FDE_ECUDA;
    if (cudaMemcpy(out, g_apply_tl, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return FDE_ECUDA;
    return (int)n;
}

long long fde_launch_count(void) { return __atomic_load_n(&g_fde_launches, __ATOMIC_RELAXED); }

// Row-block partition of the dense operator (host logic, no device needed):
// rank g owns elements [N g / G, N (g+1) / G) and their dofs (element-interleaved
// rows [e_lo P, min(e_hi P, n))); rows_max pads every shard for the all-gather.
int fde_shard_rows(int N, int P, int world, int rank, int64_t* r0, int64_t* r1, int64_t* rows_max)
{
    if (N < 1 || P < 1 || world < 1 || rank < 0 || rank >= world || !r0 || !r1 || !rows_max) return FDE_EINVAL_PARAM;
    const int64_t n = (int64_t)N * P - 1;
    auto start = [&](int g) { return std::min((int64_t)((int64_t)N * g / world) * P, n); };
    *r0 = start(rank);
    *r1 = start(rank + 1);
    int64_t mx = 1;
    for (int g = 0; g < world; ++g) mx = std::max(mx, start(g + 1) - start(g));
    *rows_max = mx;
    return FDE_OK;
}

// ------------------------------------------------------------ validation
static void validate(const fde_problem* p, const fde_mesh* m)
{
    if (!p || !m || !m->nodes) fde_fail(FDE_EINVAL_PARAM, "NULL problem/mesh");
    if (!(p->a < p->b) || !std::isfinite(p->a) || !std::isfinite(p->b))
        fde_fail(FDE_EINVAL_DOMAIN, "invalid domain: need finite a < b");
    if (!std::isfinite(p->rho) || !std::isfinite(p->c1) || !std::isfinite(p->c2))
        fde_fail(FDE_EINVAL_PARAM, "rho, c1, c2 must be finite");
    if (m->N < 1) fde_fail(FDE_EINVAL_SIZE, "invalid size: N < 1");
    if (!(p->alpha > 1.0 && p->alpha < 2.0)) fde_fail(FDE_EINVAL_PARAM, "alpha must lie in (1,2)");
    if (!(p->theta >= 0.0 && p->theta <= 1.0)) fde_fail(FDE_EINVAL_PARAM, "theta must lie in [0,1]");
    if (!(p->rho >= 0.0)) fde_fail(FDE_EINVAL_PARAM, "rho must be >= 0");
    if (m->P < 1 || m->P > FDE_MAX_P) fde_fail(FDE_EDEGREE, "P must lie in [1, FDE_MAX_P]");
    if (m->nodes[0] != p->a || m->nodes[m->N] != p->b) fde_fail(FDE_EINVAL_MESH, "mesh ends must equal a and b");
    for (int i = 0; i < m->N; ++i)
        if (!(m->nodes[i + 1] > m->nodes[i])) fde_fail(FDE_EINVAL_MESH, "mesh nodes must be strictly increasing");
}

int sem_assemble(fde_handle h, const fde_problem* prob, const fde_mesh* mesh, int flags, fde_operator* out)
{
    fde_op* op = nullptr;
    try {
    if (!h) fde_fail(FDE_EINVAL_PARAM, "sem_assemble: handle is NULL");
    if (!out) fde_fail(FDE_EINVAL_PARAM, "sem_assemble: out is NULL");
    fde_set_alloc_stream(h->stream);
    g_cur_ctx = h;
    validate(prob, mesh);
    if (!(flags & (FDE_OP_DENSE | FDE_OP_TOEPLITZ))) fde_fail(FDE_EINVAL_PARAM, "flags: DENSE and/or TOEPLITZ");
    FDE_CUDA(cudaSetDevice(h->device));
    op = new fde_op();
    op->prob = *prob;
    op->N = mesh->N;
    op->P = mesh->P;
    op->n = (int64_t)mesh->N * mesh->P - 1;
    op->flags = flags;
    op->world = h->world;
    op->g0 = 1.0 / std::tgamma(2.0 - prob->alpha);
    op->nodes_h.assign(mesh->nodes, mesh->nodes + mesh->N + 1);
    {
        const double h0 = op->nodes_h[1] - op->nodes_h[0];
        bool uni = true;
        for (int i = 0; i < op->N; ++i)
            if (std::fabs((op->nodes_h[i + 1] - op->nodes_h[i]) - h0) > 1e-12 * h0) uni = false;
        op->uniform = uni;
        // one geometric progression of element sizes: the pair
        // moments are then Toeplitz after a diagonal scaling (toeplitz.cu)
        bool geo = !uni && op->N >= 2;
        const double q = op->N >= 2 ? (op->nodes_h[2] - op->nodes_h[1]) / h0 : 1.0;
        for (int i = 1; i < op->N && geo; ++i) {
            const double hp = op->nodes_h[i] - op->nodes_h[i - 1], hi = op->nodes_h[i + 1] - op->nodes_h[i];
            if (std::fabs(hi - q * hp) > 1e-10 * hi) geo = false;   // (the matvec parity tolerance)
        }
        op->geometric = geo;
    }
    if ((flags & FDE_OP_TOEPLITZ) && !op->uniform && !op->geometric)
        fde_fail(FDE_EUNSUPPORTED_MESH, "unsupported mesh: the Toeplitz path needs a uniform or single-ratio geometric mesh");
    if (op->n < 1) fde_fail(FDE_EINVAL_SIZE, "no unknowns (N*P - 1 < 1)");
    // element partition over ranks
    const int G = h->world, N = op->N, P = op->P;
    op->rank_r0.resize(G + 1);
    for (int g = 0; g < G; ++g) {
        int64_t a0, a1, mx;
        fde_shard_rows(N, P, G, g, &a0, &a1, &mx);
        op->rank_r0[g] = a0;
        op->rank_r0[g + 1] = a1;
        op->rows_max = mx;
    }
    op->e_lo = (int)((int64_t)N * h->rank / G);
    op->e_hi = (int)((int64_t)N * (h->rank + 1) / G);
    op->r0 = op->rank_r0[h->rank];
    op->r1 = op->rank_r0[h->rank + 1];
    op->lda = round_up(op->n, 32);

    op->tm.start(h->stream);   // (the call returns without waiting: the next calls' host work overlaps it)
    asm_prepare_tables(h, op);
    FDE_CUDA(cudaEventCreateWithFlags(&op->ev_tab, cudaEventDisableTiming));
    FDE_CUDA(cudaEventRecord(op->ev_tab, h->stream));
    if (flags & FDE_OP_DENSE) {
        const int b0 = op->e_lo, b1 = std::min(op->e_hi, N - 1);
        const int64_t P2 = (int64_t)P * P;
        // (handle-owned, grow-only: 4.3 GB for c5, not re-allocated per assembly)
        if (h->hb) stream_after(h, h->stream, h->hb);   // (a build may still read the previous band)
        DBuf<double>& Krow = h->kt_row;
        DBuf<double>& Kcol = h->kt_col;
        const int64_t nrow = (int64_t)(b1 + 1) * (b1 + 2) / 2 - (int64_t)b0 * (b0 + 1) / 2;
        const int64_t ncol = (int64_t)(N - 1 - b1) * (b1 - b0 + 1);
        if (Krow.n < (size_t)std::max<int64_t>(nrow, 1) * P2) Krow.alloc((size_t)std::max<int64_t>(nrow, 1) * P2);
        if (ncol > 0 && Kcol.n < (size_t)ncol * P2) Kcol.alloc((size_t)ncol * P2);
        asm_k_triangle(h, op, b0, b1 + 1, Krow.p);
        if (ncol > 0) asm_k_rect(h, op, b1 + 1, N, b0, b1 + 1, Kcol.p);
        if (G == 1) {   // the band holds every pair: the H-matrix build may expand its leaves from it
            FDE_CUDA(cudaEventCreateWithFlags(&op->ev_k, cudaEventDisableTiming));
            FDE_CUDA(cudaEventRecord(op->ev_k, h->stream));
            op->kb_row = Krow.p;
            op->kb_col = Kcol.p;
        }
        op->A.alloc((size_t)std::max<int64_t>(op->r1 - op->r0, 1) * op->lda);
        asm_expand_dense(h, op, Krow.p, Kcol.p);   // (K tables: stream-ordered release on scope exit)
    }
    asm_boundary_columns(h, op);
    if (flags & FDE_OP_TOEPLITZ) toeplitz_prepare(h, op);
    op->xw_cols = 0;
    op->tm.stop(h->stream);
    *out = op;
    op = nullptr;
    }
    catch (FdeError& e) {
        if (h) h->err = e.msg; else g_noctx_err = e.msg;
        delete op;
        return e.code;
    }
    catch (std::exception& e) {
        if (h) h->err = e.what(); else g_noctx_err = e.what();
        delete op;
        return FDE_ENOMEM;
    }
    return FDE_OK;
}

int fde_operator_wait(fde_operator op)
{
    if (!op) return FDE_EINVAL_PARAM;
    op->tm.get();
    return FDE_OK;
}

int fde_hmatrix_wait(fde_hmatrix hm)
{
    if (!hm) return FDE_EINVAL_PARAM;
    hm->tm.get();
    return FDE_OK;
}

int fde_operator_get_info(fde_operator op, fde_operator_info* info)
{
    if (!op || !info) return FDE_EINVAL_PARAM;
    info->n = op->n;
    info->N = op->N;
    info->P = op->P;
    info->row_begin = op->r0;
    info->row_end = op->r1;
    info->lda = op->lda;
    info->flags = op->flags;
    info->uniform = op->uniform ? 1 : 0;
    info->assemble_ms = op->tm.peek();   // -1 while the (asynchronous) assembly runs
    return FDE_OK;
}

int fde_operator_dense_paper(fde_handle h, fde_operator op, double* out, int64_t ldo)
{
    API_BEGIN
    if (h->world != 1) fde_fail(FDE_EINVAL_PARAM, "dense export needs world == 1");
    if (!(op->flags & FDE_OP_DENSE)) fde_fail(FDE_EINVAL_PARAM, "operator has no dense form");
    if (ldo < op->n) fde_fail(FDE_EINVAL_SIZE, "ldo < n");
    dense_to_paper(h, op, out, ldo);
    API_END(h)
}

int fde_operator_boundary_columns(fde_handle h, fde_operator op, double* out)
{
    API_BEGIN
    bnd_to_paper(h, op, out);
    API_END(h)
}

int fde_operator_rows_internal(fde_handle h, fde_operator op, double* out, int64_t ldo)
{
    API_BEGIN
    if (!(op->flags & FDE_OP_DENSE)) fde_fail(FDE_EINVAL_PARAM, "operator has no dense form");
    if (ldo < op->n) fde_fail(FDE_EINVAL_SIZE, "ldo < n");
    const int64_t rows = op->r1 - op->r0;
    if (rows > 0)
        FDE_CUDA(cudaMemcpy2DAsync(out, (size_t)ldo * sizeof(double), op->A.p, (size_t)op->lda * sizeof(double),
                                   (size_t)op->n * sizeof(double), (size_t)rows, cudaMemcpyDeviceToDevice, h->stream));
    API_END(h)
}


// ------------------------------------------------------------------ work
static void ensure_work(fde_op* op, int nrhs)
{
    if (op->xw_cols < (size_t)nrhs) {
        op->xw.alloc((size_t)nrhs * op->lda);
        op->yw.alloc((size_t)nrhs * op->lda);
        op->gw.alloc((size_t)nrhs * op->lda);
        op->xw_cols = nrhs;
    }
}

int sem_rhs(fde_handle h, fde_operator op, const fde_forcing* f, int nrhs, double* G, int64_t ld)
{
    API_BEGIN
    if (nrhs < 1 || ld < op->n) fde_fail(FDE_EINVAL_SIZE, "sem_rhs: nrhs >= 1 and ld >= n required");
    if (!f) fde_fail(FDE_EINVAL_PARAM, "sem_rhs: forcing is NULL");
    ensure_work(op, nrhs);
    asm_rhs(h, op, f, nrhs, op->gw.p, op->lda);
    perm_internal_to_paper(h, op->N, op->P, op->gw.p, op->lda, G, ld, nrhs);
    API_END(h)
}

int stiffness_matvec(fde_handle h, fde_operator op, const double* x, double* y, int nrhs, int64_t ld, int path)
{
    API_BEGIN
    if (nrhs < 1 || ld < op->n) fde_fail(FDE_EINVAL_SIZE, "stiffness_matvec: nrhs >= 1 and ld >= n required");
    if (path == FDE_PATH_TOEPLITZ && !(op->flags & FDE_OP_TOEPLITZ))
        fde_fail(FDE_EUNSUPPORTED_MESH, "unsupported mesh: operator was assembled without the Toeplitz form");
    ensure_work(op, nrhs);
    perm_paper_to_internal(h, op->N, op->P, x, ld, op->xw.p, op->lda, nrhs);
    op_apply_internal(h, op, op->xw.p, op->lda, op->yw.p, op->lda, nrhs, path);
    perm_internal_to_paper(h, op->N, op->P, op->yw.p, op->lda, y, ld, nrhs);
    API_END(h)
}

// y_loc = A[r0:r1, :] x on this rank's shard (no all-gather): x paper order,
// y_loc internal order, rows r0..r1 of every column at stride ldy (>= rows_max)
int fde_shard_matvec(fde_handle h, fde_operator op, const double* x, int64_t ldx, double* y_loc, int64_t ldy,
                     int nrhs)
{
    API_BEGIN
    if (!(op->flags & FDE_OP_DENSE)) fde_fail(FDE_EINVAL_PARAM, "operator has no dense form");
    if (nrhs < 1 || ldx < op->n || ldy < op->rows_max) fde_fail(FDE_EINVAL_SIZE, "fde_shard_matvec: sizes");
    ensure_work(op, nrhs);
    perm_paper_to_internal(h, op->N, op->P, x, ldx, op->xw.p, op->lda, nrhs);
    dense_gemv(h, op, op->xw.p, op->lda, y_loc, ldy, nrhs);
    API_END(h)
}

// The sharded matvec's communication path on ONE GPU: a one-rank NCCL communicator
// (dlopen'ed libnccl, ncclGetUniqueId, ncclCommInitRank) carries the local GEMV's
// rows through ncclAllGather and the post-all-gather compaction, exactly as a
// world > 1 stiffness_matvec does per iteration; y must equal the world-1 A x.
int fde_debug_comm_selftest(fde_handle h, fde_operator op, const double* x, double* y, int64_t ld, int nrhs)
{
    API_BEGIN
    if (h->world != 1 || h->nccl || h->virt) fde_fail(FDE_EINVAL_PARAM, "fde_debug_comm_selftest: needs a world-1 handle");
    if (!(op->flags & FDE_OP_DENSE)) fde_fail(FDE_EINVAL_PARAM, "operator has no dense form");
    if (nrhs < 1 || ld < op->n) fde_fail(FDE_EINVAL_SIZE, "fde_debug_comm_selftest: sizes");
    char uid[128];
    comm_unique_id(uid);
    comm_init(h, uid);
    try {
        ensure_work(op, nrhs);
        perm_paper_to_internal(h, op->N, op->P, x, ld, op->xw.p, op->lda, nrhs);
        const size_t need = (size_t)op->rows_max * nrhs;
        if (h->mv_loc.n < need) h->mv_loc.alloc(need);
        dense_gemv(h, op, op->xw.p, op->lda, h->mv_loc.p, op->rows_max, nrhs);
        comm_allgather_rows(h, op, h->mv_loc.p, op->yw.p, op->lda, nrhs);
        perm_internal_to_paper(h, op->N, op->P, op->yw.p, op->lda, y, ld, nrhs);
        FDE_CUDA(cudaStreamSynchronize(h->stream));
    } catch (...) {
        comm_destroy(h);
        throw;
    }
    comm_destroy(h);
    API_END(h)
}

// the compaction + permutation step that follows the all-gather, on a buffer
// in the all-gather layout (world x nrhs x rows_max) -> y paper order (ld)
int fde_debug_compact_gather(fde_handle h, fde_operator op, const double* gathered, double* y, int64_t ld, int nrhs)
{
    API_BEGIN
    if (nrhs < 1 || ld < op->n) fde_fail(FDE_EINVAL_SIZE, "fde_debug_compact_gather: sizes");
    ensure_work(op, nrhs);
    comm_compact_gathered(h, op, gathered, op->yw.p, op->lda, nrhs);
    perm_internal_to_paper(h, op->N, op->P, op->yw.p, op->lda, y, ld, nrhs);
    API_END(h)
}

// ------------------------------------------------------------- H-matrix
// The H-matrix and its H-LU need only the operator's tables and the near-field
// pair moments, not the dense operator.  Option FDE_HBUILD_SIDE (off by default):
// build them on the handle's build stream, ordered only after the pair-moment band
// (=1: leaves expanded from the band) or after the tables (=2: near field
// recomputed), overlapping the dense assembly on the caller's stream; hlu_factor
// then joins the caller's stream to the build stream at its end.  Measured on c4
// (r2 bench): 67.2 (=1) and 61.1 (=2) against 67.7 solves/s on one stream -- the
// H-LU's critical chain slows down as much as the overlap saves, so it stays off.
static int hbuild_side_mode()
{
    static const int m = getenv("FDE_HBUILD_SIDE") ? atoi(getenv("FDE_HBUILD_SIDE")) : 0;
    return m;
}
static bool hbuild_side() { return hbuild_side_mode() != 0; }

int hmatrix_build(fde_handle h, fde_operator op, int R, double lambda, int n_min, fde_hmatrix* out)
{
    cudaStream_t orig = h ? h->stream : nullptr;
    API_BEGIN
    const bool band = hbuild_side_mode() == 1 && op->ev_k && h->world == 1;
    if (hbuild_side() && op->ev_tab && (band || hbuild_side_mode() == 2)) {
        cudaStream_t hb = build_stream(h);
        FDE_CUDA(cudaStreamWaitEvent(hb, band ? op->ev_k : op->ev_tab, 0));
        h->stream = hb;
        fde_set_alloc_stream(hb);
        try {
            *out = hm_build(h, op, R, lambda, n_min, /*recompute=*/!band, /*from_band=*/band);
        } catch (...) {
            h->stream = orig;
            fde_set_alloc_stream(orig);
            throw;
        }
        (*out)->st = hb;
        h->stream = orig;
        fde_set_alloc_stream(orig);
        // (the operator's buffers must not be released before this build read them)
        if (!op->ev_side) FDE_CUDA(cudaEventCreateWithFlags(&op->ev_side, cudaEventDisableTiming));
        FDE_CUDA(cudaEventRecord(op->ev_side, hb));
    } else {
        *out = hm_build(h, op, R, lambda, n_min);
        (*out)->st = h->stream;
    }
    API_END(h)
}

int hmatrix_build_partition(fde_handle h, fde_operator op, int R, double lambda, int n_min, int partition,
                            fde_hmatrix* out)
{
    if (partition == FDE_PARTITION_INTERLEAVED) return hmatrix_build(h, op, R, lambda, n_min, out);
    API_BEGIN
    if (partition != FDE_PARTITION_PAPER) fde_fail(FDE_EINVAL_PARAM, "hmatrix_build_partition: unknown partition");
    *out = hm_build(h, op, R, lambda, n_min, false, false, 1);
    (*out)->st = h->stream;
    API_END(h)
}

int fde_hmatrix_get_info(fde_hmatrix hm, fde_hmatrix_info* info)
{
    if (!hm || !info) return FDE_EINVAL_PARAM;
    info->nblocks_dense = hm->n_dense;
    info->nblocks_lr = hm->n_lr;
    info->depth = hm->S.depth;
    info->nclusters = (int)hm->S.cl.size();
    info->dense_entries = hm->dense_words;
    info->lr_entries = hm->lr_words;
    info->build_ms = hm->tm.peek();      // -1 while the (asynchronous) build runs
    return FDE_OK;
}

int fde_hmatrix_dense_paper(fde_handle h, fde_hmatrix hm, double* out, int64_t ldo)
{
    API_BEGIN
    stream_after(h, h->stream, hm->st);
    const int64_t n = hm->S.n;
    if (ldo < n) fde_fail(FDE_EINVAL_SIZE, "ldo < n");
    DBuf<double> tmp;
    tmp.alloc((size_t)n * n);
    hm_to_dense_internal(h, hm, tmp.p, n);
    if (hm->S.paper)   // (the paper partition's blocks are already in the paper order)
        FDE_CUDA(cudaMemcpy2DAsync(out, (size_t)ldo * sizeof(double), tmp.p, (size_t)n * sizeof(double),
                                   (size_t)n * sizeof(double), (size_t)n, cudaMemcpyDeviceToDevice, h->stream));
    else
        internal_dense_to_paper(h, hm->S.N, hm->S.P, tmp.p, n, out, ldo);
    FDE_CUDA(cudaStreamSynchronize(h->stream));
    API_END(h)
}

// ----------------------------------------------------------------- H-LU
int hlu_factor(fde_handle h, fde_hmatrix hm, double tol, fde_hlu* out)
{
    cudaStream_t orig = h ? h->stream : nullptr;
    API_BEGIN
    if (!(tol >= 0.0)) fde_fail(FDE_EINVAL_PARAM, "hlu_factor: tol must be >= 0");
    if (hm->st && hm->st != orig) {   // on the H-matrix's build stream, then join the caller's stream
        h->stream = hm->st;
        fde_set_alloc_stream(hm->st);
        try {
            *out = hlu_build(h, hm, tol);
        } catch (...) {
            h->stream = orig;
            fde_set_alloc_stream(orig);
            throw;
        }
        h->stream = orig;
        fde_set_alloc_stream(orig);
        stream_after(h, orig, hm->st);
    } else {
        *out = hlu_build(h, hm, tol);
    }
    API_END(h)
}

int fde_hlu_get_info(fde_hlu lu, fde_hlu_info* info)
{
    if (!lu || !info) return FDE_EINVAL_PARAM;
    hlu_info(lu, info);
    return FDE_OK;
}

int fde_hlu_dense_internal(fde_handle h, fde_hlu lu, double* out, int64_t ldo)
{
    API_BEGIN
    hlu_dense_internal(h, lu, out, ldo);
    API_END(h)
}

int fde_hlu_solve_debug(fde_handle h, fde_hlu lu, double* X, int64_t ldx, int nrhs, int which)
{
    API_BEGIN
    hlu_solve_debug(h, lu, X, ldx, nrhs, which);
    API_END(h)
}

int precond_apply(fde_handle h, fde_hlu lu, const double* r, double* z, int nrhs, int64_t ld)
{
    API_BEGIN
    fde_op* op = hlu_operator(lu);
    if (nrhs < 1 || ld < op->n) fde_fail(FDE_EINVAL_SIZE, "precond_apply: nrhs >= 1 and ld >= n required");
    ensure_work(op, nrhs);
    perm_paper_to_internal(h, op->N, op->P, r, ld, op->xw.p, op->lda, nrhs);
    precond_apply_internal(h, lu, op->xw.p, op->lda, op->yw.p, op->lda, nrhs);
    perm_internal_to_paper(h, op->N, op->P, op->yw.p, op->lda, z, ld, nrhs);
    API_END(h)
}

// ---------------------------------------------------------------- solve
int solve(fde_handle h, fde_operator op, fde_hlu lu, const double* G, double* X, int nrhs, int64_t ld,
          const fde_solve_opts* opts, fde_solve_report* rep)
{
    API_BEGIN
    if (nrhs < 1 || ld < op->n) fde_fail(FDE_EINVAL_SIZE, "solve: nrhs >= 1 and ld >= n required");
    if (lu && hlu_operator(lu)->n != op->n) fde_fail(FDE_EDIM, "solve: preconditioner of another problem");
    fde_solve_opts o{};
    o.method = FDE_GMRES;
    o.tol = 1e-12;
    o.maxiter = 500;
    o.restart = 50;
    o.path = FDE_PATH_AUTO;
    if (opts) o = *opts;
    fde_solve_report r{};
    ensure_work(op, nrhs);
    perm_paper_to_internal(h, op->N, op->P, G, ld, op->gw.p, op->lda, nrhs);
    FDE_CUDA(cudaEventRecord(h->ev0, h->stream));
    if (o.method == FDE_BICGSTAB)
        krylov_bicgstab(h, op, lu, op->gw.p, op->xw.p, nrhs, op->lda, &o, &r);
    else
        krylov_gmres(h, op, lu, op->gw.p, op->xw.p, nrhs, op->lda, &o, &r);
    FDE_CUDA(cudaEventRecord(h->ev1, h->stream));
    perm_internal_to_paper(h, op->N, op->P, op->xw.p, op->lda, X, ld, nrhs);
    FDE_CUDA(cudaEventSynchronize(h->ev1));
    float ms = 0;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    r.solve_ms = ms;
    if (rep) *rep = r;
    FDE_CUDA(cudaStreamSynchronize(h->stream));
    if (r.converged < nrhs) {
        char b[160];
        snprintf(b, sizeof(b), "solve: %d of %d columns did not converge (relres %.3e)", nrhs - r.converged, nrhs,
                 r.relres);
        fde_fail(FDE_EMAXITER, b);
    }
    API_END(h)
}

int fde_solve(fde_handle h, fde_operator op, fde_hlu lu, const double* G, double* X, int nrhs, int64_t ld,
              const fde_solve_opts* opts, fde_solve_report* rep)
{
    return solve(h, op, lu, G, X, nrhs, ld, opts, rep);
}

void fde_free_operator(fde_operator op)
{
    // the operator's buffers are released stream-ordered on the stream they were
    // allocated on: behind any H-matrix build that read them on the build stream
    if (op && op->ev_side && op->tab.nodes.s) cudaStreamWaitEvent(op->tab.nodes.s, op->ev_side, 0);
    delete op;
}
void fde_free_hmatrix(fde_hmatrix hm) { delete hm; }
void fde_free_hlu(fde_hlu lu) { hlu_destroy(lu); }

}  // extern "C"
