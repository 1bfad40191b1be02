// Krylov driver for the preconditioned system A~^{-1} A X = A~^{-1} G
// (Eq. (precondsys)).  BASELINE asks for GMRES (reading A13):
// left-preconditioned restarted GMRES(m) with classical Gram-Schmidt applied
// twice (CGS2), X0 = 0, stop when ||A~^{-1}(G - A X)|| <= tol ||A~^{-1} G||.
// The paper's BiCGSTAB (tol 1e-13) is the second method.
// All RHS columns iterate in lockstep (the matvec becomes a multi-RHS
// product); every reduction is a fixed-order block tree (deterministic,
// bitwise identical on every rank).
#include <cmath>
#include <vector>

#include "fde_internal.h"

// hlu.cu
void precond_apply_internal(fde_ctx* h, fde_lu* lu, const double* r, int64_t ldr, double* z, int64_t ldz, int nrhs);

#define KB 256

void krylov_add_small(cudaStream_t s, double* a, const double* b, int n);

__device__ inline double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ inline double block_sum(double v)
{
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    return r;   // valid in thread 0
}

// out[c*ldo + i] (+)= <V_i^c, w^c>, V laid out [i][c][ldv]
__global__ void k_multidot(const double* V, long long ldv, int nrhs, const double* w, long long ldw, long long n,
                           double* out, int ldo, int accumulate, const int* active)
{
    const int i = blockIdx.x, c = blockIdx.y;
    if (active && !active[c]) {
        if (threadIdx.x == 0 && !accumulate) out[c * ldo + i] = 0.0;
        return;
    }
    const double* v = V + ((long long)i * nrhs + c) * ldv;
    const double* x = w + c * ldw;
    double s = 0.0;
    for (long long r = threadIdx.x; r < n; r += blockDim.x) s = fma(v[r], x[r], s);
    s = block_sum(s);
    if (threadIdx.x == 0) out[c * ldo + i] = accumulate ? out[c * ldo + i] + s : s;
}

// w^c -= sum_{i<k} h[c*ldh + i] V_i^c
__global__ void k_sub_combo(const double* V, long long ldv, int nrhs, int k, const double* hcoef, int ldh, double* w,
                            long long ldw, long long n, const int* active)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= n || (active && !active[c])) return;
    double s = w[c * ldw + r];
    for (int i = 0; i < k; ++i) s = fma(-hcoef[c * ldh + i], V[((long long)i * nrhs + c) * ldv + r], s);
    w[c * ldw + r] = s;
}

// x^c += sum_{i<k_c} y[c*ldy + i] V_i^c
__global__ void k_add_combo(const double* V, long long ldv, int nrhs, const int* kc, const double* y, int ldy,
                            double* x, long long ldx, long long n)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= n) return;
    double s = x[c * ldx + r];
    for (int i = 0; i < kc[c]; ++i) s = fma(y[c * ldy + i], V[((long long)i * nrhs + c) * ldv + r], s);
    x[c * ldx + r] = s;
}

__global__ void k_norms(const double* w, long long ldw, long long n, double* out)
{
    const int c = blockIdx.x;
    double s = 0.0;
    for (long long r = threadIdx.x; r < n; r += blockDim.x) {
        double v = w[c * ldw + r];
        s = fma(v, v, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) out[c] = sqrt(s);
}

// dst^c = src^c / nrm[c] (0 if nrm == 0 or inactive)
__global__ void k_scale_into(const double* src, long long lds, const double* nrm, double* dst, long long ldd,
                             long long n, const int* active)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= ldd) return;
    double v = 0.0;
    if (r < n && (!active || active[c]) && nrm[c] > 0.0) v = src[c * lds + r] / nrm[c];
    dst[c * ldd + r] = v;
}

// Hessenberg column k of RHS c: H[c][(m+1)*k + i], i <= k+1, given h[0..k] (ldh = m+1) and hk1.
// Applies the previous Givens rotations, forms the new one, updates g, writes |g_{k+1}|.
__global__ void k_givens(int nrhs, int m, int k, const double* hcol, int ldh, const double* hk1, double* H,
                         double* cs, double* sn, double* g, double* res, const int* active)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs || !active[c]) return;
    double* Hc = H + (long long)c * (m + 1) * m + (long long)k * (m + 1);
    for (int i = 0; i <= k; ++i) Hc[i] = hcol[c * ldh + i];
    Hc[k + 1] = hk1[c];
    double* csc = cs + c * m;
    double* snc = sn + c * m;
    for (int i = 0; i < k; ++i) {
        double t = csc[i] * Hc[i] + snc[i] * Hc[i + 1];
        Hc[i + 1] = -snc[i] * Hc[i] + csc[i] * Hc[i + 1];
        Hc[i] = t;
    }
    double a = Hc[k], b = Hc[k + 1];
    double r = hypot(a, b);
    double cc = (r == 0.0) ? 1.0 : a / r, ss = (r == 0.0) ? 0.0 : b / r;
    csc[k] = cc;
    snc[k] = ss;
    Hc[k] = r;
    Hc[k + 1] = 0.0;
    double* gc = g + c * (m + 1);
    gc[k + 1] = -ss * gc[k];
    gc[k] = cc * gc[k];
    res[c] = fabs(gc[k + 1]);
}

// y = H(0:kc,0:kc)^{-1} g(0:kc) per RHS (back substitution)
__global__ void k_backsolve(int nrhs, int m, const int* kc, const double* H, const double* g, double* y)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs) return;
    const int k = kc[c];
    const double* Hc = H + (long long)c * (m + 1) * m;
    double* yc = y + c * (m + 1);
    for (int i = k - 1; i >= 0; --i) {
        double s = g[c * (m + 1) + i];
        for (int j = i + 1; j < k; ++j) s -= Hc[(long long)j * (m + 1) + i] * yc[j];
        yc[i] = (Hc[(long long)i * (m + 1) + i] != 0.0) ? s / Hc[(long long)i * (m + 1) + i] : 0.0;
    }
}

__global__ void k_set_g0(int nrhs, int m, const double* beta, double* g)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs) return;
    for (int i = 0; i <= m; ++i) g[c * (m + 1) + i] = 0.0;
    g[c * (m + 1)] = beta[c];
}

__global__ void k_residual(const double* b, long long ldb, const double* Ax, long long lda_, double* r, long long ldr,
                           long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= ldr) return;
    r[c * ldr + i] = (i < n) ? b[c * ldb + i] - Ax[c * lda_ + i] : 0.0;
}

struct KrylovWS {
    DBuf<double> V, H, cs, sn, g, y, hbuf, nrm, res, w, t, x;
    DBuf<int> active, kc;
};
void krylov_ws_free(fde_ctx* h)
{
    delete (KrylovWS*)h->kws;
    h->kws = nullptr;
}

static void apply_MA(fde_ctx* h, fde_op* op, fde_lu* lu, const double* x, long long ldx, double* out, long long ldo,
                     double* tmp, int nrhs, int path)
{
    if (lu) {
        op_apply_internal(h, op, x, ldx, tmp, ldo, nrhs, path);
        precond_apply_internal(h, lu, tmp, ldo, out, ldo, nrhs);
    } else {
        op_apply_internal(h, op, x, ldx, out, ldo, nrhs, path);
    }
}

// G, X internal order, ld = ldv (padded, >= lda)
void krylov_gmres(fde_ctx* h, fde_op* op, fde_lu* lu, const double* G, double* X, int nrhs, long long ldv,
                  const fde_solve_opts* o, fde_solve_report* rep)
{
    const long long n = op->n;
    const int m = std::max(1, std::min(o->restart > 0 ? o->restart : 50, 200));
    const int maxit = o->maxiter > 0 ? o->maxiter : 500;
    const double tol = o->tol > 0 ? o->tol : 1e-12;
    // handle-owned, grow-only workspace: the Krylov basis ((m+1) x nrhs x n, 0.86 GB for
    // c5) is not re-allocated per solve (pool growth behind large transient
    // allocations stalled some c5 solves by hundreds of ms)
    if (!h->kws) h->kws = new KrylovWS();
    KrylovWS& W = *(KrylovWS*)h->kws;
    auto need = [](auto& b, size_t cnt) {
        if (b.n < cnt) b.alloc(cnt);
    };
    need(W.V, (size_t)(m + 1) * nrhs * ldv);
    need(W.H, (size_t)nrhs * (m + 1) * m);
    need(W.cs, (size_t)nrhs * m);
    need(W.sn, (size_t)nrhs * m);
    need(W.g, (size_t)nrhs * (m + 1));
    need(W.y, (size_t)nrhs * (m + 1));
    need(W.hbuf, (size_t)nrhs * (m + 1));
    need(W.nrm, (size_t)nrhs);
    need(W.res, (size_t)nrhs);
    need(W.w, (size_t)nrhs * ldv);
    need(W.t, (size_t)nrhs * ldv);
    need(W.active, (size_t)nrhs);
    need(W.kc, (size_t)nrhs);
    cudaStream_t s = h->stream;
    const dim3 gv((unsigned)ceil_div(ldv, KB), (unsigned)nrhs);
    FDE_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * ldv * nrhs, s));

    std::vector<int> act(nrhs, 1), kcount(nrhs, 0);
    std::vector<double> hres(nrhs), bnorm(nrhs), beta(nrhs);
    // ||A~^{-1} G||
    if (lu) {
        precond_apply_internal(h, lu, G, ldv, W.w.p, ldv, nrhs);
    } else {
        FDE_CUDA(cudaMemcpyAsync(W.w.p, G, sizeof(double) * ldv * nrhs, cudaMemcpyDeviceToDevice, s));
    }
    k_norms<<<nrhs, KB, 0, s>>>(W.w.p, ldv, n, W.nrm.p);
    FDE_CHECK_LAUNCH();
    FDE_CUDA(cudaMemcpyAsync(bnorm.data(), W.nrm.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
    FDE_CUDA(cudaStreamSynchronize(s));
    for (int c = 0; c < nrhs; ++c) {
        if (!std::isfinite(bnorm[c]))   // (a NaN would otherwise read as a zero right-hand side)
            fde_fail(FDE_EBREAKDOWN, "GMRES: non-finite (preconditioned) right-hand side");
        if (!(bnorm[c] > 0.0)) act[c] = 0;   // zero RHS: X = 0
    }
    int it_total = 0, matvecs = 0;
    bool first = true;
    double worst = 0.0;
    std::vector<double> relres(nrhs, 0.0), relres_true(nrhs, -1.0);
    for (int vround = 0;; ++vround) {
    while (true) {
        int nact = 0;
        for (int c = 0; c < nrhs; ++c) nact += act[c];
        if (nact == 0 || it_total >= maxit) break;
        W.active.upload(act.data(), nrhs, s);
        // r0 = A~^{-1}(G - A X)
        if (first) {
            // X = 0 -> r0 = A~^{-1} G (already in W.w)
            first = false;
        } else {
            op_apply_internal(h, op, X, ldv, W.t.p, ldv, nrhs, o->path);
            ++matvecs;
            k_residual<<<gv, KB, 0, s>>>(G, ldv, W.t.p, ldv, W.w.p, ldv, n);
            FDE_CHECK_LAUNCH();
            if (lu) {
                precond_apply_internal(h, lu, W.w.p, ldv, W.t.p, ldv, nrhs);
                FDE_CUDA(cudaMemcpyAsync(W.w.p, W.t.p, sizeof(double) * ldv * nrhs, cudaMemcpyDeviceToDevice, s));
            }
        }
        k_norms<<<nrhs, KB, 0, s>>>(W.w.p, ldv, n, W.nrm.p);
        FDE_CHECK_LAUNCH();
        k_scale_into<<<gv, KB, 0, s>>>(W.w.p, ldv, W.nrm.p, W.V.p, ldv, n, W.active.p);
        FDE_CHECK_LAUNCH();
        k_set_g0<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, m, W.nrm.p, W.g.p);
        FDE_CHECK_LAUNCH();
        std::vector<int> kc(nrhs, 0);
        int k = 0;
        for (; k < m && it_total < maxit; ++k) {
            double* Vk = W.V.p + (size_t)k * nrhs * ldv;
            double* Vk1 = W.V.p + (size_t)(k + 1) * nrhs * ldv;
            apply_MA(h, op, lu, Vk, ldv, W.w.p, ldv, W.t.p, nrhs, o->path);
            ++matvecs;
            ++it_total;
            // CGS2
            k_multidot<<<dim3(k + 1, nrhs), KB, 0, s>>>(W.V.p, ldv, nrhs, W.w.p, ldv, n, W.hbuf.p, m + 1, 0,
                                                         W.active.p);
            FDE_CHECK_LAUNCH();
            k_sub_combo<<<gv, KB, 0, s>>>(W.V.p, ldv, nrhs, k + 1, W.hbuf.p, m + 1, W.w.p, ldv, n, W.active.p);
            FDE_CHECK_LAUNCH();
            k_multidot<<<dim3(k + 1, nrhs), KB, 0, s>>>(W.V.p, ldv, nrhs, W.w.p, ldv, n, W.y.p, m + 1, 0,
                                                         W.active.p);
            FDE_CHECK_LAUNCH();
            k_sub_combo<<<gv, KB, 0, s>>>(W.V.p, ldv, nrhs, k + 1, W.y.p, m + 1, W.w.p, ldv, n, W.active.p);
            FDE_CHECK_LAUNCH();
            k_norms<<<nrhs, KB, 0, s>>>(W.w.p, ldv, n, W.nrm.p);
            FDE_CHECK_LAUNCH();
            k_scale_into<<<gv, KB, 0, s>>>(W.w.p, ldv, W.nrm.p, Vk1, ldv, n, W.active.p);
            FDE_CHECK_LAUNCH();
            // Hessenberg column = first CGS pass + second CGS pass
            krylov_add_small(s, W.hbuf.p, W.y.p, nrhs * (m + 1));
            k_givens<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, m, k, W.hbuf.p, m + 1, W.nrm.p, W.H.p, W.cs.p, W.sn.p,
                                                       W.g.p, W.res.p, W.active.p);
            FDE_CHECK_LAUNCH();
            FDE_CUDA(cudaMemcpyAsync(hres.data(), W.res.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
            FDE_CUDA(cudaStreamSynchronize(s));
            bool any = false;
            for (int c = 0; c < nrhs; ++c) {
                if (!act[c]) continue;
                kc[c] = k + 1;
                relres[c] = hres[c] / bnorm[c];
                if (!(hres[c] == hres[c])) fde_fail(FDE_EBREAKDOWN, "GMRES: NaN residual");
                if (relres[c] <= tol) act[c] = 0;   // freeze this column's Hessenberg
                else any = true;
            }
            W.active.upload(act.data(), nrhs, s);
            if (!any) {
                ++k;
                break;
            }
        }
        // X += V y
        W.kc.upload(kc.data(), nrhs, s);
        k_backsolve<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, m, W.kc.p, W.H.p, W.g.p, W.y.p);
        FDE_CHECK_LAUNCH();
        k_add_combo<<<gv, KB, 0, s>>>(W.V.p, ldv, nrhs, W.kc.p, W.y.p, m + 1, X, ldv, n);
        FDE_CHECK_LAUNCH();
        FDE_CUDA(cudaStreamSynchronize(s));
        // columns still active restart; converged ones stay frozen
        (void)k;
    }
    // verification (opts->verify): the Givens estimate |g_{k+1}| equals the
    // preconditioned residual only in exact arithmetic -- recompute
    // ||A~^{-1}(G - A X)|| once and restart the columns that are above tol
    if (!o->verify) break;
    op_apply_internal(h, op, X, ldv, W.t.p, ldv, nrhs, o->path);
    ++matvecs;
    k_residual<<<gv, KB, 0, s>>>(G, ldv, W.t.p, ldv, W.w.p, ldv, n);
    FDE_CHECK_LAUNCH();
    if (lu) {
        precond_apply_internal(h, lu, W.w.p, ldv, W.t.p, ldv, nrhs);
        FDE_CUDA(cudaMemcpyAsync(W.w.p, W.t.p, sizeof(double) * ldv * nrhs, cudaMemcpyDeviceToDevice, s));
    }
    k_norms<<<nrhs, KB, 0, s>>>(W.w.p, ldv, n, W.nrm.p);
    FDE_CHECK_LAUNCH();
    FDE_CUDA(cudaMemcpyAsync(hres.data(), W.nrm.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
    FDE_CUDA(cudaStreamSynchronize(s));
    bool again = false;
    for (int c = 0; c < nrhs; ++c) {
        if (!(bnorm[c] > 0.0)) continue;
        relres_true[c] = hres[c] / bnorm[c];
        relres[c] = relres_true[c];
        if (relres[c] > tol && it_total < maxit && vround < 3) {
            act[c] = 1;   // restart from the current X (r0 is recomputed at the loop head)
            again = true;
        }
    }
    if (!again) break;
    }
    int conv = 0;
    worst = 0.0;
    for (int c = 0; c < nrhs; ++c) {
        if (!(bnorm[c] > 0.0) || relres[c] <= tol) ++conv;
        worst = std::max(worst, relres[c]);
    }
    rep->iterations = it_total;
    rep->matvecs = matvecs;
    rep->converged = conv;
    rep->relres = worst;
    double wt = -1.0;
    for (int c = 0; c < nrhs; ++c) wt = std::max(wt, relres_true[c]);
    rep->relres_true = wt;
}

__global__ void k_add_small(double* a, const double* b, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] += b[i];
}

void krylov_add_small(cudaStream_t s, double* a, const double* b, int n)
{
    k_add_small<<<ceil_div(n, 256), 256, 0, s>>>(a, b, n);
    FDE_CHECK_LAUNCH();
}

// ------------------------------------------------------------- BiCGSTAB
// Left-preconditioned BiCGSTAB (the paper's solver): two
// operator applications per iteration.  Per-column scalars live on the device.
__global__ void k_dot_cols(const double* a, long long lda_, const double* b, long long ldb, long long n, double* out)
{
    const int c = blockIdx.x;
    double s = 0.0;
    for (long long r = threadIdx.x; r < n; r += blockDim.x) s = fma(a[c * lda_ + r], b[c * ldb + r], s);
    s = block_sum(s);
    if (threadIdx.x == 0) out[c] = s;
}

// scalars per column: [rho, rho_prev, alpha, omega, beta, tmp]
#define BS 6
__global__ void k_bicg_beta(int nrhs, double* sc, const int* active)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs || !active[c]) return;
    double* s = sc + c * BS;
    s[4] = (s[0] / s[1]) * (s[2] / s[3]);
    s[1] = s[0];
}
__global__ void k_bicg_alpha(int nrhs, double* sc, const double* rv, const int* active)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs || !active[c]) return;
    double* s = sc + c * BS;
    s[2] = s[0] / rv[c];
}
__global__ void k_bicg_omega(int nrhs, double* sc, const double* ts, const double* tt, const int* active)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs || !active[c]) return;
    double* s = sc + c * BS;
    s[3] = (tt[c] != 0.0) ? ts[c] / tt[c] : 0.0;
}
// p = r + beta (p - omega v)
__global__ void k_bicg_p(double* p, const double* r, const double* v, const double* sc, long long ld, long long n,
                         const int* active)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= n || !active[c]) return;
    const double* s = sc + c * BS;
    const long long k = c * ld + i;
    p[k] = r[k] + s[4] * (p[k] - s[3] * v[k]);
}
// s = r - alpha v  (into sv)
__global__ void k_bicg_s(double* sv, const double* r, const double* v, const double* sc, long long ld, long long n,
                         const int* active)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= n || !active[c]) return;
    const long long k = c * ld + i;
    sv[k] = r[k] - sc[c * BS + 2] * v[k];
}
// x += alpha p + omega s ; r = s - omega t
__global__ void k_bicg_xr(double* x, double* r, const double* p, const double* sv, const double* t, const double* sc,
                          long long ld, long long n, const int* active, int final_half)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= n || !active[c]) return;
    const double* s = sc + c * BS;
    const long long k = c * ld + i;
    if (final_half) {   // converged on the half step: x += alpha p
        x[k] += s[2] * p[k];
        return;
    }
    x[k] += s[2] * p[k] + s[3] * sv[k];
    r[k] = sv[k] - s[3] * t[k];
}

__global__ void k_copy_rho(int nrhs, double* sc, const double* rho, const int* active)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nrhs || !active[c]) return;
    sc[c * BS + 0] = rho[c];
}

void krylov_bicgstab(fde_ctx* h, fde_op* op, fde_lu* lu, const double* G, double* X, int nrhs, long long ldv,
                     const fde_solve_opts* o, fde_solve_report* rep)
{
    const long long n = op->n;
    const int maxit = o->maxiter > 0 ? o->maxiter : 500;
    const double tol = o->tol > 0 ? o->tol : 1e-13;
    cudaStream_t s = h->stream;
    DBuf<double> r, rh, p, v, sv, t, tmp, sc, d1, d2;
    DBuf<int> active;
    const size_t sz = (size_t)nrhs * ldv;
    r.alloc(sz); rh.alloc(sz); p.alloc(sz); v.alloc(sz); sv.alloc(sz); t.alloc(sz); tmp.alloc(sz);
    sc.alloc((size_t)nrhs * BS); d1.alloc(nrhs); d2.alloc(nrhs);
    active.alloc(nrhs);
    FDE_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * sz, s));
    p.zero(s); v.zero(s); sv.zero(s); t.zero(s); r.zero(s);
    const dim3 gv((unsigned)ceil_div(n, KB), (unsigned)nrhs);
    // r0 = A~^{-1} G
    if (lu) precond_apply_internal(h, lu, G, ldv, r.p, ldv, nrhs);
    else FDE_CUDA(cudaMemcpyAsync(r.p, G, sizeof(double) * sz, cudaMemcpyDeviceToDevice, s));
    FDE_CUDA(cudaMemcpyAsync(rh.p, r.p, sizeof(double) * sz, cudaMemcpyDeviceToDevice, s));
    k_norms<<<nrhs, KB, 0, s>>>(r.p, ldv, n, d1.p);
    FDE_CHECK_LAUNCH();
    std::vector<double> bn(nrhs), nr(nrhs), relres(nrhs, 1.0);
    FDE_CUDA(cudaMemcpyAsync(bn.data(), d1.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
    FDE_CUDA(cudaStreamSynchronize(s));
    std::vector<int> act(nrhs);
    std::vector<double> sc_h((size_t)nrhs * BS);
    for (int c = 0; c < nrhs; ++c) {
        if (!std::isfinite(bn[c])) fde_fail(FDE_EBREAKDOWN, "BiCGSTAB: non-finite (preconditioned) right-hand side");
        act[c] = bn[c] > 0.0;
        relres[c] = bn[c] > 0.0 ? 1.0 : 0.0;
        double* q = &sc_h[(size_t)c * BS];
        q[0] = q[1] = q[2] = q[3] = 1.0; q[4] = 0.0; q[5] = 0.0;
    }
    sc.upload(sc_h.data(), sc_h.size(), s);
    active.upload(act.data(), nrhs, s);
    int it = 0, mv = 0;
    auto apply = [&](const double* in, double* out) {
        if (lu) {
            op_apply_internal(h, op, in, ldv, tmp.p, ldv, nrhs, o->path);
            precond_apply_internal(h, lu, tmp.p, ldv, out, ldv, nrhs);
        } else {
            op_apply_internal(h, op, in, ldv, out, ldv, nrhs, o->path);
        }
        ++mv;
    };
    while (it < maxit) {
        int nact = 0;
        for (int c = 0; c < nrhs; ++c) nact += act[c];
        if (!nact) break;
        ++it;
        // rho = <rh, r>; beta
        k_dot_cols<<<nrhs, KB, 0, s>>>(rh.p, ldv, r.p, ldv, n, d1.p);
        FDE_CHECK_LAUNCH();
        k_copy_rho<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, sc.p, d1.p, active.p);
        FDE_CHECK_LAUNCH();
        k_bicg_beta<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, sc.p, active.p);
        FDE_CHECK_LAUNCH();
        k_bicg_p<<<gv, KB, 0, s>>>(p.p, r.p, v.p, sc.p, ldv, n, active.p);
        FDE_CHECK_LAUNCH();
        apply(p.p, v.p);
        k_dot_cols<<<nrhs, KB, 0, s>>>(rh.p, ldv, v.p, ldv, n, d1.p);
        FDE_CHECK_LAUNCH();
        k_bicg_alpha<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, sc.p, d1.p, active.p);
        FDE_CHECK_LAUNCH();
        k_bicg_s<<<gv, KB, 0, s>>>(sv.p, r.p, v.p, sc.p, ldv, n, active.p);
        FDE_CHECK_LAUNCH();
        k_norms<<<nrhs, KB, 0, s>>>(sv.p, ldv, n, d2.p);
        FDE_CHECK_LAUNCH();
        FDE_CUDA(cudaMemcpyAsync(nr.data(), d2.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
        FDE_CUDA(cudaStreamSynchronize(s));
        std::vector<int> half(nrhs, 0);
        bool anyhalf = false;
        for (int c = 0; c < nrhs; ++c)
            if (act[c] && nr[c] <= tol * bn[c]) { half[c] = 1; anyhalf = true; }
        if (anyhalf) {
            DBuf<int> hm;
            hm.upload(half.data(), nrhs, s);
            k_bicg_xr<<<gv, KB, 0, s>>>(X, r.p, p.p, sv.p, t.p, sc.p, ldv, n, hm.p, 1);
            FDE_CHECK_LAUNCH();
            FDE_CUDA(cudaStreamSynchronize(s));
            for (int c = 0; c < nrhs; ++c)
                if (half[c]) { act[c] = 0; relres[c] = nr[c] / bn[c]; }
            active.upload(act.data(), nrhs, s);
        }
        apply(sv.p, t.p);
        k_dot_cols<<<nrhs, KB, 0, s>>>(t.p, ldv, sv.p, ldv, n, d1.p);
        FDE_CHECK_LAUNCH();
        k_dot_cols<<<nrhs, KB, 0, s>>>(t.p, ldv, t.p, ldv, n, d2.p);
        FDE_CHECK_LAUNCH();
        k_bicg_omega<<<ceil_div(nrhs, 64), 64, 0, s>>>(nrhs, sc.p, d1.p, d2.p, active.p);
        FDE_CHECK_LAUNCH();
        k_bicg_xr<<<gv, KB, 0, s>>>(X, r.p, p.p, sv.p, t.p, sc.p, ldv, n, active.p, 0);
        FDE_CHECK_LAUNCH();
        k_norms<<<nrhs, KB, 0, s>>>(r.p, ldv, n, d1.p);
        FDE_CHECK_LAUNCH();
        FDE_CUDA(cudaMemcpyAsync(nr.data(), d1.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
        FDE_CUDA(cudaStreamSynchronize(s));
        for (int c = 0; c < nrhs; ++c) {
            if (!act[c]) continue;
            relres[c] = nr[c] / bn[c];
            if (!(nr[c] == nr[c])) fde_fail(FDE_EBREAKDOWN, "BiCGSTAB: NaN residual (breakdown)");
            if (relres[c] <= tol) act[c] = 0;
        }
        active.upload(act.data(), nrhs, s);
    }
    int conv = 0;
    double worst = 0;
    for (int c = 0; c < nrhs; ++c) {
        if (relres[c] <= tol) ++conv;
        worst = std::max(worst, relres[c]);
    }
    rep->iterations = it;
    rep->matvecs = mv;
    rep->converged = conv;
    rep->relres = worst;
    rep->relres_true = -1.0;
}

