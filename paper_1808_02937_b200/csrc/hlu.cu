// hlu_factor / precond_apply: H-LU of A~ = L_H U_H in H format on the block tree
// of the H-matrix (Fig. fig:HLU), and the hierarchical
// forward/backward substitutions L_H y = r, U_H z = y.
//
// Formatted arithmetic (Boerm et al. §5.2.3, cited at PAPER.md:606), reading A12:
//   LU(A)  = LU(A00); A01 <- L00^{-1} A01; A10 <- A10 U00^{-1};
//            A11 <- A11 - A10 A01 (truncated); LU(A11)
// Low-rank sums are truncated to sigma_i > tol * sigma_1 (tol = 0: exact, the
// factors are then the exact LU up to rounding).  No pivoting: the symmetric
// part of A is positive definite (Theorem 2.1); a zero or
// non-finite pivot is reported as FDE_ESINGULAR_PIVOT.
//
// The host walks the block tree and issues device work; every arithmetic step
// (dense LU of the leaves, triangular solves, GEMMs, Gram matrices, the small
// Jacobi eigen-solves of the truncation) is a CUDA kernel.  The truncated rank
// is the only value read back (one pinned word per truncation).
#include <cmath>
#include <cstring>

#include "hlu.h"

// --------------------------------------------------------------- kernels
#define GT 64   // GEMM tile
#define GK 16

// C[m x n] = alpha op(A) op(B) + beta C, column-major, op = N | T
__global__ void __launch_bounds__(256) k_gemm(int m, int n, int k, double alpha, const double* __restrict__ A,
                                             long long lda, int ta, const double* __restrict__ B, long long ldb,
                                             int tb, double beta, double* __restrict__ C, long long ldc)
{
    __shared__ double sA[GK][GT + 1];
    __shared__ double sB[GK][GT + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 16 x 16 threads, 4x4 micro tile
    const int m0 = blockIdx.x * GT, n0 = blockIdx.y * GT;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < k; k0 += GK) {
        for (int t = threadIdx.x; t < GK * GT; t += 256) {
            const int kk = t / GT, mm = t - kk * GT;   // for A tile: (mm, kk)
            const int gi = m0 + mm, gk = k0 + kk;
            double va = 0.0;
            if (gi < m && gk < k) va = ta ? A[(long long)gi * lda + gk] : A[(long long)gk * lda + gi];
            sA[kk][mm] = va;
            const int gj = n0 + mm;
            double vb = 0.0;
            if (gj < n && gk < k) vb = tb ? B[(long long)gk * ldb + gj] : B[(long long)gj * ldb + gk];
            sB[kk][mm] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sA[kk][tx + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sB[kk][ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gi = m0 + tx + 16 * i, gj = n0 + ty + 16 * j;
            if (gi < m && gj < n) {
                double* c = C + (long long)gj * ldc + gi;
                *c = alpha * acc[i][j] + (beta == 0.0 ? 0.0 : beta * *c);
            }
        }
}

// in-place LU without pivoting of an m x m column-major block (one CTA)
__global__ void k_dense_lu(double* D, int m, long long ld, int* bad)
{
    __shared__ double piv;
    for (int kk = 0; kk < m; ++kk) {
        if (threadIdx.x == 0) {
            piv = D[(long long)kk * ld + kk];
            if (!(fabs(piv) > 0.0) || !isfinite(piv)) *bad = 1;
        }
        __syncthreads();
        const double p = piv;
        for (int i = kk + 1 + threadIdx.x; i < m; i += blockDim.x) D[(long long)kk * ld + i] /= p;
        __syncthreads();
        const int rem = m - kk - 1;
        for (int t = threadIdx.x; t < rem * rem; t += blockDim.x) {
            const int i = kk + 1 + t % rem, j = kk + 1 + t / rem;
            D[(long long)j * ld + i] -= D[(long long)kk * ld + i] * D[(long long)j * ld + kk];
        }
        __syncthreads();
    }
}

// triangular solves of a dense leaf factor, one warp per right-hand-side column;
// rows are distributed round-robin over the lanes (m <= 32*TR)
#define TR 24
// mode 0: X <- L^{-1} X (unit lower of D) ; 1: X <- U^{-1} X (upper of D) ; 2: X <- U^{-T} X
__global__ void k_leaf_trsm(const double* __restrict__ D, int m, long long ld, double* X, long long ldx, int ncols,
                            int mode)
{
    const int lane = threadIdx.x & 31;
    const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (col >= ncols) return;
    double* x = X + (long long)col * ldx;
    double r[TR];
    const int nr = (m + 31) / 32;
#pragma unroll
    for (int t = 0; t < TR; ++t) r[t] = (t < nr && t * 32 + lane < m) ? x[t * 32 + lane] : 0.0;
    if (mode == 0 || mode == 2) {
        for (int i = 0; i < m; ++i) {
            const int ti = i >> 5, li = i & 31;
            double xi = 0.0;
#pragma unroll
            for (int t = 0; t < TR; ++t)
                if (t == ti) xi = r[t];
            xi = __shfl_sync(0xffffffffu, xi, li);
            if (mode == 2) xi /= D[(long long)i * ld + i];
            if (lane == li) {
#pragma unroll
                for (int t = 0; t < TR; ++t)
                    if (t == ti) r[t] = xi;
            }
#pragma unroll
            for (int t = 0; t < TR; ++t) {
                const int row = t * 32 + lane;
                if (t < nr && row > i && row < m) {
                    const double l = (mode == 0) ? D[(long long)i * ld + row] : D[(long long)row * ld + i];
                    r[t] = fma(-l, xi, r[t]);
                }
            }
        }
    } else {
        for (int i = m - 1; i >= 0; --i) {
            const int ti = i >> 5, li = i & 31;
            double xi = 0.0;
#pragma unroll
            for (int t = 0; t < TR; ++t)
                if (t == ti) xi = r[t];
            xi = __shfl_sync(0xffffffffu, xi, li);
            xi /= D[(long long)i * ld + i];
            if (lane == li) {
#pragma unroll
                for (int t = 0; t < TR; ++t)
                    if (t == ti) r[t] = xi;
            }
#pragma unroll
            for (int t = 0; t < TR; ++t) {
                const int row = t * 32 + lane;
                if (t < nr && row < i) r[t] = fma(-D[(long long)i * ld + row], xi, r[t]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < TR; ++t)
        if (t < nr && t * 32 + lane < m) x[t * 32 + lane] = r[t];
}

// B (n x m) = A^T (A: m x n), column-major
__global__ void k_transpose(const double* A, long long lda, int m, int n, double* B, long long ldb)
{
    __shared__ double t[32][33];
    const int bi = blockIdx.x * 32, bj = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int i = bi + threadIdx.x, j = bj + y;
        t[y][threadIdx.x] = (i < m && j < n) ? A[(long long)j * lda + i] : 0.0;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int j = bj + threadIdx.x, i = bi + y;
        if (i < m && j < n) B[(long long)i * ldb + j] = t[threadIdx.x][y];
    }
}

__global__ void k_copy2d(const double* A, long long lda, int m, int n, double* B, long long ldb, double alpha)
{
    const long long tot = (long long)m * n;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % m), j = (int)(t / m);
        B[(long long)j * ldb + i] = alpha * A[(long long)j * lda + i];
    }
}

__global__ void k_eye(double* B, long long ldb, int m)
{
    const long long tot = (long long)m * m;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % m), j = (int)(t / m);
        B[(long long)j * ldb + i] = (i == j) ? 1.0 : 0.0;
    }
}

// ---- truncation core: parallel cyclic Jacobi on symmetric matrices in smem
// A (n x n, ld n) -> eigenvalues on the diagonal, V eigenvectors (columns).
__device__ void cta_jacobi(double* A, double* V, int n, int* pairs)
{
    // n even (caller pads)
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) V[t] = ((t % n) == (t / n)) ? 1.0 : 0.0;
    __shared__ double cs[128], sn[128];
    __shared__ int conv;
    const int half = n / 2;
    for (int sweep = 0; sweep < 30; ++sweep) {
        if (threadIdx.x == 0) conv = 1;
        __syncthreads();
        for (int round = 0; round < n - 1; ++round) {
            // tournament pairing: player 0 fixed, others rotate
            for (int k = threadIdx.x; k < half; k += blockDim.x) {
                int a = (k == 0) ? 0 : 1 + ((k - 1 + round) % (n - 1));
                int b = 1 + ((n - 2 - k + round) % (n - 1));
                int p = min(a, b), q = max(a, b);
                pairs[2 * k] = p;
                pairs[2 * k + 1] = q;
                const double app = A[p * n + p], aqq = A[q * n + q], apq = A[q * n + p];
                double c = 1.0, s = 0.0;
                if (fabs(apq) > 1e-300 && fabs(apq) > 1e-17 * sqrt(fabs(app * aqq))) {
                    conv = 0;
                    const double tau = (aqq - app) / (2.0 * apq);
                    const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    c = 1.0 / sqrt(1.0 + tt * tt);
                    s = tt * c;
                }
                cs[k] = c;
                sn[k] = s;
            }
            __syncthreads();
            // A <- A J (columns p,q), V <- V J
            for (int t = threadIdx.x; t < half * n; t += blockDim.x) {
                const int k = t / n, i = t - k * n;
                const int p = pairs[2 * k], q = pairs[2 * k + 1];
                const double c = cs[k], s = sn[k];
                const double aip = A[p * n + i], aiq = A[q * n + i];
                A[p * n + i] = c * aip - s * aiq;
                A[q * n + i] = s * aip + c * aiq;
                const double vip = V[p * n + i], viq = V[q * n + i];
                V[p * n + i] = c * vip - s * viq;
                V[q * n + i] = s * vip + c * viq;
            }
            __syncthreads();
            // A <- J^T A (rows p,q)
            for (int t = threadIdx.x; t < half * n; t += blockDim.x) {
                const int k = t / n, j = t - k * n;
                const int p = pairs[2 * k], q = pairs[2 * k + 1];
                const double c = cs[k], s = sn[k];
                const double apj = A[j * n + p], aqj = A[j * n + q];
                A[j * n + p] = c * apj - s * aqj;
                A[j * n + q] = s * apj + c * aqj;
            }
            __syncthreads();
        }
        if (conv) break;
    }
}

// Given Gram matrices Gu = U^T U and Gv = V^T V (k x k), produce transforms
// Tu, Tv (k x r) with U Tu (V Tv)^T the rank-r truncation of U V^T,
// r = #{sigma_i > tol sigma_1} (capped by rmax).  Works in smem, one CTA.
__global__ void __launch_bounds__(256) k_trunc_core(const double* Gu, const double* Gv, int k, double tol, int rmax,
                                                   double* Tu, double* Tv, int* rank_out, double* scratch)
{
    double* sm = scratch;
    const int n = (k + 1) & ~1;   // even
    double* A = sm;
    double* Eu = A + n * n;
    double* Ev = Eu + n * n;
    double* C = Ev + n * n;
    double* X = C + n * n;
    double* lu = X + n * n;       // n
    double* lv = lu + n;          // n
    int* pairs = (int*)(lv + n);  // n
    // eigen(Gu)
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int i = t % n, j = t / n;
        A[t] = (i < k && j < k) ? Gu[j * k + i] : (i == j ? 0.0 : 0.0);
    }
    __syncthreads();
    cta_jacobi(A, Eu, n, pairs);
    for (int t = threadIdx.x; t < n; t += blockDim.x) lu[t] = A[t * n + t];
    __syncthreads();
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int i = t % n, j = t / n;
        A[t] = (i < k && j < k) ? Gv[j * k + i] : 0.0;
    }
    __syncthreads();
    cta_jacobi(A, Ev, n, pairs);
    for (int t = threadIdx.x; t < n; t += blockDim.x) lv[t] = A[t * n + t];
    __syncthreads();
    // sqrt of the retained eigenvalues (drop <= 1e-14 max: below the Gram precision)
    __shared__ double mu, mv;
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int i = 0; i < n; ++i) { a = fmax(a, lu[i]); b = fmax(b, lv[i]); }
        mu = a;
        mv = b;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        lu[t] = (lu[t] > 1e-14 * mu) ? sqrt(lu[t]) : 0.0;
        lv[t] = (lv[t] > 1e-14 * mv) ? sqrt(lv[t]) : 0.0;
    }
    __syncthreads();
    // C = Ru Rv^T, Ru = diag(lu) Eu^T, Rv = diag(lv) Ev^T -> C_ij = lu_i lv_j (Eu^T Ev)_ij
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int i = t % n, j = t / n;
        double s = 0.0;
        for (int q = 0; q < n; ++q) s = fma(Eu[i * n + q], Ev[j * n + q], s);
        C[j * n + i] = lu[i] * lv[j] * s;
    }
    __syncthreads();
    // M = C C^T -> eigen -> X (left singular vectors), sigma^2
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int i = t % n, j = t / n;
        double s = 0.0;
        for (int q = 0; q < n; ++q) s = fma(C[q * n + i], C[q * n + j], s);
        A[j * n + i] = s;
    }
    __syncthreads();
    cta_jacobi(A, X, n, pairs);
    __syncthreads();
    // order singular values descending (selection, one thread)
    __shared__ int ord[256];
    __shared__ int r_sh;
    if (threadIdx.x == 0) {
        for (int i = 0; i < n; ++i) ord[i] = i;
        for (int i = 0; i < n; ++i) {
            int b = i;
            for (int j = i + 1; j < n; ++j)
                if (A[ord[j] * n + ord[j]] > A[ord[b] * n + ord[b]]) b = j;
            int tmp = ord[i]; ord[i] = ord[b]; ord[b] = tmp;
        }
        const double s1 = sqrt(fmax(A[ord[0] * n + ord[0]], 0.0));
        int r = 0;
        for (int i = 0; i < n; ++i) {
            const double si = sqrt(fmax(A[ord[i] * n + ord[i]], 0.0));
            if (s1 > 0.0 && si > tol * s1 && si > 1e-15 * s1) ++r;
        }
        if (r > rmax) r = rmax;
        r_sh = r;
        *rank_out = r;
    }
    __syncthreads();
    const int r = r_sh;
    // Tu = Eu diag(1/lu) X_r Sigma_r  ;  Tv = Ev diag(1/lv) C^T X_r Sigma_r^{-1}
    for (int t = threadIdx.x; t < k * r; t += blockDim.x) {
        const int i = t % k, c = t / k;
        const int col = ord[c];
        const double sig = sqrt(fmax(A[col * n + col], 0.0));
        double su = 0.0, sv = 0.0;
        for (int q = 0; q < n; ++q) {
            // (diag(1/lu) X)_qc
            const double xq = X[col * n + q];
            if (lu[q] > 0.0) su = fma(Eu[q * n + i], xq / lu[q] * sig, su);
            // (C^T X)_qc
            double ctx = 0.0;
            for (int p = 0; p < n; ++p) ctx = fma(C[q * n + p], X[col * n + p], ctx);
            if (lv[q] > 0.0 && sig > 0.0) sv = fma(Ev[q * n + i], ctx / (lv[q] * sig), sv);
        }
        Tu[c * k + i] = su;
        Tv[c * k + i] = sv;
    }
}

// ---------------------------------------------------------------- host side
struct LBlk {
    int type;
    int64_t m, n, r0, c0;
    int child[4];
    double* D = nullptr;   // dense: m x n, ld m
    double* U = nullptr;   // lr: m x k, ld m
    double* V = nullptr;   // lr: n x k, ld n
    int k = 0;
};

struct fde_lu {
    fde_op* op = nullptr;
    fde_ctx* h = nullptr;
    HStruct S;
    std::vector<LBlk> B;
    double tol = 0;
    int max_rank = 0;
    int64_t stored = 0;
    double factor_ms = 0;
    int nops = 0;
    int rmax = 0;
    int* pinned = nullptr;
    DBuf<int> dflag;
    std::vector<double*> live;   // allocations to free
};

struct Mat {   // owned temporary (column-major)
    double* p = nullptr;
    int64_t rows = 0, cols = 0;
};

static double* lu_alloc(fde_lu* L, size_t words)
{
    if (words == 0) return nullptr;
    void* p = nullptr;
    FDE_CUDA(cudaMallocAsync(&p, words * sizeof(double), L->h->stream));
    return (double*)p;
}
static void lu_free(fde_lu* L, double* p)
{
    if (p) FDE_CUDA(cudaFreeAsync(p, L->h->stream));
}

static void gemm(fde_lu* L, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double beta, double* C, int64_t ldc)
{
    if (m <= 0 || n <= 0) return;
    if (k <= 0 && beta == 1.0) return;
    dim3 g((unsigned)ceil_div(m, GT), (unsigned)ceil_div(n, GT));
    k_gemm<<<g, 256, 0, L->h->stream>>>((int)m, (int)n, (int)std::max<int64_t>(k, 0), alpha, A, lda, ta, B, ldb, tb,
                                        beta, C, ldc);
    FDE_CHECK_LAUNCH();
    L->nops++;
}

static void copy2d(fde_lu* L, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb,
                   double alpha = 1.0)
{
    if (m <= 0 || n <= 0) return;
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(m * n, 256), 4096);
    k_copy2d<<<g, 256, 0, L->h->stream>>>(A, lda, (int)m, (int)n, B, ldb, alpha);
    FDE_CHECK_LAUNCH();
}

static void transpose(fde_lu* L, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb)
{
    dim3 g((unsigned)ceil_div(m, 32), (unsigned)ceil_div(n, 32));
    k_transpose<<<g, dim3(32, 8), 0, L->h->stream>>>(A, lda, (int)m, (int)n, B, ldb);
    FDE_CHECK_LAUNCH();
}

static void leaf_trsm(fde_lu* L, const LBlk& D, double* X, int64_t ldx, int64_t ncols, int mode)
{
    if (ncols <= 0 || D.m == 0) return;
    if (D.m > 32 * TR) fde_fail(FDE_EINVAL_PARAM, "H-LU: leaf larger than 768 dofs (reduce n_min)");
    const int wpb = 4;
    k_leaf_trsm<<<(unsigned)ceil_div(ncols, wpb), 32 * wpb, 0, L->h->stream>>>(D.D, (int)D.m, D.m, X, ldx, (int)ncols,
                                                                                mode);
    FDE_CHECK_LAUNCH();
    L->nops++;
}

// Y += alpha op(A) X  (X: cols(op A) x nc, Y: rows(op A) x nc)
static void hmul(fde_lu* L, int b, int trans, const double* X, int64_t ldx, int64_t nc, double alpha, double* Y,
                 int64_t ldy)
{
    const LBlk& A = L->B[b];
    if (nc <= 0) return;
    if (A.type == HB_DENSE) {
        if (trans)
            gemm(L, 1, 0, A.n, nc, A.m, alpha, A.D, A.m, X, ldx, 1.0, Y, ldy);
        else
            gemm(L, 0, 0, A.m, nc, A.n, alpha, A.D, A.m, X, ldx, 1.0, Y, ldy);
        return;
    }
    if (A.type == HB_LR) {
        if (A.k == 0) return;
        double* T = lu_alloc(L, (size_t)A.k * nc);
        if (!trans) {
            gemm(L, 1, 0, A.k, nc, A.n, 1.0, A.V, A.n, X, ldx, 0.0, T, A.k);
            gemm(L, 0, 0, A.m, nc, A.k, alpha, A.U, A.m, T, A.k, 1.0, Y, ldy);
        } else {
            gemm(L, 1, 0, A.k, nc, A.m, 1.0, A.U, A.m, X, ldx, 0.0, T, A.k);
            gemm(L, 0, 0, A.n, nc, A.k, alpha, A.V, A.n, T, A.k, 1.0, Y, ldy);
        }
        lu_free(L, T);
        return;
    }
    const LBlk &c00 = L->B[A.child[0]];
    const int64_t m0 = c00.m, n0 = c00.n;
    if (!trans) {
        hmul(L, A.child[0], 0, X, ldx, nc, alpha, Y, ldy);
        hmul(L, A.child[1], 0, X + n0, ldx, nc, alpha, Y, ldy);
        hmul(L, A.child[2], 0, X, ldx, nc, alpha, Y + m0, ldy);
        hmul(L, A.child[3], 0, X + n0, ldx, nc, alpha, Y + m0, ldy);
    } else {
        hmul(L, A.child[0], 1, X, ldx, nc, alpha, Y, ldy);
        hmul(L, A.child[2], 1, X + m0, ldx, nc, alpha, Y, ldy);
        hmul(L, A.child[1], 1, X, ldx, nc, alpha, Y + n0, ldy);
        hmul(L, A.child[3], 1, X + m0, ldx, nc, alpha, Y + n0, ldy);
    }
}

// X <- L^{-1} X (b diagonal block)
static void solve_L(fde_lu* L, int b, double* X, int64_t ldx, int64_t nc)
{
    const LBlk& A = L->B[b];
    if (A.type == HB_DENSE) return leaf_trsm(L, A, X, ldx, nc, 0);
    const int64_t m0 = L->B[A.child[0]].m;
    solve_L(L, A.child[0], X, ldx, nc);
    hmul(L, A.child[2], 0, X, ldx, nc, -1.0, X + m0, ldx);
    solve_L(L, A.child[3], X + m0, ldx, nc);
}

// X <- U^{-1} X
static void solve_U(fde_lu* L, int b, double* X, int64_t ldx, int64_t nc)
{
    const LBlk& A = L->B[b];
    if (A.type == HB_DENSE) return leaf_trsm(L, A, X, ldx, nc, 1);
    const int64_t m0 = L->B[A.child[0]].m;
    solve_U(L, A.child[3], X + m0, ldx, nc);
    hmul(L, A.child[1], 0, X + m0, ldx, nc, -1.0, X, ldx);
    solve_U(L, A.child[0], X, ldx, nc);
}

// X <- U^{-T} X
static void solve_UT(fde_lu* L, int b, double* X, int64_t ldx, int64_t nc)
{
    const LBlk& A = L->B[b];
    if (A.type == HB_DENSE) return leaf_trsm(L, A, X, ldx, nc, 2);
    const int64_t m0 = L->B[A.child[0]].m;
    solve_UT(L, A.child[0], X, ldx, nc);
    hmul(L, A.child[1], 1, X, ldx, nc, -1.0, X + m0, ldx);
    solve_UT(L, A.child[3], X + m0, ldx, nc);
}

// truncate [U (m x k), V (n x k)] -> new (U', V', r); consumes U,V
static void truncate(fde_lu* L, double*& U, double*& V, int64_t m, int64_t n, int& k)
{
    if (k == 0) return;
    if (L->tol == 0.0) {   // exact formatted arithmetic: keep every column
        L->max_rank = std::max(L->max_rank, k);
        return;
    }
    if (k > 254) fde_fail(FDE_ERANK, "H-LU: low-rank sum wider than 254 columns before truncation");
    const int kk = k;
    double* G = lu_alloc(L, (size_t)2 * kk * kk);
    double* T = lu_alloc(L, (size_t)2 * kk * kk);
    gemm(L, 1, 0, kk, kk, m, 1.0, U, m, U, m, 0.0, G, kk);
    gemm(L, 1, 0, kk, kk, n, 1.0, V, n, V, n, 0.0, G + kk * kk, kk);
    const int ne = (kk + 1) & ~1;
    double* scr = lu_alloc(L, (size_t)(5 * ne * ne + 3 * ne + 8));
    k_trunc_core<<<1, 256, 0, L->h->stream>>>(G, G + kk * kk, kk, L->tol, L->rmax, T, T + kk * kk, L->dflag.p + 1,
                                              scr);
    FDE_CHECK_LAUNCH();
    L->nops++;
    FDE_CUDA(cudaMemcpyAsync(L->pinned, L->dflag.p + 1, sizeof(int), cudaMemcpyDeviceToHost, L->h->stream));
    FDE_CUDA(cudaStreamSynchronize(L->h->stream));
    const int r = *L->pinned;
    double* U2 = lu_alloc(L, (size_t)m * std::max(r, 1));
    double* V2 = lu_alloc(L, (size_t)n * std::max(r, 1));
    if (r > 0) {
        gemm(L, 0, 0, m, r, kk, 1.0, U, m, T, kk, 0.0, U2, m);
        gemm(L, 0, 0, n, r, kk, 1.0, V, n, T + kk * kk, kk, 0.0, V2, n);
    }
    lu_free(L, U);
    lu_free(L, V);
    lu_free(L, G);
    lu_free(L, T);
    lu_free(L, scr);
    U = U2;
    V = V2;
    k = r;
    L->max_rank = std::max(L->max_rank, k);
}

// C += U V^T (formatted); U: m x k (ldu), V: n x k (ldv); U, V not consumed
static void add_lr(fde_lu* L, int c, const double* U, int64_t ldu, const double* V, int64_t ldv, int k)
{
    if (k == 0) return;
    LBlk& C = L->B[c];
    if (C.type == HB_DENSE) {
        gemm(L, 0, 1, C.m, C.n, k, 1.0, U, ldu, V, ldv, 1.0, C.D, C.m);
        return;
    }
    if (C.type == HB_LR) {
        const int k2 = C.k + k;
        double* U2 = lu_alloc(L, (size_t)C.m * k2);
        double* V2 = lu_alloc(L, (size_t)C.n * k2);
        if (C.k) {
            copy2d(L, C.U, C.m, C.m, C.k, U2, C.m);
            copy2d(L, C.V, C.n, C.n, C.k, V2, C.n);
        }
        copy2d(L, U, ldu, C.m, k, U2 + C.m * C.k, C.m);
        copy2d(L, V, ldv, C.n, k, V2 + C.n * C.k, C.n);
        lu_free(L, C.U);
        lu_free(L, C.V);
        int kk = k2;
        truncate(L, U2, V2, C.m, C.n, kk);
        C.U = U2;
        C.V = V2;
        C.k = kk;
        return;
    }
    const int64_t m0 = L->B[C.child[0]].m, n0 = L->B[C.child[0]].n;
    add_lr(L, C.child[0], U, ldu, V, ldv, k);
    add_lr(L, C.child[1], U, ldu, V + n0, ldv, k);
    add_lr(L, C.child[2], U + m0, ldu, V, ldv, k);
    add_lr(L, C.child[3], U + m0, ldu, V + n0, ldv, k);
}

// A B as a low-rank pair (allocated, caller frees)
static void product_lr(fde_lu* L, int a, int b, double*& U, double*& V, int& k)
{
    const LBlk &A = L->B[a], &B = L->B[b];
    const int64_t m = A.m, n = B.n;
    if (A.type == HB_LR) {
        k = A.k;
        U = lu_alloc(L, (size_t)m * std::max(k, 1));
        V = lu_alloc(L, (size_t)n * std::max(k, 1));
        copy2d(L, A.U, A.m, m, k, U, m);
        if (k) {
            FDE_CUDA(cudaMemsetAsync(V, 0, sizeof(double) * n * k, L->h->stream));
            hmul(L, b, 1, A.V, A.n, k, 1.0, V, n);   // B^T Va
        }
        return;
    }
    if (B.type == HB_LR) {
        k = B.k;
        U = lu_alloc(L, (size_t)m * std::max(k, 1));
        V = lu_alloc(L, (size_t)n * std::max(k, 1));
        if (k) {
            FDE_CUDA(cudaMemsetAsync(U, 0, sizeof(double) * m * k, L->h->stream));
            hmul(L, a, 0, B.U, B.m, k, 1.0, U, m);   // A Ub
        }
        copy2d(L, B.V, B.n, n, k, V, n);
        return;
    }
    if (A.type == HB_HIER && B.type == HB_HIER) {
        // 2x2 block product, each quadrant a truncated sum, then agglomerated
        const int64_t m0 = L->B[A.child[0]].m, n0 = L->B[B.child[0]].n;
        double* Uq[4];
        double* Vq[4];
        int kq[4];
        int ktot = 0;
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) {
                double *u1, *v1, *u2, *v2;
                int k1, k2;
                product_lr(L, A.child[2 * i + 0], B.child[0 + j], u1, v1, k1);
                product_lr(L, A.child[2 * i + 1], B.child[2 + j], u2, v2, k2);
                const int64_t mi = L->B[A.child[2 * i]].m, nj = L->B[B.child[j]].n;
                int ks = k1 + k2;
                double* us = lu_alloc(L, (size_t)mi * std::max(ks, 1));
                double* vs = lu_alloc(L, (size_t)nj * std::max(ks, 1));
                copy2d(L, u1, mi, mi, k1, us, mi);
                copy2d(L, u2, mi, mi, k2, us + mi * k1, mi);
                copy2d(L, v1, nj, nj, k1, vs, nj);
                copy2d(L, v2, nj, nj, k2, vs + nj * k1, nj);
                lu_free(L, u1); lu_free(L, v1); lu_free(L, u2); lu_free(L, v2);
                truncate(L, us, vs, mi, nj, ks);
                Uq[2 * i + j] = us;
                Vq[2 * i + j] = vs;
                kq[2 * i + j] = ks;
                ktot += ks;
            }
        k = ktot;
        U = lu_alloc(L, (size_t)m * std::max(k, 1));
        V = lu_alloc(L, (size_t)n * std::max(k, 1));
        if (k) {
            FDE_CUDA(cudaMemsetAsync(U, 0, sizeof(double) * m * k, L->h->stream));
            FDE_CUDA(cudaMemsetAsync(V, 0, sizeof(double) * n * k, L->h->stream));
        }
        int off = 0;
        for (int q = 0; q < 4; ++q) {
            const int i = q / 2, j = q % 2;
            const int64_t mi = i ? m - m0 : m0, nj = j ? n - n0 : n0;
            copy2d(L, Uq[q], mi, mi, kq[q], U + (i ? m0 : 0) + m * off, m);
            copy2d(L, Vq[q], nj, nj, kq[q], V + (j ? n0 : 0) + n * off, n);
            off += kq[q];
            lu_free(L, Uq[q]);
            lu_free(L, Vq[q]);
        }
        truncate(L, U, V, m, n, k);
        return;
    }
    // dense involved (leaf cluster): dense product, then identity-factorised
    double* P = lu_alloc(L, (size_t)m * n);
    FDE_CUDA(cudaMemsetAsync(P, 0, sizeof(double) * m * n, L->h->stream));
    if (A.type == HB_DENSE && B.type == HB_DENSE) {
        gemm(L, 0, 0, m, n, A.n, 1.0, A.D, A.m, B.D, B.m, 0.0, P, m);
    } else if (A.type == HB_DENSE) {
        // P^T = B^T A^T
        double* At = lu_alloc(L, (size_t)A.n * m);
        transpose(L, A.D, A.m, A.m, A.n, At, A.n);
        double* Pt = lu_alloc(L, (size_t)n * m);
        FDE_CUDA(cudaMemsetAsync(Pt, 0, sizeof(double) * n * m, L->h->stream));
        hmul(L, b, 1, At, A.n, m, 1.0, Pt, n);
        transpose(L, Pt, n, n, m, P, m);
        lu_free(L, At);
        lu_free(L, Pt);
    } else {
        hmul(L, a, 0, B.D, B.m, n, 1.0, P, m);
    }
    if (m <= n) {
        k = (int)m;
        U = lu_alloc(L, (size_t)m * m);
        k_eye<<<64, 256, 0, L->h->stream>>>(U, m, (int)m);
        FDE_CHECK_LAUNCH();
        V = lu_alloc(L, (size_t)n * m);
        transpose(L, P, m, m, n, V, n);
        lu_free(L, P);
    } else {
        k = (int)n;
        U = P;
        V = lu_alloc(L, (size_t)n * n);
        k_eye<<<64, 256, 0, L->h->stream>>>(V, n, (int)n);
        FDE_CHECK_LAUNCH();
    }
    truncate(L, U, V, m, n, k);
}

__global__ void k_axpy2d(const double* A, long long lda, int m, int n, double* B, long long ldb)
{
    const long long tot = (long long)m * n;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % m), j = (int)(t / m);
        B[(long long)j * ldb + i] += A[(long long)j * lda + i];
    }
}

void lu_axpy2d(fde_lu* L, const double* A, int64_t lda, int64_t m, int64_t n, double* B, int64_t ldb)
{
    if (m <= 0 || n <= 0) return;
    k_axpy2d<<<(unsigned)std::min<int64_t>(ceil_div(m * n, 256), 4096), 256, 0, L->h->stream>>>(A, lda, (int)m, (int)n,
                                                                                               B, ldb);
    FDE_CHECK_LAUNCH();
}

// C <- C - A B
static void gemm_sub(fde_lu* L, int c, int a, int b)
{
    LBlk &C = L->B[c], &A = L->B[a], &B = L->B[b];
    if (A.type == HB_HIER && B.type == HB_HIER && C.type == HB_HIER) {
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                for (int k = 0; k < 2; ++k) gemm_sub(L, C.child[2 * i + j], A.child[2 * i + k], B.child[2 * k + j]);
        return;
    }
    if (C.type == HB_DENSE && A.type != HB_LR && B.type != HB_LR) {
        if (A.type == HB_DENSE && B.type == HB_DENSE) {
            gemm(L, 0, 0, C.m, C.n, A.n, -1.0, A.D, A.m, B.D, B.m, 1.0, C.D, C.m);
        } else if (A.type == HB_DENSE) {
            // C -= A B with A dense, B hierarchical:  (A B)^T = B^T A^T
            double* At = lu_alloc(L, (size_t)A.n * A.m);
            transpose(L, A.D, A.m, A.m, A.n, At, A.n);
            double* Pt = lu_alloc(L, (size_t)C.n * C.m);
            FDE_CUDA(cudaMemsetAsync(Pt, 0, sizeof(double) * C.n * C.m, L->h->stream));
            hmul(L, b, 1, At, A.n, A.m, -1.0, Pt, C.n);
            double* P = lu_alloc(L, (size_t)C.m * C.n);
            transpose(L, Pt, C.n, C.n, C.m, P, C.m);
            lu_axpy2d(L, P, C.m, C.m, C.n, C.D, C.m);
            lu_free(L, At);
            lu_free(L, Pt);
            lu_free(L, P);
        } else {
            hmul(L, a, 0, B.D, B.m, B.n, -1.0, C.D, C.m);
        }
        return;
    }
    double *U, *V;
    int k;
    product_lr(L, a, b, U, V, k);
    if (k) copy2d(L, U, C.m, C.m, k, U, C.m, -1.0);
    add_lr(L, c, U, C.m, V, C.n, k);
    lu_free(L, U);
    lu_free(L, V);
}

// B <- L^{-1} B (formatted), l diagonal block
static void trsm_L_blk(fde_lu* L, int l, int b)
{
    LBlk& B = L->B[b];
    if (B.type == HB_LR) {
        solve_L(L, l, B.U, B.m, B.k);
    } else if (B.type == HB_DENSE) {
        solve_L(L, l, B.D, B.m, B.n);
    } else {
        const LBlk& Lb = L->B[l];
        for (int j = 0; j < 2; ++j) {
            trsm_L_blk(L, Lb.child[0], B.child[j]);
            gemm_sub(L, B.child[2 + j], Lb.child[2], B.child[j]);
            trsm_L_blk(L, Lb.child[3], B.child[2 + j]);
        }
    }
}

// B <- B U^{-1} (formatted)
static void trsm_U_blk(fde_lu* L, int u, int b)
{
    LBlk& B = L->B[b];
    if (B.type == HB_LR) {
        solve_UT(L, u, B.V, B.n, B.k);
    } else if (B.type == HB_DENSE) {
        double* Bt = lu_alloc(L, (size_t)B.n * B.m);
        transpose(L, B.D, B.m, B.m, B.n, Bt, B.n);
        solve_UT(L, u, Bt, B.n, B.m);
        transpose(L, Bt, B.n, B.n, B.m, B.D, B.m);
        lu_free(L, Bt);
    } else {
        const LBlk& Ub = L->B[u];
        for (int i = 0; i < 2; ++i) {
            trsm_U_blk(L, Ub.child[0], B.child[2 * i]);
            gemm_sub(L, B.child[2 * i + 1], B.child[2 * i], Ub.child[1]);
            trsm_U_blk(L, Ub.child[3], B.child[2 * i + 1]);
        }
    }
}

static void hlu_rec(fde_lu* L, int a)
{
    LBlk& A = L->B[a];
    if (A.type == HB_DENSE) {
        if (A.m == 0) return;
        k_dense_lu<<<1, 512, 0, L->h->stream>>>(A.D, (int)A.m, A.m, L->dflag.p);
        FDE_CHECK_LAUNCH();
        L->nops++;
        return;
    }
    if (A.type != HB_HIER) fde_fail(FDE_EINVAL_PARAM, "H-LU: diagonal block is low rank");
    hlu_rec(L, A.child[0]);
    trsm_L_blk(L, A.child[0], A.child[1]);
    trsm_U_blk(L, A.child[0], A.child[2]);
    gemm_sub(L, A.child[3], A.child[2], A.child[1]);
    hlu_rec(L, A.child[3]);
}

fde_lu* hlu_build(fde_ctx* h, fde_hm* hm, double tol)
{
    fde_lu* L = new fde_lu();
    try {
        L->op = hm->op;
        L->h = h;
        L->S = hm->S;
        L->tol = tol;
        L->rmax = 254;
        FDE_CUDA(cudaMallocHost(&L->pinned, sizeof(int) * 4));
        L->dflag.alloc(4);
        L->dflag.zero(h->stream);
        FDE_CUDA(cudaEventRecord(h->ev0, h->stream));
        // copy the H-matrix into working blocks
        L->B.resize(L->S.bl.size());
        for (size_t b = 0; b < L->S.bl.size(); ++b) {
            const HBlock& hb = L->S.bl[b];
            LBlk& lb = L->B[b];
            lb.type = hb.type;
            lb.m = hb.m;
            lb.n = hb.n;
            lb.r0 = L->S.cl[hb.tau].r0;
            lb.c0 = L->S.cl[hb.sig].r0;
            for (int k = 0; k < 4; ++k) lb.child[k] = hb.child[k];
            if (hb.type == HB_DENSE) {
                lb.D = lu_alloc(L, (size_t)std::max<int64_t>(hb.m * hb.n, 1));
                copy2d(L, hm->dense.p + hb.off, hb.m, hb.m, hb.n, lb.D, hb.m);
            } else if (hb.type == HB_LR) {
                lb.k = hm->R;
                lb.U = lu_alloc(L, (size_t)hb.m * hm->R);
                lb.V = lu_alloc(L, (size_t)hb.n * hm->R);
                copy2d(L, hm->lr.p + hb.off, hb.m, hb.m, hm->R, lb.U, hb.m);
                copy2d(L, hm->lr.p + hb.off + hb.m * hb.kcap, hb.n, hb.n, hm->R, lb.V, hb.n);
                // compress the Taylor factors themselves (W_{.0} = 0, reading A11)
                int kk = lb.k;
                truncate(L, lb.U, lb.V, hb.m, hb.n, kk);
                lb.k = kk;
            }
        }
        hlu_rec(L, L->S.root);
        FDE_CUDA(cudaMemcpyAsync(L->pinned, L->dflag.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        FDE_CUDA(cudaEventRecord(h->ev1, h->stream));
        FDE_CUDA(cudaEventSynchronize(h->ev1));
        if (*L->pinned) fde_fail(FDE_ESINGULAR_PIVOT, "H-LU: zero or non-finite pivot in a leaf factorisation");
        float ms = 0;
        cudaEventElapsedTime(&ms, h->ev0, h->ev1);
        L->factor_ms = ms;
        L->stored = 0;
        for (auto& b : L->B) {
            if (b.type == HB_DENSE) L->stored += b.m * b.n;
            if (b.type == HB_LR) L->stored += (b.m + b.n) * b.k;
        }
    } catch (...) {
        hlu_destroy(L);
        throw;
    }
    return L;
}

void hlu_info(fde_lu* lu, fde_hlu_info* info)
{
    info->max_rank = lu->max_rank;
    info->stored_entries = lu->stored;
    info->factor_ms = lu->factor_ms;
    info->nops = lu->nops;
}

fde_op* hlu_operator(fde_lu* lu) { return lu->op; }

void hlu_destroy(fde_lu* L)
{
    if (!L) return;
    cudaStream_t s = L->h ? L->h->stream : nullptr;
    for (auto& b : L->B) {
        if (b.D) cudaFreeAsync(b.D, s);
        if (b.U) cudaFreeAsync(b.U, s);
        if (b.V) cudaFreeAsync(b.V, s);
    }
    if (s) cudaStreamSynchronize(s);
    if (L->pinned) cudaFreeHost(L->pinned);
    delete L;
}

// z = U^{-1} L^{-1} r (internal order; r may equal z)
void precond_apply_internal(fde_ctx* h, fde_lu* lu, const double* r, int64_t ldr, double* z, int64_t ldz, int nrhs)
{
    lu->h = h;
    const int pi = prof_begin(h, PROF_PRECOND, 0.0);
    if (r != z) FDE_CUDA(cudaMemcpy2DAsync(z, ldz * sizeof(double), r, ldr * sizeof(double), lu->S.n * sizeof(double),
                                           nrhs, cudaMemcpyDeviceToDevice, h->stream));
    solve_L(lu, lu->S.root, z, ldz, nrhs);
    solve_U(lu, lu->S.root, z, ldz, nrhs);
    prof_end(h, pi);
}

// test helper: the packed factors as a dense n x n matrix (internal order,
// column-major): strict lower part = L_H, upper part = U_H
void hlu_dense_internal(fde_ctx* h, fde_lu* L, double* out, int64_t ldo)
{
    L->h = h;
    for (auto& b : L->B) {
        if (b.type == HB_DENSE) {
            copy2d(L, b.D, b.m, b.m, b.n, out + b.c0 * ldo + b.r0, ldo);
        } else if (b.type == HB_LR) {
            if (b.k)
                gemm(L, 0, 1, b.m, b.n, b.k, 1.0, b.U, b.m, b.V, b.n, 0.0, out + b.c0 * ldo + b.r0, ldo);
            else
            {
                k_copy2d<<<64, 256, 0, h->stream>>>(out, 0, (int)b.m, (int)b.n, out + b.c0 * ldo + b.r0, ldo, 0.0);
                FDE_CHECK_LAUNCH();
            }
        }
    }
    FDE_CUDA(cudaStreamSynchronize(h->stream));
}

// test helper: one triangular solve on internal-order columns (which: 0 L^{-1}, 1 U^{-1}, 2 U^{-T})
void hlu_solve_debug(fde_ctx* h, fde_lu* L, double* X, int64_t ldx, int nrhs, int which)
{
    L->h = h;
    if (which == 0) solve_L(L, L->S.root, X, ldx, nrhs);
    if (which == 1) solve_U(L, L->S.root, X, ldx, nrhs);
    if (which == 2) solve_UT(L, L->S.root, X, ldx, nrhs);
    FDE_CUDA(cudaStreamSynchronize(h->stream));
}
