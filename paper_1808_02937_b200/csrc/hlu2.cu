// hlu_factor, leaf-ordered: the formatted H-LU of A~ (Fig.
// fig:HLU; arithmetic of Boerm et al. §5.2.3 cited at PAPER.md:606, reading A12)
// executed as a right-looking sweep over the leaf clusters, on the block
// partition of the H-matrix (blocks keep their H format: one dense array or one
// low-rank pair U V^T per block of the partition).
//
// For leaf k = 0 .. nl-1 (tiles (i, j) are leaf-cluster pairs, the block that
// owns a tile is its block of the partition):
//   1. LU of the diagonal tile (k, k) (dense leaf; no pivoting, Theorem 2.1)
//   2. panels:  A(k, j>k) <- L_kk^{-1} A(k, j)  (dense rows; U factor of a
//               low-rank block),  A(i>k, k) <- A(i, k) U_kk^{-1}  (dense columns;
//               V factor: V <- U_kk^{-T} V)
//   3. Schur complement A(i, j) -= A(i, k) A(k, j) for i, j > k: dense targets
//      are updated with GEMMs, low-rank targets receive the product as new
//      columns (low-rank times anything is low rank), grouped per operand
//   4. truncation of the low-rank sums to sigma_i > tol sigma_1 (formatted
//      addition), batched, when a block is about to be used as an operand or
//      its pending width would exceed TRUNC_KMAX.
// This is the same arithmetic as the recursive algorithm of hlu.cu (the LU of A~
// is unique: at tol = 0 both give the exact factors up to rounding); the order of
// the truncations differs.  Every step is a handful of batched launches whose
// descriptors are built once on the host (no host synchronisation inside).
//
// A low-rank block becomes dense (D = U V^T, exact) when a dense x dense product
// lands in it or when its width would exceed what a truncated block can hold
// (TRUNC_KMAX; in exact mode, tol = 0, half its smaller dimension).
// Requirements (else hlu_build uses the recursive algorithm): leaves of at most
// H2_MMAX dofs and dense diagonal leaf tiles.

#include <atomic>
#include <chrono>
#include <climits>
#include <memory>
#include <exception>
#include <mutex>
#include <thread>
#include <functional>
#include <cstdlib>
#include <set>
#include <cuda.h>   // (types of the green-context driver API; entry points via cudaGetDriverEntryPoint)

#define H2_MMAX 128
#define H2_STRIP 32
#ifndef H2_PCH
#define H2_PCH 16      // inverse-panel staging chunk (columns of op)
#endif
#define H2_CP_CHUNK 4096   // elements per copy CTA

struct H2Lu {
    double* D;
    long long ld;
    int m;
};
// lower-triangular solve on a strip of vectors:
//   mode 0: X (m x nvec, columns) <- L^{-1} X   (unit lower L of the packed LU T)
//   mode 1: X (m x nvec, columns) <- U^{-T} X   (U of the packed LU T)
//   mode 2: X (nvec x m, rows)    <- X U^{-1}
struct H2Panel {
    const double* T;
    long long ldt;
    double* X;
    long long ldx;
    int m, nvec, mode;
    const double* Ti;   // explicit inverse of the factor (L^{-1} for mode 0, U^{-1} else), or null
    long long ldi;
};
struct H2Term {
    const double* A;
    const double* B;
    long long lda, ldb;
    int k, ta, tb;
    double alpha;
};
struct H2Task {
    double* C;
    long long ldc;
    int m, n;
    double beta;
    int t_lo, t_hi;
};
struct H2Tile {
    int task, m0, n0;
};
struct H2Copy {   // kind 0: dst = alpha src, 1: dst = 0, 2: dst = I
    const double* src;
    long long lds;
    double* dst;
    long long ldd;
    int m, n, kind;
    double alpha;
};

// ----------------------------------------------------------------- kernels

__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// LU without pivoting of an m x m tile (m <= 128), right-looking in shared memory
// with all 512 threads: thread (ti, tj) updates rows k+1+ti+32a and columns
// k+1+tj+16b of the trailing matrix; the multipliers of column k are scaled one
// step late (nobody reads the column any more); one barrier per pivot.  The tile is
// padded to 128 x 128 with the identity (the factors of diag(A, I) are diag(L, I),
// diag(U, I)), so the leading dimension is a compile-time constant and no
// element needs a bounds check.  (Measured against blocked / register-resident
// variants in tools/mb_lu.cu: this one is the fastest, ~130 us for m = 128.)
__global__ void __launch_bounds__(512) k_h2_lu(const H2Lu* tk, int* bad)
{
    constexpr int LD = H2_MMAX + 1, M = H2_MMAX;
    extern __shared__ double lsm[];
    const H2Lu d = tk[blockIdx.x];
    const int m = d.m, tid = threadIdx.x, ti = tid & 31, tj = tid >> 5;
    if (g_h2_check && !h2_chk(d.D, ((long long)(m - 1) * d.ld + m) * 8, 30, m, 0)) return;
    double* S = lsm;
    __shared__ double rp[M];
    for (int t = tid; t < M * M; t += 512) {
        const int i = t & (M - 1), j = t / M;
        if (i < m && j < m) cp_async8(S + j * LD + i, d.D + (long long)j * d.ld + i);
        else S[j * LD + i] = (i == j) ? 1.0 : 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    if (tid == 0) {
        const double p0 = S[0];
        if (!(fabs(p0) > 0.0) || !isfinite(p0)) *bad = 1;
        rp[0] = 1.0 / p0;
    }
    __syncthreads();
    for (int k = 0; k < M - 1; ++k) {
        const double rpk = rp[k];
        if (k > 0 && tj == 0)
            for (int i = k + ti; i < M; i += 32) S[(k - 1) * LD + i] *= rp[k - 1];
        const int i0 = k + 1 + ti, j0 = k + 1 + tj;
        double* base = S + j0 * LD + i0;
        const double* colk = S + k * LD + i0;
        const double* rowk = S + j0 * LD + k;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            if (k + 1 + 32 * a < M) {   // warp-uniform
                const double l = (i0 + 32 * a < M) ? colk[32 * a] * rpk : 0.0;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (j0 + 16 * b < M && i0 + 32 * a < M) {
                        const double u = rowk[16 * b * LD];
                        base[16 * b * LD + 32 * a] = fma(-l, u, base[16 * b * LD + 32 * a]);
                    }
                }
            }
        }
        if (tid == 0) {   // (k+1, k+1) is updated by thread 0
            const double pn = S[(k + 1) * LD + k + 1];
            if (k + 1 < m && (!(fabs(pn) > 0.0) || !isfinite(pn))) *bad = 1;
            rp[k + 1] = 1.0 / pn;
        }
        __syncthreads();
    }
    if (tid == 0) S[(M - 2) * LD + M - 1] *= rp[M - 2];
    __syncthreads();
    for (int t = tid; t < m * m; t += 512) {
        const int i = t % m, j = t / m;
        d.D[(long long)j * d.ld + i] = S[j * LD + i];
    }
}

// The same LU with the tile in registers: thread (tr, tc) = (tid & 31, tid >> 5)
// owns rows tr + 32a (a < 4) and columns tc + 16b (b < 8), cyclically, so that
// for pivot j = 16 jj + tcol (jj unrolled) the owned row / column of the pivot
// have compile-time register indices (a = jj / 2, b = jj) and whole register
// rows / columns that are already eliminated are skipped at compile time.  Per
// pivot the owners publish row j and column j (raw, after the update of pivot
// j-1) in double-buffered shared vectors; one barrier; every thread forms the
// multipliers l_i = a_ij / a_jj of its rows and updates its trailing elements.
// Same arithmetic as k_h2_lu (l = a_ij * (1 / a_jj), a_ik - l u_jk as one fma).
__global__ void __launch_bounds__(512) k_h2_lu_reg(const H2Lu* tk, int* bad)
{
    constexpr int M = H2_MMAX;
    static_assert(M == 128, "register LU: 128 x 128 tile, 512 threads");
    __shared__ double rowb[2][M], colb[2][M], rpb[2];
    const H2Lu d = tk[blockIdx.x];
    const int m = d.m, tid = threadIdx.x, tr = tid & 31, tc = tid >> 5;
    if (g_h2_check && !h2_chk(d.D, ((long long)(m - 1) * d.ld + m) * 8, 30, m, 0)) return;
    double R[4][8];
#pragma unroll
    for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int i = tr + 32 * a, k = tc + 16 * b;
            R[a][b] = (i < m && k < m) ? d.D[(long long)k * d.ld + i] : (i == k ? 1.0 : 0.0);
        }
    int nbad = 0;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int aj = jj >> 1;   // register row of rows 32 aj .. 32 aj + 31
        for (int tcol = 0; tcol < 16; ++tcol) {
            const int j = 16 * jj + tcol, buf = j & 1;
            const int jr = j & 31;   // owner lane of row j
            // publish row j (owners: tr == jr) and column j (owner warp: tc == tcol)
            if (tr == jr) {
#pragma unroll
                for (int b = jj; b < 8; ++b) rowb[buf][tc + 16 * b] = R[aj][b];
                if (tc == tcol) {
                    const double p = R[aj][jj];
                    if (j < m && (!(fabs(p) > 0.0) || !isfinite(p))) nbad = 1;
                    rpb[buf] = rcp_nr(p);   // (MUFU reciprocal + 2 Newton steps: on the pivot chain)
                }
            }
            if (tc == tcol) {
#pragma unroll
                for (int a = aj; a < 4; ++a) colb[buf][tr + 32 * a] = R[a][jj];
            }
            __syncthreads();
            const double rp = rpb[buf];
            double l[4];
#pragma unroll
            for (int a = aj; a < 4; ++a) l[a] = colb[buf][tr + 32 * a] * rp;
            double u[8];
#pragma unroll
            for (int b = jj; b < 8; ++b) u[b] = rowb[buf][tc + 16 * b];
#pragma unroll
            for (int a = aj; a < 4; ++a) {
                const bool ra = (a > aj) || (tr + 32 * a > j);
#pragma unroll
                for (int b = jj; b < 8; ++b) {
                    const bool cb = (b > jj) || (tc > tcol);
                    if (ra && cb) R[a][b] = fma(-l[a], u[b], R[a][b]);
                }
                if (tc == tcol && ra) R[a][jj] = l[a];   // multipliers of column j
            }
        }
    }
    if (nbad) *bad = 1;
#pragma unroll
    for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int i = tr + 32 * a, k = tc + 16 * b;
            if (i < m && k < m) d.D[(long long)k * d.ld + i] = R[a][b];
        }
}

// One CTA per strip of <= 32 vectors.  The packed LU tile T (m x m) and the strip
// are staged in shared memory with asynchronous copies; T' (lower) is read from
// the staged tile: mode 0: T'[i][j] = L[i][j] = Ts[j ldT + i] (unit diagonal),
// modes 1, 2: T'[i][j] = U[j][i] = Ts[i ldT + j].
template <int MODE>
__device__ __forceinline__ double h2_tp(const double* Ts, int ldT, int i, int j)
{
    return MODE == 0 ? Ts[j * ldT + i] : Ts[i * ldT + j];
}

// panel as a product with the explicit inverse of the factor (computed on the
// LU stream right after the tile's LU): X <- Li X (mode 0), X <- Ui^T X (mode 1),
// X <- X Ui (mode 2, rows).  op is staged as Ts[q ldT + i] = op(i, q); thread
// (lane, w) computes rows lane + 32a and vectors w + 8u (a, u < 4).
template <int MODE>
__device__ void h2_panel_inv_body(const H2Panel& p, double* psm)
{
    // op is staged in chunks of H2_PCH columns, double-buffered (the next chunk's
    // copies are in flight while one is multiplied; small shared footprint: the
    // CTA has to fit beside the bulk-update GEMMs of the previous step)
    // strides = 4 (mod 16) doubles: the DMMA fragment loads (lane = 4 row + k, 16 lanes
    // per 128-byte wavefront) hit 16 distinct bank pairs (m + 1 = 129: up to 4-way conflicts)
    const int m = p.m, ldT = m + (20 - m % 16) % 16, ldB = ldT;
    double* Bs = psm;                 // vector c, element i at Bs[c * ldB + i]
    double* Ts = psm + H2_STRIP * ldB;   // Ts[qq * ldT + i] = op(i, q0 + qq)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nv = p.nvec;
    const bool full = (m == H2_MMAX) && (nv == H2_STRIP);   // (shift / mask index forms)
    if (MODE == 2) {
        if (full)
            for (int t = tid; t < H2_STRIP * H2_MMAX; t += 256) {
                const int c = t & (H2_STRIP - 1), i = t / H2_STRIP;
                cp_async8(Bs + c * ldB + i, p.X + (long long)i * p.ldx + c);
            }
        else
            for (int t = tid; t < nv * m; t += 256) {
                const int c = t % nv, i = t / nv;
                cp_async8(Bs + c * ldB + i, p.X + (long long)i * p.ldx + c);
            }
    } else {
        if (full)
            for (int t = tid; t < H2_STRIP * H2_MMAX; t += 256) {
                const int i = t & (H2_MMAX - 1), c = t / H2_MMAX;
                cp_async8(Bs + c * ldB + i, p.X + (long long)c * p.ldx + i);
            }
        else
            for (int t = tid; t < nv * m; t += 256) {
                const int i = t % m, c = t / m;
                cp_async8(Bs + c * ldB + i, p.X + (long long)c * p.ldx + i);
            }
    }
    // FP64 tensor cores (mma.sync m8n8k4): warp w owns rows wm..wm+31 and vectors
    // wn..wn+15 of the 128 x 32 output (4 x 2 fragments of 8 x 8)
    const int wm = (w & 3) * 32, wn = (w >> 2) * 16;
    double dacc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dacc[i][j][0] = dacc[i][j][1] = 0.0;
    auto stage = [&](int q0, double* Tb) {
        const int nq = min(H2_PCH, m - q0);
        if (m == H2_MMAX && nq == H2_PCH) {   // full chunk: compile-time index forms
#pragma unroll
            for (int u = 0; u < H2_PCH * H2_MMAX / 256; ++u) {
                const int t = tid + 256 * u;
                if (MODE == 0) {
                    const int i = t & (H2_MMAX - 1), qq = t / H2_MMAX;
                    cp_async8(Tb + qq * ldT + i, p.Ti + (long long)(q0 + qq) * p.ldi + i);
                } else {
                    const int qq = t & (H2_PCH - 1), i = t / H2_PCH;
                    cp_async8(Tb + qq * ldT + i, p.Ti + (long long)i * p.ldi + q0 + qq);
                }
            }
            return;
        }
        if (MODE == 0) {   // op(i, q) = Ti(i, q): columns q0.. of Ti
            for (int t = tid; t < nq * m; t += 256) {
                const int i = t % m, qq = t / m;
                cp_async8(Tb + qq * ldT + i, p.Ti + (long long)(q0 + qq) * p.ldi + i);
            }
        } else {           // op(i, q) = Ti(q, i): rows q0.. of Ti
            for (int t = tid; t < nq * m; t += 256) {
                const int qq = t % nq, i = t / nq;
                cp_async8(Tb + qq * ldT + i, p.Ti + (long long)i * p.ldi + q0 + qq);
            }
        }
    };
    stage(0, Ts);
    cp_async_commit_group();   // (with the vectors)
    for (int q0 = 0, c = 0; q0 < m; q0 += H2_PCH, ++c) {
        const int nq = min(H2_PCH, m - q0);
        double* Tc = Ts + (c & 1) * H2_PCH * ldT;
        if (q0 + H2_PCH < m) {
            stage(q0 + H2_PCH, Ts + ((c + 1) & 1) * H2_PCH * ldT);
            cp_async_commit_group();
            cp_async_wait_group<1>();
        } else {
            cp_async_wait_group<0>();
        }
        __syncthreads();
        // (rows >= m / vectors >= nv of the staging buffers are stale: they only
        // reach outputs that are not stored; k beyond the chunk is zeroed)
#pragma unroll
        for (int kk = 0; kk < H2_PCH; kk += 4) {
            const int kr = kk + (lane & 3);
            const bool kv = kr < nq;
            double a[4], b[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = kv ? Tc[kr * ldT + wm + i * 8 + (lane >> 2)] : 0.0;
#pragma unroll
            for (int j = 0; j < 2; ++j) b[j] = kv ? Bs[(wn + j * 8 + (lane >> 2)) * ldB + q0 + kr] : 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma(dacc[i][j][0], dacc[i][j][1], a[i], b[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int r = wm + i * 8 + (lane >> 2), cv = wn + j * 8 + 2 * (lane & 3) + hh;
                if (r < m && cv < nv) {
                    if (MODE == 2) p.X[(long long)r * p.ldx + cv] = dacc[i][j][hh];
                    else p.X[(long long)cv * p.ldx + r] = dacc[i][j][hh];
                }
            }
}

// Substitution panel: the 32-column block panels of T' are staged one at a time,
// double-buffered (~100 KB of shared memory instead of the whole 128 x 128 tile:
// the CTA then fits beside the bulk-update GEMMs and starts without waiting for
// an SM to drain).  Tb[q ldT + i] = T'(i, b0 + q) for the rows i >= b0 it needs.
template <int MODE>
__device__ void h2_panel_body(const H2Panel& p, double* psm)
{
    const int m = p.m, ldT = (m & 1) ? m + 2 : m + 1, ldB = ldT;
    double* Bs = psm;                         // vector c, element i at Bs[c * ldB + i]
    double* Tb = psm + H2_STRIP * ldB;        // two block panels of 32 columns
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nv = p.nvec;
    if (MODE == 2) {   // rows of X are the vectors
        for (int t = tid; t < nv * m; t += 256) {
            const int c = t % nv, i = t / nv;
            cp_async8(Bs + c * ldB + i, p.X + (long long)i * p.ldx + c);
        }
    } else {
        for (int t = tid; t < nv * m; t += 256) {
            const int i = t % m, c = t / m;
            cp_async8(Bs + c * ldB + i, p.X + (long long)c * p.ldx + i);
        }
    }
    auto stage = [&](int bi, double* dst) {
        const int b0 = bi * 32, bs = min(32, m - b0), nr = m - b0;
        if (MODE == 0) {   // T'(i, j) = L[i][j] = T[j ldt + i]
            for (int t = tid; t < bs * nr; t += 256) {
                const int q = t / nr, i = b0 + t % nr;
                cp_async8(dst + q * ldT + i, p.T + (long long)(b0 + q) * p.ldt + i);
            }
        } else {           // T'(i, j) = U[j][i] = T[i ldt + j]
            for (int t = tid; t < bs * nr; t += 256) {
                const int q = t % bs, i = b0 + t / bs;
                cp_async8(dst + q * ldT + i, p.T + (long long)i * p.ldt + b0 + q);
            }
        }
    };
    const int nb = (m + 31) / 32;
    stage(0, Tb);
    cp_async_commit_group();   // (with the vectors)
    for (int bi = 0; bi < nb; ++bi) {
        const int b0 = bi * 32, bs = min(32, m - b0);
        const double* Tc = Tb + (bi & 1) * 32 * ldT;
        if (bi + 1 < nb) {
            stage(bi + 1, Tb + ((bi + 1) & 1) * 32 * ldT);
            cp_async_commit_group();
            cp_async_wait_group<1>();
        } else {
            cp_async_wait_group<0>();
        }
        __syncthreads();
        // diagonal block: warp w solves vectors w + 8u (u = 0..3) together (lane = row)
        {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = w + 8 * u;
                v[u] = (c < nv && lane < bs) ? Bs[c * ldB + b0 + lane] : 0.0;
            }
            for (int q = 0; q < bs; ++q) {
                const double tq = (lane > q && lane < bs) ? Tc[q * ldT + b0 + lane] : 0.0;
                const double rq = MODE == 0 ? 1.0 : 1.0 / Tc[q * ldT + b0 + q];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double y = __shfl_sync(0xffffffffu, v[u], q) * rq;
                    if (lane == q) v[u] = y;
                    else v[u] = fma(-tq, y, v[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = w + 8 * u;
                if (c < nv && lane < bs) Bs[c * ldB + b0 + lane] = v[u];
            }
        }
        __syncthreads();
        // trailing rows: B[i][c] -= sum_q T'[i][b0+q] Y[q][c]
        const int r0 = b0 + bs;
        if (r0 < m) {
            for (int t = tid; t < (m - r0) * nv; t += 256) {
                const int i = r0 + t % (m - r0), c = t / (m - r0);
                double s = Bs[c * ldB + i];
#pragma unroll 8
                for (int q = 0; q < bs; ++q) s = fma(-Tc[q * ldT + i], Bs[c * ldB + b0 + q], s);
                Bs[c * ldB + i] = s;
            }
        }
        __syncthreads();
    }
    if (MODE == 2) {
        for (int t = tid; t < nv * m; t += 256) {
            const int c = t % nv, i = t / nv;
            p.X[(long long)i * p.ldx + c] = Bs[c * ldB + i];
        }
    } else {
        for (int t = tid; t < nv * m; t += 256) {
            const int i = t % m, c = t / m;
            p.X[(long long)c * p.ldx + i] = Bs[c * ldB + i];
        }
    }
}

__global__ void __launch_bounds__(256) k_h2_panel(const H2Panel* P)
{
    pdl_trigger();
    extern __shared__ double psm[];
    const H2Panel p = P[blockIdx.x];
    pdl_wait();
    if (g_h2_check) {
        const long long ex = p.mode == 2 ? ((long long)(p.m - 1) * p.ldx + p.nvec) : ((long long)(p.nvec - 1) * p.ldx + p.m);
        if (!h2_chk(p.T, ((long long)(p.m - 1) * p.ldt + p.m) * 8, 20, p.m, p.mode) || !h2_chk(p.X, ex * 8, 21, p.nvec, p.mode))
            return;
    }
    if (p.Ti) {
        if (p.mode == 0) h2_panel_inv_body<0>(p, psm);
        else if (p.mode == 1) h2_panel_inv_body<1>(p, psm);
        else h2_panel_inv_body<2>(p, psm);
    } else {
        if (p.mode == 0) h2_panel_body<0>(p, psm);
        else if (p.mode == 1) h2_panel_body<1>(p, psm);
        else h2_panel_body<2>(p, psm);
    }
}

// grouped multi-term GEMM: every CTA owns a 64 x 64 tile of one task,
// C_tile = beta C_tile + sum_terms alpha op(A) op(B); terms in a fixed order.
// The (term, 16-deep slice) sequence of the tile runs through a 3-stage
// asynchronous-copy pipeline in shared memory (8-byte cp.async: any operand
// layout / transpose), so two slices are in flight while one is multiplied.
#ifndef H2G_ST
#define H2G_ST 3
#endif
#define H2G_TMAX 48
#ifndef H2G_EPI
#define H2G_EPI 2     // C elements loaded before they are stored in the GEMM epilogue
#endif
#ifndef H2C_B
#define H2C_B 8       // elements per thread loaded before they are stored in k_h2_copy
#endif
#ifndef H2G_PFC
#define H2G_PFC 0     // prefetch the C tile into L2 at the start of a GEMM tile
#endif
#ifndef H2G_MINB
#define H2G_MINB 4    // __launch_bounds__ minimum CTAs per SM of k_h2_gemm
#endif
#ifndef H2G_PAD
#define H2G_PAD 4     // row padding of the staged operand slices: 4 (mod 16) doubles, conflict-free fragment loads
#endif
#define H2G_SMEM(TM, TN) (H2G_ST * GK * ((TM) + (TN) + 2 * H2G_PAD) * (int)sizeof(double))
struct H2Cursor {   // position in the (term, slice) sequence of a tile
    int q, k0;
};
__device__ __forceinline__ void h2_next(const H2Term* terms, int t_hi, H2Cursor& c)
{
    c.k0 += GK;
    if (c.k0 >= terms[c.q].k) {
        c.k0 = 0;
        ++c.q;
        while (c.q < t_hi && terms[c.q].k <= 0) ++c.q;
    }
}
template <int TM, int TN>
__device__ __forceinline__ void h2_stage(const H2Term& T, int m0, int n0, int m, int n, int k0, double* sA, double* sB,
                                         bool stageB = true)
{
    // sA[kk][mm] (ld TM + 1), sB[kk][nn] (ld TN + 1); zero outside the operands
#pragma unroll
    for (int u = 0; u < (TM * GK + 255) / 256; ++u) {
        const int t = threadIdx.x + 256 * u;
        if (TM * GK < 256 && t >= TM * GK) break;
        int kk, mm;
        if (T.ta) { mm = t / GK; kk = t % GK; } else { kk = t / TM; mm = t % TM; }
        const int gi = m0 + mm, gk = k0 + kk;
        double* da = sA + kk * (TM + H2G_PAD) + mm;
        if (gi < m && gk < T.k) cp_async8(da, T.ta ? T.A + (long long)gi * T.lda + gk : T.A + (long long)gk * T.lda + gi);
        else *da = 0.0;
    }
    if (!stageB) return;
#pragma unroll
    for (int u = 0; u < (TN * GK + 255) / 256; ++u) {
        const int t = threadIdx.x + 256 * u;
        if (TN * GK < 256 && t >= TN * GK) break;
        int kk, nn;
        if (T.tb) { kk = t / TN; nn = t % TN; } else { nn = t / GK; kk = t % GK; }
        const int gj = n0 + nn, gk2 = k0 + kk;
        double* db = sB + kk * (TN + H2G_PAD) + nn;
        if (gj < n && gk2 < T.k) cp_async8(db, T.tb ? T.B + (long long)gk2 * T.ldb + gj : T.B + (long long)gj * T.ldb + gk2);
        else *db = 0.0;
    }
}

// warp grid of the DMMA path (8 x 8 fragments of mma.sync.m8n8k4.f64): WM x WN warps
template <int TM, int TN> struct H2Warps {
    static constexpr int WM = (TN == 16 && TM >= 128) ? 8 : (TM >= 32 ? 4 : 2);
    static constexpr int WN = (TN == 16 && TM >= 128) ? 1 : 2;
};
template <int TM, int TN, bool DM>
__device__ __forceinline__ void h2_gemm_tile(const H2Tile* tiles, int tile, const H2Task* tasks, const H2Term* terms)
{
    constexpr int RM = TM / 16, RN = TN / 16;   // register tile RM x RN per thread (16 x 16 threads)
    constexpr int WM = H2Warps<TM, TN>::WM, WN = H2Warps<TM, TN>::WN;
    constexpr int FM = TM / (8 * WM), FN = TN / (8 * WN);   // DMMA fragments per warp
    static_assert(FM >= 1 && FN >= 1 && WM * WN <= 8, "warp grid");
    extern __shared__ double gsm[];   // H2G_SMEM bytes: [stage] A slice, [stage] B slice
    double (*sA)[GK * (TM + H2G_PAD)] = reinterpret_cast<double (*)[GK * (TM + H2G_PAD)]>(gsm);
    double (*sB)[GK * (TN + H2G_PAD)] = reinterpret_cast<double (*)[GK * (TN + H2G_PAD)]>(gsm + H2G_ST * GK * (TM + H2G_PAD));
    __shared__ double sAlpha[H2G_ST];
    __shared__ H2Term sT[H2G_TMAX];   // the task's term descriptors (one global read each)
    const H2Tile tl = tiles[tile];
    const H2Task tk = tasks[tl.task];
    int nt = tk.t_hi - tk.t_lo;
    const H2Term* tm = terms + tk.t_lo;
    if (nt <= H2G_TMAX) {
        for (int q = threadIdx.x; q < nt; q += blockDim.x) sT[q] = terms[tk.t_lo + q];
        __syncthreads();
        tm = sT;
    }
    pdl_wait();   // (descriptors above; operands and C below may come from the previous kernel)
    // fused core (planner, rmax <= 16): the task W = V_c core carries the core
    // definition core = U_c[k]^T V_b[k] as a leading term (ta == 3: A = U_c[k],
    // B = V_b[k], k = rows of the sweep tile); the CTA forms the core itself in
    // shared memory (one K slice, 16 x 16) instead of a separate launch
    H2Term cdef;
    const bool coremode = (TN == 16) && nt == 2 && tm[0].ta == 3;
    if (coremode) {
        cdef = tm[0];
        ++tm;
        nt = 1;
    }
#if H2G_PFC
    if (tk.beta != 0.0) {   // C tile lines into L2 now, read in the epilogue
        const int mm = min(TM, tk.m - tl.m0), nn = min(TN, tk.n - tl.n0);
        const int lines = (mm * 8 + 127) / 128;   // 128-byte lines per column
        for (int t = threadIdx.x; t < lines * nn; t += blockDim.x) {
            const int j = t / lines, l = t - j * lines;
            const double* a = tk.C + (long long)(tl.n0 + j) * tk.ldc + tl.m0 + l * 16;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        }
    }
#endif
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = tl.m0, n0 = tl.n0, m = tk.m, n = tk.n;
    __shared__ int sbad;
    if (threadIdx.x == 0) sbad = 0;
    if (g_h2_check && threadIdx.x == 0) {
        // C: columns [n0, n0+64) rows [m0, m0+64) clipped
        const int mm = min(TM, m - m0), nn = min(TN, n - n0);
        if (mm > 0 && nn > 0) h2_chk(tk.C + (long long)n0 * tk.ldc + m0, ((long long)(nn - 1) * tk.ldc + mm) * 8, 1, m, n);
        for (int q = 0; q < nt; ++q) {
            const H2Term T = terms[tk.t_lo + q];
            if (T.k <= 0 || T.ta == 3) continue;
            // A: op(A) is m x k; stored (ta ? k x m : m x k) column-major with lda
            const long long ea = T.ta ? ((long long)(m0 + mm - 1) * T.lda + T.k) : ((long long)(T.k - 1) * T.lda + m0 + mm);
            const long long sa = T.ta ? (long long)m0 * T.lda : m0;
            h2_chk(T.A + sa, (ea - sa) * 8, 2, q, T.k);
            const long long eb = T.tb ? ((long long)(T.k - 1) * T.ldb + n0 + nn) : ((long long)(n0 + nn - 1) * T.ldb + T.k);
            const long long sb = T.tb ? n0 : (long long)n0 * T.ldb;
            h2_chk(T.B + sb, (eb - sb) * 8, 3, q, T.k);
        }
        sbad = g_h2_bad_flag;
    }
    __syncthreads();
    if (sbad) return;
    double acc[RM][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = 0.0;
    double dacc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dacc[i][j][0] = dacc[i][j][1] = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp % WM) * (TM / WM), wn = (warp / WM) * (TN / WN);
    const bool wact = warp < WM * WN;
    H2Cursor ld{0, -GK};   // next slice to load
    while (ld.q < nt && tm[ld.q].k <= 0) ++ld.q;
    ld.k0 = 0;
    int nslice = 0;
    for (int q = 0; q < nt; ++q) nslice += (tm[q].k + GK - 1) / GK;
    // prologue: stages 0 .. H2G_ST-2
#pragma unroll
    for (int st = 0; st < H2G_ST - 1; ++st) {
        if (st < nslice) {
            const H2Term& T = tm[ld.q];
            h2_stage<TM, TN>(T, m0, n0, m, n, ld.k0, sA[st], sB[st], !coremode);
            if (threadIdx.x == 0) sAlpha[st] = T.alpha;
            h2_next(tm, nt, ld);
        }
        cp_async_commit_group();
    }
    if (TN == 16 && TM * GK >= 2048 && H2G_ST >= 3 && coremode) {
        // U_c[k] (rows x kq) and V_b[k] (rows x n) -> sA[1], sA[2] as [col][row] (ld 129),
        // then core[kk][nn] = sum_r U[r][kk] V[r][nn] (fixed order) -> the B stage of slice 0
        const int rows = cdef.k, kq = tm[0].k;
        double* sU = sA[1];
        double* sV = sA[2];
        for (int t = threadIdx.x; t < rows * kq; t += blockDim.x) {
            const int r = t % rows, c = t / rows;
            cp_async8(sU + c * 129 + r, cdef.A + (long long)c * cdef.lda + r);
        }
        for (int t = threadIdx.x; t < rows * n; t += blockDim.x) {
            const int r = t % rows, c = t / rows;
            cp_async8(sV + c * 129 + r, cdef.B + (long long)c * cdef.ldb + r);
        }
        cp_async_commit_group();
        cp_async_wait_group<0>();
        __syncthreads();
        {
            const int kk = threadIdx.x & 15, nn = threadIdx.x >> 4;
            double v = 0.0;
            if (kk < kq && nn < n)
                for (int r = 0; r < rows; ++r) v = fma(sU[kk * 129 + r], sV[nn * 129 + r], v);
            sB[0][kk * (TN + H2G_PAD) + nn] = v;
        }
        __syncthreads();
    }
    for (int sl = 0; sl < nslice; ++sl) {
        cp_async_wait_group<H2G_ST - 2>();
        __syncthreads();
        // refill the stage consumed H2G_ST-1 slices ago
        const int nx = sl + H2G_ST - 1;
        if (nx < nslice) {
            const int st = nx % H2G_ST;
            const H2Term& T = tm[ld.q];
            h2_stage<TM, TN>(T, m0, n0, m, n, ld.k0, sA[st], sB[st]);
            if (threadIdx.x == 0) sAlpha[st] = T.alpha;
            h2_next(tm, nt, ld);
        }
        cp_async_commit_group();
        const int cs = sl % H2G_ST;
        const double* a_s = sA[cs];
        const double* b_s = sB[cs];
        const double al = sAlpha[cs];
        if (DM) {   // FP64 tensor cores: one mma per 8 x 8 x 4 block
            if (wact) {
#pragma unroll
                for (int kk = 0; kk < GK; kk += 4) {
                    double a[FM], b[FN];
                    const int kr = kk + (lane & 3);
#pragma unroll
                    for (int i = 0; i < FM; ++i) a[i] = al * a_s[kr * (TM + H2G_PAD) + wm + i * 8 + (lane >> 2)];
#pragma unroll
                    for (int j = 0; j < FN; ++j) b[j] = b_s[kr * (TN + H2G_PAD) + wn + j * 8 + (lane >> 2)];
#pragma unroll
                    for (int i = 0; i < FM; ++i)
#pragma unroll
                        for (int j = 0; j < FN; ++j) dmma(dacc[i][j][0], dacc[i][j][1], a[i], b[j]);
                }
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < GK; ++kk) {
                double a[RM], b[RN];
#pragma unroll
                for (int i = 0; i < RM; ++i) a[i] = al * a_s[kk * (TM + H2G_PAD) + tx + 16 * i];
#pragma unroll
                for (int j = 0; j < RN; ++j) b[j] = b_s[kk * (TN + H2G_PAD) + ty + 16 * j];
#pragma unroll
                for (int i = 0; i < RM; ++i)
#pragma unroll
                    for (int j = 0; j < RN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
        }
    }
    cp_async_wait_group<0>();
    // epilogue C = acc + beta C: the C values of a fragment row are all loaded before
    // any of them is stored (a load after a store to a possibly aliasing address
    // cannot be hoisted by the compiler: one global round trip per element otherwise)
    const bool rdc = tk.beta != 0.0;
    if (DM) {
        // batches of H2G_EPI (j, h) elements of one fragment row
        constexpr int NE = 2 * FN, EB = (H2G_EPI < NE) ? H2G_EPI : NE;
        if (wact)
#pragma unroll
            for (int i = 0; i < FM; ++i) {
                const int gi = m0 + wm + i * 8 + (lane >> 2);
#pragma unroll
                for (int e0 = 0; e0 < NE; e0 += EB) {
                    double cv[EB];
#pragma unroll
                    for (int e = 0; e < EB; ++e) {
                        const int j = (e0 + e) >> 1, h = (e0 + e) & 1;
                        const int gj = n0 + wn + j * 8 + 2 * (lane & 3) + h;
                        cv[e] = (rdc && gi < m && gj < n) ? tk.C[(long long)gj * tk.ldc + gi] : 0.0;
                    }
#pragma unroll
                    for (int e = 0; e < EB; ++e) {
                        const int j = (e0 + e) >> 1, h = (e0 + e) & 1;
                        const int gj = n0 + wn + j * 8 + 2 * (lane & 3) + h;
                        if (gi < m && gj < n) tk.C[(long long)gj * tk.ldc + gi] = dacc[i][j][h] + (rdc ? tk.beta * cv[e] : 0.0);
                    }
                }
            }
        return;
    }
#pragma unroll
    for (int i = 0; i < RM; ++i) {
        double cv[RN];
        const int gi = m0 + tx + 16 * i;
#pragma unroll
        for (int j = 0; j < RN; ++j) {
            const int gj = n0 + ty + 16 * j;
            cv[j] = (rdc && gi < m && gj < n) ? tk.C[(long long)gj * tk.ldc + gi] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < RN; ++j) {
            const int gj = n0 + ty + 16 * j;
            if (gi < m && gj < n) tk.C[(long long)gj * tk.ldc + gi] = acc[i][j] + (rdc ? tk.beta * cv[j] : 0.0);
        }
    }
}

// grid-stride over the tiles: a capped grid leaves SMs to the critical stream
template <int TM, int TN, bool DM>
__global__ void __launch_bounds__(256, (TM * TN > 4096) ? 2 : H2G_MINB) k_h2_gemm(const H2Tile* tiles, const H2Task* tasks, const H2Term* terms, int ntile)
{
    pdl_trigger();
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
        h2_gemm_tile<TM, TN, DM>(tiles, t, tasks, terms);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_h2_copy(const H2Copy* C)
{
    pdl_trigger();
    const H2Copy c = C[blockIdx.x];
    pdl_wait();
    const long long tot = (long long)c.m * c.n;
    if (g_h2_check) {
        bool ok = h2_chk(c.dst, ((long long)(c.n - 1) * c.ldd + c.m) * 8, 10, c.m, c.n);
        if (c.kind == 0) ok = ok && h2_chk(c.src, ((long long)(c.n - 1) * c.lds + c.m) * 8, 11, c.m, c.n);
        if (!ok) return;
    }
    // batches of 8 elements per thread: the 8 loads are issued before the 8 stores
    // (one global round trip per batch instead of one per element)
    constexpr int B = H2C_B;
    for (long long t0 = threadIdx.x; t0 < tot; t0 += (long long)B * blockDim.x) {
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const long long t = t0 + (long long)u * blockDim.x;
            const int i = (int)(t % c.m), j = (int)(t / c.m);
            if (t >= tot) v[u] = 0.0;
            else if (c.kind == 0) v[u] = c.src[(long long)j * c.lds + i];
            else if (c.kind == 1) v[u] = 0.0;
            else v[u] = (i == j) ? 1.0 : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const long long t = t0 + (long long)u * blockDim.x;
            if (t < tot) {
                const int i = (int)(t % c.m), j = (int)(t / c.m);
                c.dst[(long long)j * c.ldd + i] = c.kind == 0 ? c.alpha * v[u] : v[u];
            }
        }
    }
}

__global__ void k_h2_spin(long long us)   // (debug FDE_H2_HOLD_US)
{
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < (unsigned long long)us * 1000ull);
}

// ------------------------------------------------------------------ plan
// Pointers are resolved after the arena layout is known: a reference is
// (space, id, offset): space 0 = dense block id, 1 = U of block id, 2 = V of
// block id, 3 = step scratch, 4 = leaf inverse id (L^{-1}), 5 = (U^{-1}).
struct VRef {
    int sp, id;
    int64_t off;
};
struct VTerm {
    VRef A, B;
    int64_t lda, ldb;
    int k, ta, tb;
    double alpha;
};
// the terms of a task: one inline, the rest on the heap (most dense-update tasks
// have one term; a heap vector per task cost ~1.5 ms of host planning on c4)
struct VTermList {
    VTerm inl[1];
    int n = 0;
    int off = 1;   // list index of more[0] (0 once a whole vector was adopted)
    std::vector<VTerm> more;
    void push_back(const VTerm& t)
    {
        if (n < off) inl[n] = t;
        else more.push_back(t);
        ++n;
    }
    // take over a vector of terms without copying them (on an empty list)
    void adopt(std::vector<VTerm>&& v)
    {
        more = std::move(v);
        n = (int)more.size();
        off = 0;
    }
    size_t size() const { return (size_t)n; }
    const VTerm& operator[](int i) const { return i < off ? inl[i] : more[i - off]; }
    struct It {
        const VTermList* l;
        int i;
        const VTerm& operator*() const { return (*l)[i]; }
        It& operator++() { ++i; return *this; }
        bool operator!=(const It& o) const { return i != o.i; }
    };
    It begin() const { return {this, 0}; }
    It end() const { return {this, n}; }
};
struct VTask {
    VRef C;
    int64_t ldc;
    int m, n;
    double beta;
    VTermList terms;
};
struct VCopy {
    VRef src, dst;
    int64_t lds, ldd;
    int m, n, kind;
    double alpha;
};
struct VPanel {
    VRef T;     // packed LU of the diagonal tile (ld ldt)
    int64_t ldt;
    VRef X;
    int64_t ldx;
    int m, nvec, mode;
    VRef Ti{-1, 0, 0};   // its explicit inverse (see H2Panel), if computed
    int64_t ldi = 0;
};
struct VTrunc {
    int blk, k;
};
struct VStep {
    std::vector<VTrunc> trunc;      // panel operands of this step (before the panels)
    std::vector<VTrunc> trunc_ov;   // targets about to overflow (before this step's new columns)
    int lu_blk = -1;
    int64_t lu_off = 0;
    std::vector<VPanel> panel;
    std::vector<VPanel> npanel;          // the neighbour tiles (k+1, k), (k, k+1): on the LU stream
    std::vector<VTask> g0, g1, g2, g3;   // conversions to dense, cores, products, dense updates
    // dense-target updates recorded compactly by the plan and expanded into g3 when the
    // step is flattened (the expansion then overlaps the device; without deferral)
    struct DPair { int b, c; int64_t w, su, sv; int kcb, kcc; bool bl, cl; };
    std::vector<DPair> dpairs;
    std::vector<std::pair<int, int>> dts;   // (pair, dense target block)
    int sid = 0, mk = 0;
    std::vector<VTask> g3r;              // dense updates of tiles off row / column k+1 (lookahead stream)
    std::vector<char> g3crit;            // per g3 task: 2 tile (k+1, k+1), 1 row / column k+1 or (k+2, k+2), 0 rest
    std::vector<std::vector<VCopy>> cpr;    // new low-rank target columns, by round
    std::vector<VCopy> snap;                // operand factor snapshots (after the panels)
    std::vector<std::vector<VTrunc>> trmid; // truncations between rounds
    int64_t scratch = 0;
};

// Green contexts (SM partitions) for the H-LU sweep: the bulk dense updates on
// `nbulk` SMs, the binding chain (panels, products, truncations, new columns, LU)
// on the others, so the latency-bound chain kernels never share an SM with the
// long bulk-update CTAs.  Driver entry points through the runtime (no libcuda link).
static bool h2_green_streams(fde_ctx* h, int nbulk)
{
    if (h->green_n == nbulk) return true;
    if (h->green_n != 0) return false;   // (one partition per handle)
    typedef CUresult (*FGet)(CUdevice*, int);
    typedef CUresult (*FRes)(CUdevice, CUdevResource*, CUdevResourceType);
    typedef CUresult (*FSplit)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
    typedef CUresult (*FDesc)(CUdevResourceDesc*, CUdevResource*, unsigned);
    typedef CUresult (*FCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
    typedef CUresult (*FStream)(CUstream*, CUgreenCtx, unsigned, int);
    void *pg = nullptr, *pr = nullptr, *ps = nullptr, *pd = nullptr, *pc = nullptr, *pt = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuDeviceGet", &pg, cudaEnableDefault, &q) != cudaSuccess || !pg ||
        cudaGetDriverEntryPoint("cuDeviceGetDevResource", &pr, cudaEnableDefault, &q) != cudaSuccess || !pr ||
        cudaGetDriverEntryPoint("cuDevSmResourceSplitByCount", &ps, cudaEnableDefault, &q) != cudaSuccess || !ps ||
        cudaGetDriverEntryPoint("cuDevResourceGenerateDesc", &pd, cudaEnableDefault, &q) != cudaSuccess || !pd ||
        cudaGetDriverEntryPoint("cuGreenCtxCreate", &pc, cudaEnableDefault, &q) != cudaSuccess || !pc ||
        cudaGetDriverEntryPoint("cuGreenCtxStreamCreate", &pt, cudaEnableDefault, &q) != cudaSuccess || !pt)
        return false;
    int dev = 0;
    FDE_CUDA(cudaGetDevice(&dev));
    CUdevice cd;
    if (((FGet)pg)(&cd, dev) != CUDA_SUCCESS) return false;
    CUdevResource all, grp[1], rem;
    unsigned ng = 1;
    if (((FRes)pr)(cd, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return false;
    if (((FSplit)ps)(grp, &ng, &all, &rem, 0, (unsigned)nbulk) != CUDA_SUCCESS || ng != 1 || rem.sm.smCount < 8)
        return false;
    CUdevResourceDesc d1, d2;
    CUgreenCtx g1, g2;
    if (((FDesc)pd)(&d1, &grp[0], 1) != CUDA_SUCCESS || ((FDesc)pd)(&d2, &rem, 1) != CUDA_SUCCESS) return false;
    if (((FCreate)pc)(&g1, d1, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        ((FCreate)pc)(&g2, d2, cd, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
        return false;
    int lo = 0, hi = 0;
    FDE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUstream st;
    if (((FStream)pt)(&st, g1, CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS) return false;
    h->g_bulk = (cudaStream_t)st;
    for (int i = 0; i < 6; ++i) {
        if (((FStream)pt)(&st, g2, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS) return false;
        h->g_chain[i] = (cudaStream_t)st;
    }
    h->green_n = nbulk;   // (the green contexts live as long as the process: a handle keeps its streams)
    return true;
}

struct H2Trunc {       // one batched truncation: ranges in the flat entry / chunk arrays
    int e0 = 0, ne = 0, c0 = 0, nc = 0, kmax = 0;
};
struct H2Launch {      // ranges in the flat device arrays
    H2Trunc tr, tr_ov;
    std::vector<std::pair<int, int>> cpr;   // new low-rank columns by round (cp0, ncp)
    int snap0 = 0, nsnap = 0;               // operand factor snapshots
    std::vector<H2Trunc> trmid;             // truncations between the rounds
    int lu = -1;
    int pan0 = 0, npan = 0;
    int np0 = 0, nnp = 0;                   // neighbour-tile panels (LU stream)
    int pi0 = 0, npi = 0;                   // inverses of the factors of this step's tile (after its LU)
    int g_tile0[6] = {0, 0, 0, 0, 0, 0}, g_ntile[6] = {0, 0, 0, 0, 0, 0}, g_shape[6] = {0, 0, 0, 0, 0, 0};
    int cp0 = 0, ncp = 0;
    bool diag_scr = false;                  // the diagonal-tile update reads step scratch
};

struct H2Plan {
    int nl = 0;
    std::vector<H2Launch> fin_lv;            // leaf inverses: one level per tile distance
    std::vector<H2Launch> steps;
    H2Launch init, fin;   // initial copies + compression; final inverses
    DBuf<H2Lu> lu;
    DBuf<H2Panel> pan;
    DBuf<H2Term> terms;
    DBuf<H2Task> tasks;
    DBuf<H2Tile> tiles;
    DBuf<H2Copy> cps;
    DBuf<TEntry> te;
    DBuf<TChunk> tc;
    double* tr_part = nullptr;
    double* tr_T = nullptr;
    double* tr_part2 = nullptr;   // overflow truncations (their own stream)
    double* tr_T2 = nullptr;
    double* tr_scr = nullptr;    // k_bcore global fallback (BCORE_GSCR per entry)
    double* tr_scr2 = nullptr;
    int launches = 0;
};

static void hlu2_plan_free(H2Plan* p) { delete p; }

// per-step (target block, key) -> value with a short list per target (replaces
// std::map / std::set in the plan: no allocation per entry)
struct TKMap {
    std::vector<int> stamp, head, kk, vv, nx;
    int sid = 0;
    void init(int nb)
    {
        stamp.assign(nb, 0);
        head.assign(nb, -1);
    }
    void clear()
    {
        ++sid;
        kk.clear();
        vv.clear();
        nx.clear();
    }
    int* find(int t, int key)
    {
        if (stamp[t] != sid) return nullptr;
        for (int e = head[t]; e >= 0; e = nx[e])
            if (kk[e] == key) return &vv[e];
        return nullptr;
    }
    void put(int t, int key, int v)
    {
        if (stamp[t] != sid) {
            stamp[t] = sid;
            head[t] = -1;
        }
        kk.push_back(key);
        vv.push_back(v);
        nx.push_back(head[t]);
        head[t] = (int)kk.size() - 1;
    }
};
// Planner worker threads: run(f) calls f(0) here and f(1..n-1) on the workers and
// returns when all are done (spin-wait handshake: one call per sweep step costs a
// few microseconds; the workers exist only while a plan is built).
struct PlanPool {
    int n = 1;
    std::vector<std::thread> th;
    std::atomic<int> gen{0}, left{0};
    std::atomic<bool> quit{false};
    const std::function<void(int)>* fn = nullptr;
    std::exception_ptr err;
    std::mutex em;
    explicit PlanPool(int nt) : n(std::max(1, nt))
    {
        for (int t = 1; t < n; ++t)
            th.emplace_back([this, t]() {
                int seen = 0;
                for (;;) {
                    int g;
                    while ((g = gen.load(std::memory_order_acquire)) == seen) {
                        if (quit.load(std::memory_order_acquire)) return;
                        std::this_thread::yield();
                    }
                    seen = g;
                    try {
                        (*fn)(t);
                    } catch (...) {
                        std::lock_guard<std::mutex> l(em);
                        if (!err) err = std::current_exception();
                    }
                    left.fetch_sub(1, std::memory_order_acq_rel);
                }
            });
    }
    void run(const std::function<void(int)>& f)
    {
        fn = &f;
        left.store(n - 1, std::memory_order_release);
        gen.fetch_add(1, std::memory_order_acq_rel);
        std::exception_ptr mine;
        try {
            f(0);
        } catch (...) {
            mine = std::current_exception();
        }
        while (left.load(std::memory_order_acquire) > 0) std::this_thread::yield();
        if (mine) std::rethrow_exception(mine);
        if (err) std::rethrow_exception(err);
    }
    ~PlanPool()
    {
        quit.store(true, std::memory_order_release);
        for (auto& t : th) t.join();
    }
};

int g_hlu2_stop = -1;   // debug: run only the first g_hlu2_stop leaf steps

static bool hlu2_factor(fde_lu* L, fde_hm* hm)
{
    const auto t_plan0 = std::chrono::steady_clock::now();
    const HStruct& S = L->S;
    const bool trunc = L->tol > 0.0;
    static const bool pan_inv = !getenv("FDE_H2_PANEL_SUBST");
    // neighbour-tile panels by substitution on the LU stream, so the tile inverses
    // (needed by the other panels only) run beside them on a stream of their own
    static const bool np_subst = pan_inv && getenv("FDE_H2_NP_INV") == nullptr;   // (FDE_H2_NP_INV: old order)
    static const bool split_np = !getenv("FDE_H2_NOSPLIT");
    // deferred dense updates: a dense tile (i, j) gets the terms of the steps before
    // min(i, j) - 1 in ONE multi-term task at step min(i, j) - 2 (one read / write of
    // the tile instead of one per step); the step scratch is kept per step for them
    static const bool pretrunc = !getenv("FDE_H2_NOPRETRUNC");
    const int R = hm->R, rmax = L->rmax;
    if (trunc && (R > TRUNC_KMAX || rmax > TRUNC_KMAX)) return false;
    // ---- sweep tiles: the leaves of the cluster tree, each split into equal
    // chunks of at most H2_MMAX dofs (the partition itself is unchanged: a dense
    // leaf block then spans several tiles)
    std::vector<int> leafcl;
    for (size_t c = 0; c < S.cl.size(); ++c)
        if (S.cl[c].child[0] < 0 && S.cl[c].r1 > S.cl[c].r0) leafcl.push_back((int)c);
    std::sort(leafcl.begin(), leafcl.end(), [&](int a, int b) { return S.cl[a].r0 < S.cl[b].r0; });
    if (leafcl.empty()) return false;
    std::vector<int64_t> lr0;
    for (size_t q = 0; q < leafcl.size(); ++q) {
        const int64_t a = S.cl[leafcl[q]].r0, b = S.cl[leafcl[q]].r1;
        if (q + 1 < leafcl.size() ? S.cl[leafcl[q + 1]].r0 != b : b != S.n) return false;
        const int64_t nch = ceil_div(b - a, H2_MMAX);
        for (int64_t c = 0; c < nch; ++c) lr0.push_back(a + (b - a) * c / nch);
    }
    lr0.push_back(S.n);
    const int nl = (int)lr0.size() - 1;
    // Deferral pays with many sweep tiles (measured: c5, 256 tiles, 7 % faster per solve;
    // c4, 64 tiles, 4 % slower: a larger scratch ring for little saved traffic there).
    // FDE_H2_DEFER=0/1 forces it.
    const char* e_def = getenv("FDE_H2_DEFER");
    const bool defer = !getenv("FDE_H2_NODEFER") && (e_def ? atoi(e_def) != 0 : nl >= 128);
    // step scratch ring: a pending term from step s is flushed at step s + nring - 2 at the
    // latest (its task runs on the bulk stream before the critical stream's products of
    // step s + nring rewrite the buffer); 2 without deferral (double buffering)
    const int nring = defer ? std::max(3, getenv("FDE_H2_RING") ? atoi(getenv("FDE_H2_RING")) : 8) : 2;
    // leaves of the partition as tile ranges (the substitutions run over leaves)
    const int nleaf = (int)leafcl.size();
    std::vector<int> lq0(nleaf), lq1(nleaf), leaf_of(nl);
    for (int q = 0, f = 0; f < nleaf; ++f) {
        lq0[f] = q;
        while (q < nl && lr0[q + 1] <= S.cl[leafcl[f]].r1) leaf_of[q++] = f;
        lq1[f] = q - 1;
    }
    auto lfm = [&](int f) { return (int64_t)(lr0[lq1[f] + 1] - lr0[lq0[f]]); };
    // offset of tile (i, j) inside the inverse of leaf f (ld = leaf size)
    auto ioff = [&](int f, int i, int j) { return (lr0[j] - lr0[lq0[f]]) * lfm(f) + (lr0[i] - lr0[lq0[f]]); };
    auto lm = [&](int q) { return (int)(lr0[q + 1] - lr0[q]); };
    // tile range of a cluster (clusters are unions of consecutive tiles)
    auto lrange = [&](int cl, int& a, int& b) {
        a = (int)(std::lower_bound(lr0.begin(), lr0.end() - 1, S.cl[cl].r0) - lr0.begin());
        b = (int)(std::lower_bound(lr0.begin(), lr0.end() - 1, S.cl[cl].r1) - lr0.begin()) - 1;
        if (S.cl[cl].r1 == S.n) b = nl - 1;
    };
    const int nb = (int)S.bl.size();
    std::vector<int> t0(nb, -1), t1(nb, -1), s0(nb, -1), s1(nb, -1);
    std::vector<int> owner((size_t)nl * nl, -1);
    for (int b = 0; b < nb; ++b) {
        const HBlock& hb = S.bl[b];
        if (hb.type == HB_HIER || hb.m == 0 || hb.n == 0) continue;
        lrange(hb.tau, t0[b], t1[b]);
        lrange(hb.sig, s0[b], s1[b]);
        for (int i = t0[b]; i <= t1[b]; ++i)
            for (int j = s0[b]; j <= s1[b]; ++j) {
                if (owner[(size_t)i * nl + j] >= 0) return false;
                owner[(size_t)i * nl + j] = b;
            }
    }
    for (int q = 0; q < nl; ++q) {
        const int d = owner[(size_t)q * nl + q];
        if (d < 0 || S.bl[d].type != HB_DENSE) return false;
    }
    for (size_t t = 0; t < owner.size(); ++t)
        if (owner[t] < 0) return false;
    auto own = [&](int i, int j) { return owner[(size_t)i * nl + j]; };
    std::vector<char> dyn(nb, 0);   // low-rank blocks converted to dense during the sweep
    std::vector<int> conv_step(nb, 1 << 30);
    auto isLR = [&](int b) { return S.bl[b].type == HB_LR && !dyn[b]; };
    auto row0 = [&](int b) { return S.cl[S.bl[b].tau].r0; };
    auto col0 = [&](int b) { return S.cl[S.bl[b].sig].r0; };
    // offset of tile (i, j) inside dense block b (column-major, ld m_b)
    auto toff = [&](int b, int i, int j) { return (lr0[j] - col0(b)) * S.bl[b].m + (lr0[i] - row0(b)); };

    // ---- simulation: column counts of the low-rank blocks, per-step op lists
    std::vector<int> kc(nb, 0), kcap(nb, 0);
    for (int b = 0; b < nb; ++b)
        if (S.bl[b].type == HB_LR) kc[b] = kcap[b] = R;
    std::vector<char> pend(nb, 0);
    std::vector<VTrunc> init_trunc;
    if (trunc) {
        for (int b = 0; b < nb; ++b)
            if (S.bl[b].type == HB_LR && t0[b] >= 0) {
                init_trunc.push_back({b, kc[b]});
                kc[b] = rmax;
                kcap[b] = std::max(kcap[b], rmax);
            }
    }
    // (FDE_DEBUG_PLAN: cumulative host time of the simulation phases)
    double psec[8] = {0};
    int plast = -1;
    auto ptp = std::chrono::steady_clock::now();
    auto ptick = [&](int ph) {
        const auto now = std::chrono::steady_clock::now();
        if (plast >= 0) psec[plast] += std::chrono::duration<double, std::milli>(now - ptp).count();
        plast = ph;
        ptp = now;
    };
    std::vector<VStep> steps(nl);
    TKMap lgrp, gseen;
    lgrp.init(nb);
    gseen.init(nb);
    std::vector<int> rnd_stamp(nb, 0), rnd_val(nb, 0);
    int rnd_sid = 0;
    size_t g3_hint = 64;
    std::vector<std::vector<VTerm>> dpend(defer ? (size_t)nl * nl : 0);   // deferred dense-update terms per tile
    std::vector<int> dpend_k(defer ? (size_t)nl * nl : 0, 0);            // their summed inner dimension
    std::vector<size_t> dfull;
    std::vector<int> dfirst(defer ? (size_t)nl * nl : 0, -1);            // step of a tile's oldest pending term
    std::vector<std::vector<size_t>> dstarted(defer ? nl : 0);           // tiles whose pending list started at step s
    // the pending (deferred) dense terms of a step are built by planner threads, the
    // tiles split by row (each tile's terms keep the serial order; c5: 680k terms)
    const int plan_threads = getenv("FDE_H2_PLAN_THREADS")
                                        ? std::max(1, atoi(getenv("FDE_H2_PLAN_THREADS")))
                                        : (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));   // (c5, 16 cores: 8 -> 16 threads 340 -> 350 RHS/s)
    const int npt = defer ? plan_threads : 1;
    std::unique_ptr<PlanPool> ppool(new PlanPool(npt));
    std::vector<std::vector<size_t>> tl_started(npt), tl_full(npt);
    // a tile whose pending terms reach this inner dimension is updated right away
    // (bounds the serial work of one GEMM tile; the tile is still read / written
    // once per KFLUSH of accumulated rank instead of once per step)
    const int kflush = getenv("FDE_H2_KFLUSH") ? std::max(16, atoi(getenv("FDE_H2_KFLUSH"))) : 256;
    // products W = V_c (U_c[k]^T V_b[k]) form their 16 x 16 core in-CTA (the 128 x 16 tile
    // shape of rmax <= 16) instead of a separate launch on the binding chain.  Pays with
    // few sweep tiles (c4, 64 tiles: factorisation 11.39 -> 11.28 ms); with many, every
    // W tile re-forming its core costs more than the launch (c5, 256: 154.4 -> 156.7 ms).
    // FDE_H2_FUSECORE=0/1 forces it.
    const char* e_fc = getenv("FDE_H2_FUSECORE");
    const bool fuse_core = rmax <= 16 && !getenv("FDE_H2_SHAPES") && (e_fc ? atoi(e_fc) != 0 : nl < 128);
    std::vector<int> stamp(nb, 0), tile_stamp((size_t)nl * nl, 0), tile_task((size_t)nl * nl, 0);
    int stamp_id = 0, tile_stamp_id = 0;
    for (int k = 0; k < nl; ++k) {
        VStep& st = steps[k];
        ptick(0);
        const int sid = k % nring;   // step scratch buffer (a ring: deferred dense updates read earlier steps' scratch)
        const int mk = lm(k);
        st.sid = sid;
        st.mk = mk;
        const int dk = own(k, k);
        std::vector<int> Cb, Rc;   // column-panel blocks (rows > k), row-panel blocks (cols > k)
        for (int i = k + 1; i < nl; ++i) {
            const int b = own(i, k);
            if (Cb.empty() || Cb.back() != b) Cb.push_back(b);
        }
        for (int j = k + 1; j < nl; ++j) {
            const int c = own(k, j);
            if (Rc.empty() || Rc.back() != c) Rc.push_back(c);
        }
        for (int b : Cb)   // only dense blocks may straddle tile k (leaf blocks over several tiles)
            if (t1[b] <= k || (t0[b] <= k && S.bl[b].type != HB_DENSE)) return false;
        for (int c : Rc)
            if (s1[c] <= k || (s0[c] <= k && S.bl[c].type != HB_DENSE)) return false;
        // truncation of panel operands with pending columns
        std::vector<char> in_tr(nb, 0);
        auto add_trunc = [&](int b, bool overflow) {
            if (!trunc || !pend[b] || in_tr[b]) return;
            in_tr[b] = 1;
            (overflow ? st.trunc_ov : st.trunc).push_back({b, kc[b]});
            kc[b] = rmax;
            pend[b] = 0;
        };
        for (int b : Cb)
            if (isLR(b)) add_trunc(b, false);
        for (int c : Rc)
            if (isLR(c)) add_trunc(c, false);
        // panels (after truncation: widths are the current kc of the operands; types
        // before this step's conversions, which run after the products)
        st.lu_blk = dk;
        st.lu_off = toff(dk, k, k);
        const VRef Tk{0, dk, toff(dk, k, k)};
        const int64_t ldk = S.bl[dk].m;
        // the panels of the neighbour tiles (k+1, k) and (k, k+1) go to their own
        // launch on the LU stream when both are dense: the update of tile (k+1, k+1)
        // and LU(k+1) then wait only for them, not for the whole panel launch
        const bool nsplit = split_np && k + 1 < nl && !isLR(own(k + 1, k)) && !isLR(own(k, k + 1));
        for (int b : Cb) {
            const HBlock& B = S.bl[b];
            if (isLR(b)) {
                st.panel.push_back({Tk, ldk, {2, b, lr0[k] - col0(b)}, B.n, mk, kc[b], 1});
            } else {   // rows of tiles > k of the column of tile k
                int i0 = std::max(t0[b], k + 1);
                if (nsplit && i0 == k + 1) {
                    st.npanel.push_back({Tk, ldk, {0, b, toff(b, k + 1, k)}, B.m, mk, lm(k + 1), 2});
                    ++i0;
                }
                if (i0 <= t1[b])
                    st.panel.push_back({Tk, ldk, {0, b, toff(b, i0, k)}, B.m, mk, (int)(lr0[t1[b] + 1] - lr0[i0]), 2});
            }
        }
        for (int c : Rc) {
            const HBlock& C = S.bl[c];
            if (isLR(c)) {
                st.panel.push_back({Tk, ldk, {1, c, lr0[k] - row0(c)}, C.m, mk, kc[c], 0});
            } else {   // columns of tiles > k of the row of tile k
                int j0 = std::max(s0[c], k + 1);
                if (nsplit && j0 == k + 1) {
                    st.npanel.push_back({Tk, ldk, {0, c, toff(c, k, k + 1)}, C.m, mk, lm(k + 1), 0});
                    ++j0;
                }
                if (j0 <= s1[c])
                    st.panel.push_back({Tk, ldk, {0, c, toff(c, k, j0)}, C.m, mk, (int)(lr0[s1[c] + 1] - lr0[j0]), 0});
            }
        }
        if (pan_inv) {   // panels as products with the tile inverses (computed after LU(k))
            const int f = leaf_of[k];
            for (auto* pl : {&st.panel, &st.npanel})
                for (auto& pv : *pl) {
                    if (np_subst && pl == &st.npanel) continue;
                    pv.Ti = {pv.mode == 0 ? 4 : 5, f, ioff(f, k, k)};
                    pv.ldi = lfm(f);
                }
        }
        ptick(1);
        // products: pair scratch offsets
        struct Pair { int b, c; int64_t w; int rw; bool bl, cl; };   // bl/cl: operand types at this step   // w: W (n_c x kc_b) or Z (m_b x kc_c) scratch offset
        std::vector<Pair> pairs;
        int64_t scr = 0;
        // snapshots of the low-rank operand factors read by this step's dense-target
        // updates (U_b of the column panel, V_c of the row panel): the updates run
        // concurrently with step k+1, whose truncations / panels rewrite the factors
        std::map<int, int64_t> snapU, snapV;
        for (int b : Cb)
            if (isLR(b)) {
                snapU[b] = scr;
                st.snap.push_back({{1, b, 0}, {3, sid, scr}, S.bl[b].m, S.bl[b].m, (int)S.bl[b].m, kc[b], 0, 1.0});
                scr += S.bl[b].m * kc[b];
            }
        for (int c : Rc)
            if (isLR(c)) {
                snapV[c] = scr;
                st.snap.push_back({{2, c, 0}, {3, sid, scr}, S.bl[c].n, S.bl[c].n, (int)S.bl[c].n, kc[c], 0, 1.0});
                scr += S.bl[c].n * kc[c];
            }
        for (int b : Cb)
            for (int c : Rc) {
                Pair pr{b, c, -1, 0, isLR(b), isLR(c)};
                const HBlock &B = S.bl[b], &C = S.bl[c];
                if (isLR(b)) {
                    int64_t core = -1;
                    const bool fuse = fuse_core && isLR(c) && kc[c] <= 16 && kc[b] <= 16;
                    if (isLR(c)) {   // core = U_c[k]^T V_b[k]  (kc_c x kc_b)
                        core = scr;
                        scr += (int64_t)kc[c] * kc[b];
                        if (!fuse) {
                            VTask t{{3, sid, core}, kc[c], kc[c], kc[b], 0.0, {}};
                            t.terms.push_back({{1, c, lr0[k] - row0(c)}, {2, b, lr0[k] - col0(b)}, C.m, B.n, mk, 1, 0, 1.0});
                            st.g1.push_back(t);
                        }
                    }
                    pr.w = scr;
                    pr.rw = kc[b];
                    scr += C.n * kc[b];
                    VTask t{{3, sid, pr.w}, C.n, (int)C.n, kc[b], 0.0, {}};
                    if (fuse)      // the core definition rides with the product (formed in-CTA)
                        t.terms.push_back({{1, c, lr0[k] - row0(c)}, {2, b, lr0[k] - col0(b)}, C.m, B.n, mk, 3, 0, 1.0});
                    if (isLR(c))   // W = V_c core
                        t.terms.push_back({{2, c, 0}, {3, sid, core}, C.n, kc[c], kc[c], 0, 0, 1.0});
                    else           // W = D_c[k rows, :]^T V_b[k]
                        t.terms.push_back({{0, c, lr0[k] - row0(c)}, {2, b, lr0[k] - col0(b)}, C.m, B.n, mk, 1, 0, 1.0});
                    st.g2.push_back(t);
                } else if (isLR(c)) {   // Z = D_b[:, k cols] U_c[k]   (m_b x kc_c)
                    pr.w = scr;
                    pr.rw = kc[c];
                    scr += B.m * kc[c];
                    VTask t{{3, sid, pr.w}, B.m, (int)B.m, kc[c], 0.0, {}};
                    t.terms.push_back({{0, b, (lr0[k] - col0(b)) * B.m}, {1, c, lr0[k] - row0(c)}, B.m, C.m, mk, 0, 0, 1.0});
                    st.g2.push_back(t);
                }
                pairs.push_back(pr);
            }
        ptick(2);
        // targets
        st.g3.reserve(g3_hint);
        st.g3crit.reserve(g3_hint);
        ++tile_stamp_id;   // dense target tile (i, j) -> g3 task (stamped flat table)
        struct Grp { int t, key, rank; int64_t slot; int round; };
        lgrp.clear();                                 // (target, key) -> group index
        std::vector<Grp> grps;
        std::vector<int> incoming(nb, 0);
        std::vector<std::pair<int, int>> lterms;     // (pair index, group index)
        // targets of every pair
        std::vector<std::vector<int>> ptg(pairs.size());
        for (size_t pi = 0; pi < pairs.size(); ++pi) {
            const int b = pairs[pi].b, c = pairs[pi].c;
            ++stamp_id;
            for (int i = std::max(t0[b], k + 1); i <= t1[b];) {
                int inext = t1[b] + 1;
                for (int j = std::max(s0[c], k + 1); j <= s1[c];) {   // jump over the column run of each owner
                    const int t = own(i, j);
                    if (stamp[t] != stamp_id) {
                        stamp[t] = stamp_id;
                        ptg[pi].push_back(t);
                    }
                    inext = std::min(inext, t1[t] + 1);
                    j = s1[t] + 1;
                }
                i = std::max(i + 1, inext);   // rows of the same owners repeat the same targets
            }
        }
        ptick(3);
        // low-rank targets that must become dense: a dense x dense product lands
        // in them, or their width would exceed what a low-rank block can hold
        // (TRUNC_KMAX after truncation; min(m, n) / 2 in exact mode)
        {
            gseen.clear();
            std::vector<char> conv(nb, 0);
            for (size_t pi = 0; pi < pairs.size(); ++pi) {
                const int b = pairs[pi].b, c = pairs[pi].c;
                const bool bl = pairs[pi].bl, cl = pairs[pi].cl;
                for (int t : ptg[pi]) {
                    if (!isLR(t)) continue;
                    if (!bl && !cl) { conv[t] = 1; continue; }
                    const int key = bl ? b : (nb + c);
                    if (!gseen.find(t, key)) {
                        gseen.put(t, key, 1);
                        incoming[t] += bl ? kc[b] : kc[c];
                    }
                }
            }
            for (int t = 0; t < nb; ++t) {
                if (!isLR(t) || (!incoming[t] && !conv[t])) continue;
                const HBlock& T = S.bl[t];
                const int lim = trunc ? TRUNC_KMAX : (int)std::max<int64_t>(1, std::min(T.m, T.n) / 2);
                if (!conv[t] && kc[t] + incoming[t] > lim) {
                    // truncated blocks: make room first; more new columns than a block can
                    // hold are added in rounds with a truncation in between (below).
                    // Exact mode (tol = 0): a block that would get wider than half its
                    // smaller dimension is better stored dense.
                    if (trunc) add_trunc(t, true);
                    else conv[t] = 1;
                }
                if (conv[t]) {   // D_t = U_t V_t^T, then a dense block for good
                    VTask tk{{0, t, 0}, T.m, (int)T.m, (int)T.n, 0.0, {}};
                    tk.terms.push_back({{1, t, 0}, {2, t, 0}, T.m, T.n, kc[t], 0, 1, 1.0});
                    st.g0.push_back(tk);
                    dyn[t] = 1;
                    conv_step[t] = k;
                    pend[t] = 0;
                    incoming[t] = 0;
                }
            }
        }
        ptick(4);
        for (size_t pi = 0; pi < pairs.size(); ++pi) {
            const Pair& pr = pairs[pi];
            const int b = pr.b, c = pr.c;
            const int64_t su_b = pr.bl ? snapU[b] : 0, sv_c = (!pr.bl && pr.cl) ? snapV[c] : 0;   // (hoisted lookups)
            if (!defer) {   // compact record; expanded at flatten time
                st.dpairs.push_back({b, c, pr.w, su_b, sv_c, kc[b], kc[c], pr.bl, pr.cl});
            }
            for (int t : ptg[pi]) {
                const HBlock& T = S.bl[t];
                if (!isLR(t) && !defer) {
                    st.dts.push_back({(int)st.dpairs.size() - 1, t});
                } else if (!isLR(t)) {
                    const int jlo1 = std::max(std::max(s0[c], s0[t]), k + 1), jhi1 = std::min(s1[c], s1[t]);
                    for (int i = std::max(std::max(t0[b], t0[t]), k + 1); i <= std::min(t1[b], t1[t]); ++i) {
                        int jlo = jlo1, jhi = jhi1;
                        if (npt > 1 && i != k + 1) {   // the pending tiles are the planner threads' share (below)
                            if (jlo1 != k + 1) continue;
                            jhi = k + 1;
                        }
                        for (int j = jlo; j <= jhi; ++j) {
                            const size_t key = (size_t)i * nl + j;
                            const bool to_pend = defer && i != k + 1 && j != k + 1;
                            int ti = -1;
                            if (to_pend) {
                                // (the term is built below and appended to pend[key])
                            } else if (tile_stamp[key] != tile_stamp_id) {
                                ti = (int)st.g3.size();
                                tile_stamp[key] = tile_stamp_id;
                                tile_task[key] = ti;
                                st.g3.push_back(VTask{{0, t, (lr0[j] - col0(t)) * T.m + (lr0[i] - row0(t))}, T.m, lm(i), lm(j), 1.0, {}});
                                // 2: the next diagonal tile (input of LU(k+1), right after the panels);
                                // 1: row / column k+1 and the diagonal tile after it (critical stream);
                                // 0: the rest (lookahead stream)
                                st.g3crit.push_back((i == k + 1 && j == k + 1) ? 2
                                                    : (i == k + 1 || j == k + 1 || (i == k + 2 && j == k + 2)));
                            } else {
                                ti = tile_task[key];
                            }
                            const HBlock &B = S.bl[b], &C = S.bl[c];
                            VTerm term;
                            if (!pr.bl && !pr.cl) {
                                term = {{0, b, (lr0[k] - col0(b)) * B.m + (lr0[i] - row0(b))},
                                        {0, c, (lr0[j] - col0(c)) * C.m + (lr0[k] - row0(c))}, B.m, C.m, mk, 0, 0, -1.0};
                            } else if (pr.bl) {   // U_b[i rows] W[j rows]^T
                                term = {{3, sid, su_b + (lr0[i] - row0(b))}, {3, sid, pr.w + (lr0[j] - col0(c))}, B.m, C.n,
                                        kc[b], 0, 1, -1.0};
                            } else {               // Z[i rows] V_c[j rows]^T
                                term = {{3, sid, pr.w + (lr0[i] - row0(b))}, {3, sid, sv_c + (lr0[j] - col0(c))}, B.m, C.n,
                                        kc[c], 0, 1, -1.0};
                            }
                            if (to_pend) {
                                if (dpend[key].empty()) {
                                    dfirst[key] = k;
                                    dstarted[k].push_back(key);
                                    dpend[key].reserve(16);   // (~16 terms reach kflush)
                                }
                                dpend[key].push_back(term);
                                if ((dpend_k[key] += term.k) >= kflush) dfull.push_back(key);
                            }
                            else st.g3[ti].terms.push_back(term);
                        }
                    }
                } else {
                    const int key = pr.bl ? b : (nb + c);
                    int gi;
                    if (int* f = lgrp.find(t, key)) {
                        gi = *f;
                    } else {
                        gi = (int)grps.size();
                        lgrp.put(t, key, gi);
                        grps.push_back({t, key, pr.bl ? kc[b] : kc[c], -1, 0});
                    }
                    lterms.push_back({(int)pi, gi});
                }
            }
        }
        if (defer && npt > 1) {   // the pending tiles, rows i = tid mod npt per thread
            std::vector<std::pair<int64_t, int64_t>> psnap(pairs.size());
            for (size_t pi = 0; pi < pairs.size(); ++pi) {
                const Pair& pr = pairs[pi];
                psnap[pi] = {pr.bl ? snapU[pr.b] : 0, (!pr.bl && pr.cl) ? snapV[pr.c] : 0};
            }
            const std::function<void(int)> work = [&](int tid) {
                std::vector<size_t>& started = tl_started[tid];
                std::vector<size_t>& full = tl_full[tid];
                started.clear();
                full.clear();
                for (size_t pi = 0; pi < pairs.size(); ++pi) {
                    const Pair& pr = pairs[pi];
                    const int b = pr.b, c = pr.c;
                    const int64_t su_b = psnap[pi].first, sv_c = psnap[pi].second;
                    const HBlock &B = S.bl[b], &C = S.bl[c];
                    for (int t : ptg[pi]) {
                        if (isLR(t)) continue;
                        const int ilo = std::max(std::max(t0[b], t0[t]), k + 2), ihi = std::min(t1[b], t1[t]);
                        const int jlo = std::max(std::max(s0[c], s0[t]), k + 2), jhi = std::min(s1[c], s1[t]);
                        for (int i = ilo + (((tid - ilo) % npt) + npt) % npt; i <= ihi; i += npt)
                            for (int j = jlo; j <= jhi; ++j) {
                                const size_t key = (size_t)i * nl + j;
                                VTerm term;
                                if (!pr.bl && !pr.cl) {
                                    term = {{0, b, (lr0[k] - col0(b)) * B.m + (lr0[i] - row0(b))},
                                            {0, c, (lr0[j] - col0(c)) * C.m + (lr0[k] - row0(c))}, B.m, C.m, mk, 0, 0, -1.0};
                                } else if (pr.bl) {
                                    term = {{3, sid, su_b + (lr0[i] - row0(b))}, {3, sid, pr.w + (lr0[j] - col0(c))}, B.m,
                                            C.n, kc[b], 0, 1, -1.0};
                                } else {
                                    term = {{3, sid, pr.w + (lr0[i] - row0(b))}, {3, sid, sv_c + (lr0[j] - col0(c))}, B.m,
                                            C.n, kc[c], 0, 1, -1.0};
                                }
                                std::vector<VTerm>& pv = dpend[key];
                                if (pv.empty()) {
                                    dfirst[key] = k;
                                    started.push_back(key);
                                    pv.reserve(16);
                                }
                                pv.push_back(term);
                                if ((dpend_k[key] += term.k) >= kflush) full.push_back(key);
                            }
                    }
                }
            };
            ppool->run(work);
            for (int q = 0; q < npt; ++q) {
                dstarted[k].insert(dstarted[k].end(), tl_started[q].begin(), tl_started[q].end());
                dfull.insert(dfull.end(), tl_full[q].begin(), tl_full[q].end());
            }
        }
        if (defer) {   // flush full tiles, and the pending terms of row / column k+2
            const int m2 = k + 2;
            auto flush = [&](int i, int j) {
                std::vector<VTerm>& pv = dpend[(size_t)i * nl + j];
                if (pv.empty()) return;
                dpend_k[(size_t)i * nl + j] = 0;
                dfirst[(size_t)i * nl + j] = -1;
                const int t = own(i, j);
                const HBlock& T = S.bl[t];
                VTask tk{{0, t, (lr0[j] - col0(t)) * T.m + (lr0[i] - row0(t))}, T.m, lm(i), lm(j), 1.0, {}};
                tk.terms.adopt(std::move(pv));   // (the pending vector moves into the task)
                st.g3.push_back(std::move(tk));
                // (k+2, k+2) on the critical stream: it is the input of LU(k+2) next step
                st.g3crit.push_back(i == m2 && j == m2 ? 1 : 0);
                pv = std::vector<VTerm>();
            };
            for (size_t key : dfull) flush((int)(key / nl), (int)(key % nl));
            dfull.clear();
            const int s_old = k - nring + 2;   // scratch buffer of step s_old is rewritten at step s_old + nring
            if (s_old >= 0) {
                for (size_t key : dstarted[s_old])
                    if (dfirst[key] == s_old) flush((int)(key / nl), (int)(key % nl));
                std::vector<size_t>().swap(dstarted[s_old]);
            }
            if (m2 < nl) {
                for (int j = m2; j < nl; ++j) flush(m2, j);
                for (int i = m2 + 1; i < nl; ++i) flush(i, m2);
            }
        }
        g3_hint = st.g3.size() + 64;   // (reserve for the next step: fewer reallocations)
        ptick(5);
        // early truncation of the panel operands of step k+1 that are not operands of
        // this step: they run off the critical stream (with the overflow truncations,
        // before this step's new columns), so that step k+1 only has to recompress
        // the columns step k adds (rmax + one group instead of up to TRUNC_KMAX)
        if (trunc && pretrunc && k + 1 < nl) {
            std::set<int> opnd(Cb.begin(), Cb.end());
            opnd.insert(Rc.begin(), Rc.end());
            for (int i = k + 2; i < nl; ++i) {
                const int b = own(i, k + 1);
                if (isLR(b) && !opnd.count(b)) add_trunc(b, true);
            }
            for (int j = k + 2; j < nl; ++j) {
                const int c = own(k + 1, j);
                if (isLR(c) && !opnd.count(c)) add_trunc(c, true);
            }
        }
        ptick(6);
        // slots and copies; a target whose new columns do not fit gets them in rounds,
        // truncated between rounds (formatted addition of the partial sums)
        std::vector<char> u_done(grps.size(), 0);
        ++rnd_sid;   // target -> current round (stamped)
        for (size_t g = 0; g < grps.size(); ++g) {
            const int t = grps[g].t;
            if (rnd_stamp[t] != rnd_sid) {
                rnd_stamp[t] = rnd_sid;
                rnd_val[t] = 0;
            }
            int& r = rnd_val[t];
            if (trunc && kc[t] + grps[g].rank > TRUNC_KMAX) {
                if (rmax + grps[g].rank > TRUNC_KMAX) return false;   // a single group never exceeds it
                if ((int)st.trmid.size() <= r) st.trmid.resize(r + 1);
                st.trmid[r].push_back({t, kc[t]});
                ++r;
                kc[t] = rmax;
            }
            grps[g].round = r;
            grps[g].slot = kc[t];
            kc[t] += grps[g].rank;
            kcap[t] = std::max(kcap[t], kc[t]);
            pend[t] = 1;
        }
        int nround = 1;
        for (auto& g : grps) nround = std::max(nround, g.round + 1);
        st.cpr.resize(nround);
        for (auto& lt : lterms) {
            const Pair& pr = pairs[lt.first];
            Grp& g = grps[lt.second];
            const int t = g.t, b = pr.b, c = pr.c;
            const HBlock &T = S.bl[t], &B = S.bl[b], &C = S.bl[c];
            const int ia = std::max(std::max(t0[b], t0[t]), k + 1), ib = std::min(t1[b], t1[t]);
            const int ja = std::max(std::max(s0[c], s0[t]), k + 1), jb = std::min(s1[c], s1[t]);
            const int64_t R0 = lr0[ia], R1 = lr0[ib + 1], C0 = lr0[ja], C1 = lr0[jb + 1];
            const int64_t us = g.slot * T.m + (R0 - row0(t)), vs = g.slot * T.n + (C0 - col0(t));
            if (pr.bl) {
                if (!u_done[lt.second]) {   // U slot rows R = U_b rows (once per group)
                    u_done[lt.second] = 1;
                    st.cpr[g.round].push_back({{1, b, R0 - row0(b)}, {1, t, us}, B.m, T.m, (int)(R1 - R0), g.rank, 0, 1.0});
                }
                st.cpr[g.round].push_back({{3, sid, pr.w + (C0 - col0(c))}, {2, t, vs}, C.n, T.n, (int)(C1 - C0), g.rank, 0, -1.0});
            } else {
                if (!u_done[lt.second]) {   // V slot rows C = -V_c rows (once per group)
                    u_done[lt.second] = 1;
                    st.cpr[g.round].push_back({{2, c, C0 - col0(c)}, {2, t, vs}, C.n, T.n, (int)(C1 - C0), g.rank, 0, -1.0});
                }
                st.cpr[g.round].push_back({{3, sid, pr.w + (R0 - row0(b))}, {1, t, us}, B.m, T.m, (int)(R1 - R0), g.rank, 0, 1.0});
            }
        }
        st.scratch = scr;
    }
    if (trunc)
        for (int b = 0; b < nb; ++b)
            if (pend[b]) return false;   // every update precedes a use (see header)

    auto ms_since = [&](std::chrono::steady_clock::time_point t) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
    };
    ptick(7);
    ppool.reset();   // (the planner threads end with the simulation)
    const double ms_sim = ms_since(t_plan0);
    const auto t_alloc0 = std::chrono::steady_clock::now();
    // ---- arena layout
    std::vector<int64_t> offD(nb, -1), offU(nb, -1), offV(nb, -1);
    int64_t words = 0;
    for (int b = 0; b < nb; ++b) {
        const HBlock& hb = S.bl[b];
        if (hb.type == HB_DENSE || dyn[b]) { offD[b] = words; words += hb.m * hb.n; }
    }
    const int64_t lr_lo = words;
    for (int b = 0; b < nb; ++b) {
        const HBlock& hb = S.bl[b];
        if (hb.type == HB_LR) {
            offU[b] = words; words += hb.m * kcap[b];
            offV[b] = words; words += hb.n * kcap[b];
        }
    }
    const int64_t lr_hi = words;
    // inverses of the leaf factors L_f^{-1}, U_f^{-1} (leaf size squared each)
    std::vector<int64_t> offLi(nleaf), offUi(nleaf);
    const int64_t inv_lo = words;
    for (int f = 0; f < nleaf; ++f) {
        offLi[f] = words; words += lfm(f) * lfm(f);
        offUi[f] = words; words += lfm(f) * lfm(f);
    }
    const int64_t inv_hi = words;
    int64_t scr_max = 1;
    for (auto& st : steps) scr_max = std::max(scr_max, st.scratch);
    int maxnt = 1;
    for (int f = 0; f < nleaf; ++f) maxnt = std::max(maxnt, lq1[f] - lq0[f] + 1);
    for (int dd = 1; dd < maxnt; ++dd) {   // scratch of the block-triangular inversion levels
        int64_t w = 0;
        for (int f = 0; f < nleaf; ++f)
            for (int i = lq0[f]; i <= lq1[f]; ++i)
                for (int j = lq0[f]; j <= lq1[f]; ++j)
                    if (std::abs(i - j) == dd) w += (int64_t)lm(i) * lm(j);
        scr_max = std::max(scr_max, w);
    }
    // step scratch (W / Z products, cores, operand snapshots).  Deferred dense
    // updates read the scratch of earlier steps: one buffer per step.  Otherwise
    // double-buffered: the products of step k are read by the copies (stream sb) and
    // the bulk updates (stream sc) of step k, which complete before the critical
    // stream reaches the products of step k+2.
    const int64_t off_scr = words;
    words += (int64_t)nring * scr_max;
    // truncation workspace (max over batches)
    int64_t gmax = 1, tmax = 1, emax = 1;
    auto tr_size = [&](const std::vector<VTrunc>& v) {
        int64_t g = 0, tt = 0;
        for (auto& e : v) {
            const HBlock& hb = S.bl[e.blk];
            g += (ceil_div(hb.m, TRUNC_CHUNK) + ceil_div(hb.n, TRUNC_CHUNK)) * GRAM_SLOT(e.k);
            tt += 2LL * e.k * rmax;
        }
        gmax = std::max(gmax, g);
        tmax = std::max(tmax, tt);
        emax = std::max(emax, (int64_t)v.size());
    };
    tr_size(init_trunc);
    for (auto& st : steps) {
        tr_size(st.trunc);
        tr_size(st.trunc_ov);
        for (auto& v : st.trmid) tr_size(v);
    }
    const int64_t off_part = words;
    words += 2 * gmax;   // [operand truncations | overflow truncations] (two streams)
    const int64_t off_T = words;
    words += 2 * tmax;
    const int64_t off_cs = words;
    words += 2 * emax * BCORE_GSCR;

    H2Plan* P = new H2Plan();
    L->plan = P;
    P->nl = nl;
    cudaStream_t s = L->h->stream;
    {
        void* p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, (size_t)words * sizeof(double), s);
        if (e != cudaSuccess) throw FdeError{FDE_ENOMEM, "hlu_factor: arena allocation failed"};
        L->arena = (double*)p;
    }
    double* A = L->arena;
    P->tr_part = A + off_part;
    P->tr_T = A + off_T;
    P->tr_part2 = A + off_part + gmax;
    P->tr_T2 = A + off_T + tmax;
    P->tr_scr = A + off_cs;
    P->tr_scr2 = A + off_cs + emax * BCORE_GSCR;
    auto res = [&](const VRef& r) -> double* {
        switch (r.sp) {
            case 0: return A + offD[r.id] + r.off;
            case 1: return A + offU[r.id] + r.off;
            case 2: return A + offV[r.id] + r.off;
            case 3: return A + off_scr + r.id * scr_max + r.off;
            case 4: return A + offLi[r.id] + r.off;
            case 5: return A + offUi[r.id] + r.off;
            case 6: return hm->dense.p + r.off;   // the H-matrix's own arenas (init copies)
            default: return hm->lr.p + r.off;
        }
    };

    const double ms_alloc = ms_since(t_alloc0);
    const auto t_flat0 = std::chrono::steady_clock::now();
    // ---- flatten descriptors
    std::vector<H2Lu> vlu;
    std::vector<H2Panel> vpan;
    std::vector<H2Term> vterm;
    std::vector<H2Task> vtask;
    std::vector<H2Tile> vtile;
    std::vector<H2Copy> vcp;
    std::vector<TEntry> vte;
    std::vector<TChunk> vtc;
    auto put_trunc = [&](const std::vector<VTrunc>& v, H2Trunc& ln) {
        ln.e0 = (int)vte.size();
        ln.c0 = (int)vtc.size();
        long long gofs = 0, tofs = 0;
        for (auto& e : v) {
            const HBlock& hb = S.bl[e.blk];
            TEntry te;
            te.U = A + offU[e.blk];
            te.V = A + offV[e.blk];
            te.Uo = A + offU[e.blk];
            te.Vo = A + offV[e.blk];
            te.m = hb.m;
            te.n = hb.n;
            te.k = e.k;
            te.zero_tail = 1;
            te.c_lo = (int)vtc.size() - ln.c0;
            for (int side = 0; side < 2; ++side) {
                const long long rows = side ? hb.n : hb.m;
                for (long long r = 0; r < rows; r += TRUNC_CHUNK)
                    vtc.push_back(TChunk{(int)(vte.size() - ln.e0), side, r,
                                         (int)std::min<long long>(TRUNC_CHUNK, rows - r)});
            }
            te.c_hi = (int)vtc.size() - ln.c0;
            te.gofs = gofs;
            gofs += (long long)(te.c_hi - te.c_lo) * GRAM_SLOT(e.k);
            te.tofs = tofs;
            tofs += 2LL * e.k * rmax;
            ln.kmax = std::max(ln.kmax, e.k);
            vte.push_back(te);
        }
        ln.ne = (int)vte.size() - ln.e0;
        ln.nc = (int)vtc.size() - ln.c0;
    };
    double gstat_flop[6] = {0}, gstat_cbytes[6] = {0};   // (FDE_DEBUG_PLAN statistics)
    // GEMM tile per launch group (cores, products, crit, conversions, rest, diag):
    // 32 x 32 where a launch has few tiles (latency: more CTAs, shorter chains)
    // tile shape per launch group (0 cores, 1 products, 2 crit, 3 conversions, 4 rest,
    // 5 diag): 0 = 64 x 64, 1 = 32 x 32 (few tiles: more CTAs, shorter chains),
    // 2 = 128 x 16 (products: outputs rmax wide), 3 = 16 x 16 (cores: rmax x rmax)
    int gemm_shape[6] = {rmax <= 16 ? 3 : 1, rmax <= 16 ? 2 : 0, 0, 0, 0, 1};
    if (const char* e = getenv("FDE_H2_SHAPES"))   // debug: six digits
        for (int w = 0; w < 6 && e[w]; ++w) gemm_shape[w] = std::min(5, std::max(0, e[w] - '0'));
    const bool plan_stats = getenv("FDE_DEBUG_PLAN") != nullptr;
    // tasks of v (then v2) with sel[q] == want (sel null: all), in order
    auto put_gemm_sel = [&](const std::vector<VTask>& v, const std::vector<char>* sel, char want, H2Launch& ln,
                            int which, int shape, const std::vector<VTask>* v2 = nullptr,
                            const std::vector<char>* sel2 = nullptr) {
        ln.g_shape[which] = shape;
        ln.g_tile0[which] = (int)vtile.size();
        static const int shm[6] = {64, 32, 128, 16, 128, 64}, shn[6] = {64, 32, 16, 16, 64, 128};
        const int tm = shm[shape], tn = shn[shape];
        const size_t n1 = v.size(), n2 = v2 ? v2->size() : 0;
        for (size_t q = 0; q < n1 + n2; ++q) {
            if (q < n1 ? (sel && (*sel)[q] != want) : (*sel2)[q - n1] != want) continue;
            const VTask& t = q < n1 ? v[q] : (*v2)[q - n1];
            H2Task d;
            d.C = res(t.C);
            d.ldc = t.ldc;
            d.m = t.m;
            d.n = t.n;
            d.beta = t.beta;
            d.t_lo = (int)vterm.size();
            for (auto& q : t.terms)
                vterm.push_back({res(q.A), res(q.B), q.lda, q.ldb, q.k, q.ta, q.tb, q.alpha});
            d.t_hi = (int)vterm.size();
            if (plan_stats) {
                for (auto& q : t.terms) gstat_flop[which] += 2.0 * t.m * t.n * q.k;
                gstat_cbytes[which] += 16.0 * t.m * t.n;
            }
            const int ti = (int)vtask.size();
            vtask.push_back(d);
            for (int m0 = 0; m0 < t.m; m0 += tm)
                for (int n0 = 0; n0 < t.n; n0 += tn) vtile.push_back({ti, m0, n0});
        }
        ln.g_ntile[which] = (int)vtile.size() - ln.g_tile0[which];
    };
    auto put_gemm = [&](const std::vector<VTask>& v, H2Launch& ln, int which, int shape) {
        put_gemm_sel(v, nullptr, 0, ln, which, shape);
    };
    auto put_copy = [&](const std::vector<VCopy>& v, H2Launch& ln) {
        ln.cp0 = (int)vcp.size();
        for (auto& c : v) {
            if (c.m <= 0 || c.n <= 0) continue;
            double* dst = res(c.dst);
            const double* src = c.kind == 0 ? res(c.src) : nullptr;
            if (c.kind == 2 || (int64_t)c.m * c.n <= H2_CP_CHUNK) {
                vcp.push_back({src, c.lds, dst, c.ldd, c.m, c.n, c.kind, c.alpha});
                continue;
            }
            // large copies: one CTA per chunk of <= H2_CP_CHUNK elements
            const int rm = std::min(c.m, H2_CP_CHUNK), cn = std::max(1, H2_CP_CHUNK / rm);
            for (int c0 = 0; c0 < c.n; c0 += cn)
                for (int r0 = 0; r0 < c.m; r0 += rm)
                    vcp.push_back({src ? src + (int64_t)c0 * c.lds + r0 : nullptr, c.lds, dst + (int64_t)c0 * c.ldd + r0,
                                   c.ldd, std::min(rm, c.m - r0), std::min(cn, c.n - c0), c.kind, c.alpha});
        }
        ln.ncp = (int)vcp.size() - ln.cp0;
    };
    auto put_panel = [&](const std::vector<VPanel>& v, H2Launch& ln) {
        ln.pan0 = (int)vpan.size();
        static const int inv_strip = getenv("FDE_H2_INV_STRIP") ? std::max(8, std::min(H2_STRIP, atoi(getenv("FDE_H2_INV_STRIP")))) : 16;
        static const bool sub_all = !(getenv("FDE_H2_SUB_STRIP_ALL") && atoi(getenv("FDE_H2_SUB_STRIP_ALL")) == 0);   // (also the neighbour panels)
        for (auto& p : v) {
            // (the tile inverses -- substitutions on identity strips, X in the inverse
            // arenas -- may use narrower strips: more CTAs, shorter trailing updates)
            const int strip = (sub_all || p.X.sp == 4 || p.X.sp == 5) && p.Ti.sp < 0 ? inv_strip : H2_STRIP;
            for (int c0 = 0; c0 < p.nvec; c0 += strip) {
                H2Panel d;
                d.T = res(p.T);
                d.ldt = p.ldt;
                const int nv = std::min(strip, p.nvec - c0);
                d.X = res(p.X) + (p.mode == 2 ? c0 : c0 * p.ldx);
                d.ldx = p.ldx;
                d.m = p.m;
                d.nvec = nv;
                d.mode = p.mode;
                d.Ti = p.Ti.sp >= 0 ? res(p.Ti) : nullptr;
                d.ldi = p.ldi;
                vpan.push_back(d);
            }
        }
        ln.npan = (int)vpan.size() - ln.pan0;
    };
    // ---- the op lists of the init and final phases
    std::vector<VCopy> init_cp;   // dense blocks and the R Taylor columns, from the H-matrix arenas
    for (int b = 0; b < nb; ++b) {
        const HBlock& hb = S.bl[b];
        if (t0[b] < 0) continue;
        if (hb.type == HB_DENSE) {
            init_cp.push_back({{6, b, hb.off}, {0, b, 0}, hb.m, hb.m, (int)hb.m, (int)hb.n, 0, 1.0});
        } else if (hb.type == HB_LR) {
            init_cp.push_back({{7, b, hb.off}, {1, b, 0}, hb.m, hb.m, (int)hb.m, R, 0, 1.0});
            init_cp.push_back({{7, b, hb.off + hb.m * hb.kcap}, {2, b, 0}, hb.n, hb.n, (int)hb.n, R, 0, 1.0});
        }
    }
    // final: explicit inverses of the leaf factors (for the substitutions).  Tile
    // inverses on the diagonal, then the off-diagonal tiles level by level:
    //   L^{-1}(i,j) = -Linv(i,i) sum_{k=j}^{i-1} L(i,k) L^{-1}(k,j)       (i > j)
    //   U^{-1}(i,j) = -Uinv(i,i) sum_{k=i+1}^{j} U(i,k) U^{-1}(k,j)       (i < j)
    std::vector<VCopy> fin_cp;
    std::vector<VPanel> fin_pv;
    std::vector<std::vector<VTask>> fin_tt(std::max(0, maxnt - 1)), fin_tx(std::max(0, maxnt - 1));
    for (int q = 0; q < nl; ++q) {
        const int d = own(q, q), f = leaf_of[q];
        const VRef Tq{0, d, toff(d, q, q)};
        fin_cp.push_back({{4, f, 0}, {4, f, ioff(f, q, q)}, 0, lfm(f), lm(q), lm(q), 2, 1.0});
        fin_cp.push_back({{5, f, 0}, {5, f, ioff(f, q, q)}, 0, lfm(f), lm(q), lm(q), 2, 1.0});
        fin_pv.push_back({Tq, S.bl[d].m, {4, f, ioff(f, q, q)}, lfm(f), lm(q), lm(q), 0});
        fin_pv.push_back({Tq, S.bl[d].m, {5, f, ioff(f, q, q)}, lfm(f), lm(q), lm(q), 2});
    }
    for (int dd = 1; dd < maxnt; ++dd) {
        int64_t scr = 0;
        for (int f = 0; f < nleaf; ++f) {
            const int d = own(lq0[f], lq0[f]);
            const int64_t md = S.bl[d].m, mf = lfm(f);
            for (int i = lq0[f]; i <= lq1[f]; ++i)
                for (int j = lq0[f]; j <= lq1[f]; ++j) {
                    if (std::abs(i - j) != dd) continue;
                    const bool low = i > j;
                    const int sp = low ? 4 : 5;
                    VTask t{{3, 0, scr}, lm(i), lm(i), lm(j), 0.0, {}};
                    for (int k = low ? j : i + 1; k <= (low ? i - 1 : j); ++k)
                        t.terms.push_back({{0, d, toff(d, i, k)}, {sp, f, ioff(f, k, j)}, md, mf, lm(k), 0, 0, 1.0});
                    fin_tt[dd - 1].push_back(t);
                    VTask x{{sp, f, ioff(f, i, j)}, mf, lm(i), lm(j), 0.0, {}};
                    x.terms.push_back({{sp, f, ioff(f, i, i)}, {3, 0, scr}, mf, lm(i), lm(i), 0, 0, -1.0});
                    fin_tx[dd - 1].push_back(x);
                    scr += (int64_t)lm(i) * lm(j);
                }
        }
    }
    // ---- exact descriptor counts -> device arrays and the pinned staging buffer
    size_t n_pan = 0, n_task = 0, n_term = 0, n_tile = 0, n_cp = 0, n_te = 0, n_tc = 0;
    auto cnt_tasks = [&](const std::vector<VTask>& v, int shape) {
        static const int shm[6] = {64, 32, 128, 16, 128, 64}, shn[6] = {64, 32, 16, 16, 64, 128};
        for (auto& t : v) {
            ++n_task;
            n_term += t.terms.size();
            n_tile += (size_t)(ceil_div(t.m, shm[shape]) * ceil_div(t.n, shn[shape]));
        }
    };
    auto cnt_trunc = [&](const std::vector<VTrunc>& v) {
        for (auto& e : v) {
            ++n_te;
            n_tc += (size_t)(ceil_div(S.bl[e.blk].m, TRUNC_CHUNK) + ceil_div(S.bl[e.blk].n, TRUNC_CHUNK));
        }
    };
    auto cnt_pan = [&](const std::vector<VPanel>& v) {   // (8: the narrowest inverse strip, FDE_H2_INV_STRIP)
        for (auto& q : v) n_pan += (size_t)ceil_div(q.nvec, q.Ti.sp < 0 ? 8 : H2_STRIP);
    };
    auto cnt_cp = [&](const std::vector<VCopy>& v) {
        for (auto& c : v) {
            if (c.m <= 0 || c.n <= 0) continue;
            if (c.kind == 2 || (int64_t)c.m * c.n <= H2_CP_CHUNK) {
                ++n_cp;
                continue;
            }
            const int rm = std::min(c.m, H2_CP_CHUNK), cn = std::max(1, H2_CP_CHUNK / rm);
            n_cp += (size_t)(ceil_div(c.n, cn) * ceil_div(c.m, rm));
        }
    };
    cnt_cp(init_cp);
    cnt_trunc(init_trunc);
    for (auto& st : steps) {
        cnt_trunc(st.trunc);
        cnt_trunc(st.trunc_ov);
        cnt_pan(st.panel);
        cnt_pan(st.npanel);
        cnt_tasks(st.g0, gemm_shape[3]);
        cnt_tasks(st.g1, gemm_shape[0]);
        cnt_tasks(st.g2, gemm_shape[1]);
        cnt_tasks(st.g3, 1);   // (crit / rest / diag: at most the tiles of the 32 x 32 shape)
        for (auto& dt : st.dts) {   // compact dense work (expanded later): one term, at most one task per tile
            const auto& dp = st.dpairs[dt.first];
            const int t = dt.second;
            const int k = (int)(&st - &steps[0]);
            const int64_t ni = std::max(0, std::min(t1[dp.b], t1[t]) - std::max(std::max(t0[dp.b], t0[t]), k + 1) + 1);
            const int64_t nj = std::max(0, std::min(s1[dp.c], s1[t]) - std::max(std::max(s0[dp.c], s0[t]), k + 1) + 1);
            n_term += (size_t)(ni * nj);
            n_task += (size_t)(ni * nj);
            n_tile += (size_t)(ni * nj) * ceil_div(H2_MMAX, 32) * ceil_div(H2_MMAX, 32);
        }
        for (auto& v : st.cpr) cnt_cp(v);
        cnt_cp(st.snap);
        for (auto& v : st.trmid) cnt_trunc(v);
    }
    cnt_cp(fin_cp);
    cnt_pan(fin_pv);
    for (auto& v : fin_tt) cnt_tasks(v, 0);
    for (auto& v : fin_tx) cnt_tasks(v, 0);
    vlu.reserve(nl); vpan.reserve(n_pan); vterm.reserve(n_term); vtask.reserve(n_task);
    vtile.reserve(n_tile); vcp.reserve(n_cp); vte.reserve(n_te); vtc.reserve(n_tc);
    P->lu.alloc(std::max<size_t>(nl, 1));
    P->pan.alloc(std::max<size_t>(n_pan, 1));
    P->terms.alloc(std::max<size_t>(n_term, 1));
    P->tasks.alloc(std::max<size_t>(n_task, 1));
    P->tiles.alloc(std::max<size_t>(n_tile, 1));
    P->cps.alloc(std::max<size_t>(n_cp, 1));
    P->te.alloc(std::max<size_t>(n_te, 1));
    P->tc.alloc(std::max<size_t>(n_tc, 1));
    // staged uploads: every phase's new descriptors go host -> pinned -> device on a
    // copy stream, so the host flattens step k+1 while the device runs step k
    struct Stage {
        const void* src;   // host vector data (capacity reserved: never reallocated)
        size_t elem, done;
        void* dev;
        size_t pin;        // byte offset in the pinned buffer
    };
    auto al16 = [](size_t b) { return (b + 15) & ~(size_t)15; };
    Stage stg[8] = {{vlu.data(), sizeof(H2Lu), 0, P->lu.p, 0},       {vpan.data(), sizeof(H2Panel), 0, P->pan.p, 0},
                    {vterm.data(), sizeof(H2Term), 0, P->terms.p, 0}, {vtask.data(), sizeof(H2Task), 0, P->tasks.p, 0},
                    {vtile.data(), sizeof(H2Tile), 0, P->tiles.p, 0}, {vcp.data(), sizeof(H2Copy), 0, P->cps.p, 0},
                    {vte.data(), sizeof(TEntry), 0, P->te.p, 0},      {vtc.data(), sizeof(TChunk), 0, P->tc.p, 0}};
    const size_t cap[8] = {(size_t)nl, n_pan, n_term, n_task, n_tile, n_cp, n_te, n_tc};
    size_t pin_bytes = 0;
    for (int a = 0; a < 8; ++a) {
        stg[a].pin = pin_bytes;
        pin_bytes += al16(cap[a] * stg[a].elem);
    }
    char* pin = (char*)ctx_stage(L->h, pin_bytes);
    // sa: high-priority internal stream ordered after the caller's stream s (and s
    // after sa at the end): the critical chain must not queue behind bulk updates
    cudaStream_t sa = aux_stream5(L->h), sb = aux_stream(L->h), sc = aux_stream2(L->h), sd = aux_stream3(L->h);
    cudaStream_t sl = aux_stream4(L->h);   // the diagonal-tile LUs
    cudaEvent_t evS = L->h->ev_aux[9];
    FDE_CUDA(cudaEventRecord(evS, s));
    FDE_CUDA(cudaStreamWaitEvent(sa, evS, 0));
    cudaEvent_t evA = L->h->ev_aux[0], evOp = L->h->ev_aux[1];
    cudaEvent_t evP = L->h->ev_aux[3], evC = L->h->ev_aux[4], evB = L->h->ev_aux[5], evD = L->h->ev_aux[6];
    cudaEvent_t evLU = L->h->ev_aux[7], evDg = L->h->ev_aux[8];
    cudaEvent_t evCp = L->h->ev_aux[10], evOv = L->h->ev_aux[11];
    cudaEvent_t evPan = L->h->ev_aux[12], evSnap = L->h->ev_aux[13];
    cudaEvent_t evNP = L->h->ev_aux[14], evCrit = L->h->ev_aux[15];
    cudaStream_t se = aux_stream6(L->h);   // overflow truncations
    cudaStream_t si = aux_stream7(L->h);   // tile inverses (np_subst)
    cudaEvent_t evLUo = L->h->ev_aux[16], evInv = L->h->ev_aux[17];
    // operand snapshots on a stream of their own, right after the operand
    // truncations (they read nothing the panels / products write), so they leave
    // the t -> panels -> products -> t chain (FDE_H2_SNAP_EARLY=0: after the products)
    const bool snap_early = !(getenv("FDE_H2_SNAP_EARLY") && atoi(getenv("FDE_H2_SNAP_EARLY")) == 0);
    cudaStream_t ss = aux_stream8(L->h);
    // SM partition (FDE_H2_GREEN = SMs of the bulk dense updates, multiple of 8; 0: off)
    if (const char* g = getenv("FDE_H2_GREEN")) {
        const int nbulk = atoi(g);
        if (nbulk > 0 && h2_green_streams(L->h, nbulk)) {
            sc = L->h->g_bulk;
            if (!(getenv("FDE_H2_GREEN_CHAIN") && atoi(getenv("FDE_H2_GREEN_CHAIN")) == 0)) {
                sa = L->h->g_chain[0];
                sb = L->h->g_chain[1];
                sl = L->h->g_chain[2];
                se = L->h->g_chain[3];
                si = L->h->g_chain[4];
                ss = L->h->g_chain[5];
            }
        }
    }
    // debug: fold auxiliary streams back onto the critical one (race bisection)
    if (const char* f = getenv("FDE_H2_FOLD")) {
        const std::string fs(f);
        if (fs.find('c') != std::string::npos) sc = sa;
        if (fs.find('e') != std::string::npos) se = sb;
        if (fs.find('l') != std::string::npos) sl = sa;
        if (fs.find('b') != std::string::npos) sb = sa;
        if (fs.find('a') != std::string::npos) { sb = sa; sc = sa; se = sa; sl = sa; }
    }
    FDE_CUDA(cudaEventRecord(evA, sa));   // (sa is ordered after the arena / descriptor allocations on s)
    FDE_CUDA(cudaStreamWaitEvent(sd, evA, 0));
    const bool sync_push = getenv("FDE_H2_SYNCPUSH") != nullptr;   // debug
    auto sizes_now = [&](size_t* now) {
        const size_t v[8] = {vlu.size(), vpan.size(), vterm.size(), vtask.size(),
                             vtile.size(), vcp.size(), vte.size(), vtc.size()};
        for (int a = 0; a < 8; ++a) now[a] = v[a];
    };
    auto push = [&](const size_t* given = nullptr) {
        size_t now[8];
        if (given) for (int a = 0; a < 8; ++a) now[a] = given[a];
        else sizes_now(now);
        for (int a = 0; a < 8; ++a)
            if (now[a] > cap[a]) fde_fail(FDE_EINVAL_PARAM, "hlu_factor: descriptor count exceeds the plan (internal)");
        for (int a = 0; a < 8; ++a) {
            if (now[a] == stg[a].done) continue;
            const size_t off = stg[a].done * stg[a].elem, bytes = (now[a] - stg[a].done) * stg[a].elem;
            memcpy(pin + stg[a].pin + off, (const char*)stg[a].src + off, bytes);
            FDE_CUDA(cudaMemcpyAsync((char*)stg[a].dev + off, pin + stg[a].pin + off, bytes, cudaMemcpyHostToDevice, sd));
            stg[a].done = now[a];
        }
        FDE_CUDA(cudaEventRecord(evD, sd));
        if (sync_push) FDE_CUDA(cudaStreamSynchronize(sd));
    };
    const double ms_flat0 = ms_since(t_flat0);
    L->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_plan0).count();

    // ---- execute.  Three streams.  sa: the critical chain LU(k) -> panels ->
    // products -> conversions -> dense updates of row / column k+1 (needed by step
    // k+1); sb: truncations (operands before the panels, overflowing targets before
    // the new columns) and the new low-rank columns; sc: the remaining dense updates
    // of step k, which overlap LU(k+1) and the panels of step k+1 (lookahead).
    const int pan_smem = (H2_STRIP + 64) * (H2_MMAX + 2) * (int)sizeof(double);   // (two 32-column block panels)
    set_smem_once((const void*)k_h2_panel, pan_smem);
    const int pan_smem_inv = (H2_STRIP + 2 * H2_PCH) * (H2_MMAX + 16) * (int)sizeof(double);   // (double-buffered op)
    const int lu_smem = H2_MMAX * (H2_MMAX + 1) * (int)sizeof(double);   // padded 128 x 129
    set_smem_once((const void*)k_h2_lu, lu_smem);
    static const bool use_dmma = !getenv("FDE_H2_NODMMA");
    set_smem_once((const void*)k_h2_gemm<64, 64, true>, H2G_SMEM(64, 64));
    set_smem_once((const void*)k_h2_gemm<128, 16, true>, H2G_SMEM(128, 16));
    set_smem_once((const void*)k_h2_gemm<32, 32, true>, H2G_SMEM(32, 32));
    set_smem_once((const void*)k_h2_gemm<16, 16, true>, H2G_SMEM(16, 16));
    set_smem_once((const void*)k_h2_gemm<64, 64, false>, H2G_SMEM(64, 64));
    set_smem_once((const void*)k_h2_gemm<128, 16, false>, H2G_SMEM(128, 16));
    set_smem_once((const void*)k_h2_gemm<32, 32, false>, H2G_SMEM(32, 32));
    set_smem_once((const void*)k_h2_gemm<16, 16, false>, H2G_SMEM(16, 16));
    set_smem_once((const void*)k_h2_gemm<128, 64, true>, H2G_SMEM(128, 64));
    set_smem_once((const void*)k_h2_gemm<64, 128, true>, H2G_SMEM(64, 128));
    set_smem_once((const void*)k_h2_gemm<128, 64, false>, H2G_SMEM(128, 64));
    set_smem_once((const void*)k_h2_gemm<64, 128, false>, H2G_SMEM(64, 128));
    int nlaunch = 0;
    // FDE_DEBUG_SERIAL: synchronise after every launch and name the first failing one
    const bool dbg_serial = getenv("FDE_DEBUG_SERIAL") != nullptr;
    // debug switches in __device__ variables: copied only when they change (a copy from
    // pageable host memory waits for the stream to drain -- here, for the assembly and
    // the H-matrix build -- so the host could not run ahead into the first steps)
    {
        static int set_dev[64] = {};   // per device: 1 + (check << 1) + (serial << 2)
        const int on = getenv("FDE_H2_CHECK") ? 1 : 0;
        const int chk = dbg_serial ? 1 : 0;
        int dev = 0;
        FDE_CUDA(cudaGetDevice(&dev));
        const int state = 1 + (on << 1) + (chk << 2);
        if (on) {   // (the bounds checks need this factorisation's arena: every time)
            const char* lo[4] = {(const char*)A, (const char*)hm->dense.p, (const char*)hm->lr.p, nullptr};
            const char* hi[4] = {(const char*)(A + words), (const char*)(hm->dense.p + hm->dense.n),
                                 (const char*)(hm->lr.p + hm->lr.n), nullptr};
            FDE_CUDA(cudaMemcpyToSymbolAsync(g_h2_lo, lo, sizeof(lo), 0, cudaMemcpyHostToDevice, sa));
            FDE_CUDA(cudaMemcpyToSymbolAsync(g_h2_hi, hi, sizeof(hi), 0, cudaMemcpyHostToDevice, sa));
        }
        if (set_dev[dev & 63] != state) {
            FDE_CUDA(cudaMemcpyToSymbolAsync(g_h2_check, &on, sizeof(int), 0, cudaMemcpyHostToDevice, sa));
            FDE_CUDA(cudaMemcpyToSymbolAsync(g_trunc_check, &chk, sizeof(int), 0, cudaMemcpyHostToDevice, sa));
            static const double jeps = getenv("FDE_TRUNC_JEPS") ? atof(getenv("FDE_TRUNC_JEPS")) : 0.0;
            FDE_CUDA(cudaMemcpyToSymbolAsync(g_trunc_jeps, &jeps, sizeof(double), 0, cudaMemcpyHostToDevice, sa));
            FDE_CUDA(cudaStreamSynchronize(sa));   // (the host values are stack / static: copied before use)
            set_dev[dev & 63] = state;
        }
    }
    int dbg_step = -1;
    auto dbg = [&](const char* what) {
        if (!dbg_serial) return;
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            fprintf(stderr, "hlu2 debug: %s at step %d failed: %s\n", what, dbg_step, cudaGetErrorString(e));
            fde_fail(FDE_ECUDA, std::string("hlu2 debug: ") + what + ": " + cudaGetErrorString(e));
        }
    };
    auto run_copy = [&](const H2Launch& ln, cudaStream_t st) {
        if (!ln.ncp) return;
        k_h2_copy<<<ln.ncp, 256, 0, st>>>(P->cps.p + ln.cp0);
        FDE_CHECK_LAUNCH();
        ++nlaunch;
        dbg("copy");
    };
    std::function<void(int)> tmark = [](int) {};
    // programmatic dependent launches (FDE_H2_PDL=0: off) for the kernels that follow
    // another kernel of the same stream on the binding chain (truncation core and
    // apply behind the Gram partials, the product groups behind the panels)
    const bool use_pdl = !(getenv("FDE_H2_PDL") && atoi(getenv("FDE_H2_PDL")) == 0);
    auto run_trunc = [&](const H2Trunc& tr, cudaStream_t st, int ws) {
        if (!tr.ne) return;
        const TEntry* E = P->te.p + tr.e0;
        const TChunk* C = P->tc.p + tr.c0;
        double* part = ws ? P->tr_part2 : P->tr_part;
        double* Tt = ws ? P->tr_T2 : P->tr_T;
        k_bgram<<<tr.nc, 256, 0, st>>>(E, C, part);
        FDE_CHECK_LAUNCH();
        dbg("bgram");
        if (!ws) tmark(0);
        const int kmax = tr.kmax;
        launch_pdl(use_pdl, k_bcore, tr.ne, BCORE_THREADS, 0, st, E, C, part, L->tol, rmax, Tt, L->dflag.p + 1,
                   ws ? P->tr_scr2 : P->tr_scr);
        FDE_CHECK_LAUNCH();
        dbg("bcore");
        if (!ws) tmark(1);
        const size_t asmem = (size_t)(kmax * rmax + TRUNC_CHUNK * kmax) * sizeof(double);
        set_smem_once((const void*)k_bapply, (int)asmem);
        launch_pdl(use_pdl, k_bapply, tr.nc, 256, asmem, st, E, C, (const double*)Tt, rmax);
        FDE_CHECK_LAUNCH();
        dbg("bapply");
        nlaunch += 3;
    };
    static const bool lu_old = getenv("FDE_H2_LU_OLD") != nullptr;
    // debug (critical-path analysis only: results are garbage): FDE_H2_SKIP lists launch
    // classes to leave out -- l LU, i tile inverses, n neighbour panels, d diagonal-tile
    // update, p panels, g products, s snapshots, x row/column k+1 update, r other
    // updates, t operand truncations, o overflow truncations, c new columns
    const std::string skipset = getenv("FDE_H2_SKIP") ? getenv("FDE_H2_SKIP") : "";
    auto skip = [&](char c) { return skipset.find(c) != std::string::npos; };
    // debug (sensitivity analysis, results intact): FDE_H2_DELAY=c:us adds a us-long
    // one-thread spin behind every launch of class c on its stream; the growth of the
    // step period per added us says how far that class sits on the binding chain
    const char* dly_e = getenv("FDE_H2_DELAY");
    const char dly_c = (dly_e && dly_e[0] && dly_e[1] == ':') ? dly_e[0] : 0;
    const long long dly_us = dly_c ? atoll(dly_e + 2) : 0;
    auto delay = [&](char c, cudaStream_t st) {
        if (c != dly_c || dly_us <= 0) return;
        k_h2_spin<<<1, 1, 0, st>>>(dly_us);
        FDE_CHECK_LAUNCH();
    };
    auto launch_lu = [&](int kk, cudaStream_t st) {   // LU of tile kk, then the inverses of its factors
        const H2Lu* t = P->lu.p + P->steps[kk].lu;
        if (skip('l')) {
        } else if (lu_old) k_h2_lu<<<1, 512, lu_smem, st>>>(t, L->dflag.p);
        else k_h2_lu_reg<<<1, 512, 0, st>>>(t, L->dflag.p);
        FDE_CHECK_LAUNCH();
        delay('l', st);
        if (P->steps[kk].npi) {
            cudaStream_t sv = st;
            if (np_subst) {
                FDE_CUDA(cudaEventRecord(evLUo, st));
                FDE_CUDA(cudaStreamWaitEvent(si, evLUo, 0));
                sv = si;
            }
            if (!skip('i')) k_h2_panel<<<P->steps[kk].npi, 256, pan_smem, sv>>>(P->pan.p + P->steps[kk].pi0);
            FDE_CHECK_LAUNCH();
            delay('i', sv);
            ++nlaunch;
            if (np_subst) FDE_CUDA(cudaEventRecord(evInv, si));
        }
    };
    int gemm_cap[6];
    for (int w = 0; w < 6; ++w) gemm_cap[w] = 1 << 30;
    {
        const char* e = getenv("FDE_H2_REST_CTAS");
        gemm_cap[4] = e ? std::max(1, atoi(e)) : gemm_cap[4];
    }
    const int rest_smem = getenv("FDE_H2_REST_SMEM") ? std::max(H2G_SMEM(64, 64), atoi(getenv("FDE_H2_REST_SMEM"))) : 0;
    if (rest_smem > 0) {
        FDE_CUDA(cudaFuncSetAttribute(k_h2_gemm<64, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, rest_smem));
        FDE_CUDA(cudaFuncSetAttribute(k_h2_gemm<64, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, rest_smem));
    }
    auto run_gemm = [&](const H2Launch& ln, int w, cudaStream_t st, bool pdl = false) {
        pdl = pdl && use_pdl;
        if (!ln.g_ntile[w]) return;
        const int grid = std::min(ln.g_ntile[w], gemm_cap[w]);
        const H2Tile* tl = P->tiles.p + ln.g_tile0[w];
#define H2G_LAUNCH(TM_, TN_)                                                                                   \
    (use_dmma ? launch_pdl(pdl, k_h2_gemm<TM_, TN_, true>, grid, 256, H2G_SMEM(TM_, TN_), st, tl, P->tasks.p, P->terms.p, ln.g_ntile[w]) \
              : launch_pdl(pdl, k_h2_gemm<TM_, TN_, false>, grid, 256, H2G_SMEM(TM_, TN_), st, tl, P->tasks.p, P->terms.p, ln.g_ntile[w]))
        switch (ln.g_shape[w]) {
            case 0: if (w == 4 && rest_smem > 0) {   // (debug FDE_H2_REST_SMEM: fewer bulk-update CTAs per SM)
                        launch_pdl(false, use_dmma ? k_h2_gemm<64, 64, true> : k_h2_gemm<64, 64, false>, grid, 256,
                                   rest_smem, st, tl, P->tasks.p, P->terms.p, ln.g_ntile[w]);
                        break;
                    }
                    H2G_LAUNCH(64, 64); break;
            case 1: H2G_LAUNCH(32, 32); break;
            case 2: H2G_LAUNCH(128, 16); break;
            case 3: H2G_LAUNCH(16, 16); break;
            case 4: H2G_LAUNCH(128, 64); break;   // (debug shapes: bulk tiles of 128 x 64 / 64 x 128)
            case 5: H2G_LAUNCH(64, 128); break;
            default: H2G_LAUNCH(64, 64);
        }
#undef H2G_LAUNCH
        FDE_CHECK_LAUNCH();
        ++nlaunch;
        static const char* gname[6] = {"gemm cores", "gemm products", "gemm crit", "gemm conversions", "gemm rest",
                                       "gemm diag"};
        dbg(gname[w]);
    };
    auto run_panel = [&](const H2Launch& ln) {
        if (!ln.npan) return;
        k_h2_panel<<<ln.npan, 256, (&ln != &P->fin && pan_inv) ? pan_smem_inv : pan_smem, sa>>>(P->pan.p + ln.pan0);
        FDE_CHECK_LAUNCH();
        ++nlaunch;
        dbg("panel");
    };
    // init (+ every diagonal-tile LU descriptor: LU(k+1) is issued during step k)
    if (pan_inv) init_cp.insert(init_cp.end(), fin_cp.begin(), fin_cp.end());   // identities of the tile inverses
    put_copy(init_cp, P->init);
    put_trunc(init_trunc, P->init.tr);
    P->steps.resize(nl);
    for (int k = 0; k < nl; ++k) {
        P->steps[k].lu = (int)vlu.size();
        vlu.push_back({A + offD[steps[k].lu_blk] + steps[k].lu_off, S.bl[steps[k].lu_blk].m, lm(k)});
        if (pan_inv) {
            H2Launch tmp;
            put_panel({fin_pv[2 * k], fin_pv[2 * k + 1]}, tmp);
            P->steps[k].pi0 = tmp.pan0;
            P->steps[k].npi = tmp.npan;
        }
    }
    push();
    FDE_CUDA(cudaMemsetAsync(A + lr_lo, 0, (size_t)(lr_hi - lr_lo) * sizeof(double), sa));
    if (pan_inv) FDE_CUDA(cudaMemsetAsync(A + inv_lo, 0, (size_t)(inv_hi - inv_lo) * sizeof(double), sa));
    FDE_CUDA(cudaStreamWaitEvent(sa, evD, 0));
    if (const char* e = getenv("FDE_H2_HOLD_US")) {   // debug: hold the device while the host enqueues
        k_h2_spin<<<1, 1, 0, sa>>>(atoll(e));          // (the timeline then shows the device-bound period)
        FDE_CHECK_LAUNCH();
    }
    run_copy(P->init, sa);
    run_trunc(P->init.tr, sa, 0);
    FDE_CUDA(cudaEventRecord(evA, sa));
    FDE_CUDA(cudaStreamWaitEvent(sb, evA, 0));
    FDE_CUDA(cudaStreamWaitEvent(sc, evA, 0));
    FDE_CUDA(cudaStreamWaitEvent(sl, evA, 0));
    FDE_CUDA(cudaStreamWaitEvent(se, evA, 0));
    FDE_CUDA(cudaEventRecord(evC, sc));
    const int kstop = g_hlu2_stop >= 0 ? std::min(g_hlu2_stop, nl) : nl;   // debug: partial sweep
    // debug timeline (FDE_DEBUG_TIMELINE): timed events per step and stream
    const bool tline = getenv("FDE_DEBUG_TIMELINE") != nullptr;
    const bool skip_rest = getenv("FDE_H2_SKIPREST") != nullptr;
    enum { T_LU = 0, T_PAN, T_PROD, T_CRIT, T_OP, T_OV, T_CP, T_REST, T_SNAP, T_DIAG, T_G1, T_G2, T_GRAM, T_CORE, T_PUSH, T_N };
    std::vector<cudaEvent_t> tev;
    std::vector<double> thost;
    double eq_us[3] = {0, 0, 0};   // host: flatten, push, launches (timeline mode)
    double fl_us[3] = {0, 0, 0};   // flatten: plan lists, dense-target expansion, split + dense tasks
    const auto th0 = std::chrono::steady_clock::now();
    cudaEvent_t t0ev = nullptr;
    if (tline) {
        tev.resize((size_t)kstop * T_N);
        for (auto& e : tev) FDE_CUDA(cudaEventCreate(&e));
        FDE_CUDA(cudaEventCreate(&t0ev));
        FDE_CUDA(cudaEventRecord(t0ev, sa));
    }
    std::vector<int> xtile_stamp((size_t)nl * nl, 0), xtile_task((size_t)nl * nl, 0);   // (flatten-time tile -> task)
    int xtile_stamp_id = 0;
    std::vector<VTask> xg3;    // the expanded dense-target tasks of the current step (capacity reused)
    std::vector<char> xg3c;
    auto mark = [&](int k, int w, cudaStream_t st) {
        if (tline) FDE_CUDA(cudaEventRecord(tev[(size_t)k * T_N + w], st));
    };
    // flatten of step k: the host descriptor lists of step k (writes only P->steps[k],
    // the descriptor vectors -- capacity reserved, never reallocated -- and the
    // flatten scratch)
    auto flatten = [&](int k, std::chrono::steady_clock::time_point te0) {
        // flatten step k (the device is still busy with step k-1) and stage it
        H2Launch& ln = P->steps[k];
        VStep& st = steps[k];
        put_trunc(st.trunc, ln.tr);
        put_trunc(st.trunc_ov, ln.tr_ov);
        put_panel(st.panel, ln);
        {
            H2Launch tmp;
            put_panel(st.npanel, tmp);
            ln.np0 = tmp.pan0;
            ln.nnp = tmp.npan;
        }
        put_gemm(st.g0, ln, 3, gemm_shape[3]);
        put_gemm(st.g1, ln, 0, gemm_shape[0]);
        put_gemm(st.g2, ln, 1, gemm_shape[1]);
        {
            H2Launch tmp;
            put_copy(st.snap, tmp);
            ln.snap0 = tmp.cp0;
            ln.nsnap = tmp.ncp;
        }
        ln.cpr.clear();
        ln.trmid.clear();
        for (size_t r = 0; r < st.cpr.size(); ++r) {
            H2Launch tmp;
            put_copy(st.cpr[r], tmp);
            ln.cpr.push_back({tmp.cp0, tmp.ncp});
            if (r < st.trmid.size()) {
                ln.trmid.emplace_back();
                put_trunc(st.trmid[r], ln.trmid.back());
            }
        }
        const auto tf1 = std::chrono::steady_clock::now();
        xg3.clear();
        xg3c.clear();
        if (!st.dts.empty()) {   // expand the compact dense-target work of the plan (same order as before)
            ++xtile_stamp_id;
            const int sid = st.sid, mk = st.mk;
            for (size_t q = 0; q < st.dts.size(); ++q) {
                const auto& dp = st.dpairs[st.dts[q].first];
                const int t = st.dts[q].second, b = dp.b, c = dp.c;
                const HBlock &T = S.bl[t], &B = S.bl[b], &C = S.bl[c];
                for (int i = std::max(std::max(t0[b], t0[t]), k + 1); i <= std::min(t1[b], t1[t]); ++i)
                    for (int j = std::max(std::max(s0[c], s0[t]), k + 1); j <= std::min(s1[c], s1[t]); ++j) {
                        const size_t key = (size_t)i * nl + j;
                        int ti;
                        if (xtile_stamp[key] != xtile_stamp_id) {
                            ti = (int)xg3.size();
                            xtile_stamp[key] = xtile_stamp_id;
                            xtile_task[key] = ti;
                            xg3.push_back(VTask{{0, t, (lr0[j] - col0(t)) * T.m + (lr0[i] - row0(t))}, T.m, lm(i), lm(j), 1.0, {}});
                            xg3c.push_back((i == k + 1 && j == k + 1) ? 2
                                                : (i == k + 1 || j == k + 1 || (i == k + 2 && j == k + 2)));
                        } else {
                            ti = xtile_task[key];
                        }
                        VTerm term;
                        if (!dp.bl && !dp.cl) {
                            term = {{0, b, (lr0[k] - col0(b)) * B.m + (lr0[i] - row0(b))},
                                    {0, c, (lr0[j] - col0(c)) * C.m + (lr0[k] - row0(c))}, B.m, C.m, mk, 0, 0, -1.0};
                        } else if (dp.bl) {   // U_b[i rows] W[j rows]^T
                            term = {{3, sid, dp.su + (lr0[i] - row0(b))}, {3, sid, dp.w + (lr0[j] - col0(c))}, B.m, C.n,
                                    dp.kcb, 0, 1, -1.0};
                        } else {               // Z[i rows] V_c[j rows]^T
                            term = {{3, sid, dp.w + (lr0[i] - row0(b))}, {3, sid, dp.sv + (lr0[j] - col0(c))}, B.m, C.n,
                                    dp.kcc, 0, 1, -1.0};
                        }
                        xg3[ti].terms.push_back(term);
                    }
            }
        }
        const auto tf2 = std::chrono::steady_clock::now();
        if (tline) {
            fl_us[0] += std::chrono::duration<double, std::micro>(tf1 - te0).count();
            fl_us[1] += std::chrono::duration<double, std::micro>(tf2 - tf1).count();
        }
        {   // split the dense updates: row / column k+1 (needed by step k+1) vs the rest
            // (selected in place: no task moves)
            ln.diag_scr = false;
            for (size_t q = 0; q < st.g3.size(); ++q)
                if (st.g3crit[q] == 2)
                    for (auto& tm : st.g3[q].terms) ln.diag_scr |= tm.A.sp == 3 || tm.B.sp == 3;
            for (size_t q = 0; q < xg3.size(); ++q)
                if (xg3c[q] == 2)
                    for (auto& tm : xg3[q].terms) ln.diag_scr |= tm.A.sp == 3 || tm.B.sp == 3;
            put_gemm_sel(st.g3, &st.g3crit, 1, ln, 2, gemm_shape[2], &xg3, &xg3c);
            put_gemm_sel(st.g3, &st.g3crit, 0, ln, 4, gemm_shape[4], &xg3, &xg3c);
            put_gemm_sel(st.g3, &st.g3crit, 2, ln, 5, gemm_shape[5], &xg3, &xg3c);
        }
    };
    // host pipeline (FDE_H2_PIPE, default on; the debug timeline turns it off): a
    // worker thread flattens the steps ahead of this thread, which pushes step k's
    // descriptors as soon as the worker has published their counts.  The vectors
    // never reallocate (capacity = the plan's exact counts; checked), so [done,
    // size_k) is final once published and the worker only appends past it.
    const bool pipe = !(getenv("FDE_H2_PIPE") && atoi(getenv("FDE_H2_PIPE")) == 0) && !tline && kstop > 1;
    std::vector<size_t> step_sz((size_t)std::max(kstop, 1) * 8);
    std::atomic<int> flat_done{0};
    std::exception_ptr flat_err;
    std::thread flat_worker;
    auto stg_src = [&](int a) -> const void* {
        const void* d[8] = {vlu.data(), vpan.data(), vterm.data(), vtask.data(),
                            vtile.data(), vcp.data(), vte.data(), vtc.data()};
        return d[a];
    };
    struct Joiner {
        std::thread& t;
        ~Joiner() { if (t.joinable()) t.join(); }
    } flat_join{flat_worker};
    if (pipe) {
        flat_worker = std::thread([&]() {
            try {
                for (int k = 0; k < kstop; ++k) {
                    flatten(k, std::chrono::steady_clock::now());
                    size_t* szk = &step_sz[(size_t)k * 8];
                    sizes_now(szk);
                    for (int a = 0; a < 8; ++a)
                        if (szk[a] > cap[a] || (szk[a] && stg_src(a) != stg[a].src))
                            fde_fail(FDE_EINVAL_PARAM, "hlu_factor: descriptor count exceeds the plan (internal)");
                    flat_done.store(k + 1, std::memory_order_release);
                }
            } catch (...) {
                flat_err = std::current_exception();
                flat_done.store(INT_MAX, std::memory_order_release);
            }
        });
    }
    for (int k = 0; k < kstop; ++k) {
        dbg_step = k;
        const auto te0 = std::chrono::steady_clock::now();
        size_t* szk = &step_sz[(size_t)k * 8];
        if (pipe) {
            int got;
            while ((got = flat_done.load(std::memory_order_acquire)) <= k) std::this_thread::yield();
            if (got == INT_MAX) break;   // the worker failed: rethrown below
        } else {
            flatten(k, te0);
            sizes_now(szk);
        }
        H2Launch& ln = P->steps[k];
        const auto te1 = std::chrono::steady_clock::now();
        push(szk);
        const auto te2 = std::chrono::steady_clock::now();
        mark(k, T_PUSH, sd);
        dbg("push");
        FDE_CUDA(cudaStreamWaitEvent(sa, evD, 0));
        FDE_CUDA(cudaStreamWaitEvent(sb, evD, 0));
        FDE_CUDA(cudaStreamWaitEvent(sc, evD, 0));
        FDE_CUDA(cudaStreamWaitEvent(sl, evD, 0));
        FDE_CUDA(cudaStreamWaitEvent(se, evD, 0));
        // sb (after the new columns of step k-1 and the panels of step k-1)
        // se: overflow truncations, concurrently with the operand truncations (the
        // blocks are disjoint); they only have to precede this step's new columns
        FDE_CUDA(cudaEventRecord(evCp, sb));
        FDE_CUDA(cudaStreamWaitEvent(se, evCp, 0));
        FDE_CUDA(cudaStreamWaitEvent(se, evSnap, 0));   // snapshots of step k-1 taken
        FDE_CUDA(cudaStreamWaitEvent(se, evP, 0));      // products of step k-1 done (their operands)
        if (!skip('o')) run_trunc(ln.tr_ov, se, 1);
        delay('o', se);
        FDE_CUDA(cudaEventRecord(evOv, se));
        mark(k, T_OV, se);
        FDE_CUDA(cudaStreamWaitEvent(sb, evSnap, 0));
        if (tline) tmark = [&](int w) { mark(k, w ? T_CORE : T_GRAM, sb); };
        if (!skip('t')) run_trunc(ln.tr, sb, 0);
        delay('t', sb);
        tmark = [](int) {};
        FDE_CUDA(cudaEventRecord(evOp, sb));
        mark(k, T_OP, sb);
        if (snap_early) {
            // ss: snapshots of this step's operand factors once they are truncated; the
            // ring scratch they fill was last read by the bulk updates of step k-2,
            // which precede the row / column update of step k-1 (evCrit)
            FDE_CUDA(cudaStreamWaitEvent(ss, evOp, 0));
            FDE_CUDA(cudaStreamWaitEvent(ss, evCrit, 0));
            FDE_CUDA(cudaStreamWaitEvent(ss, evD, 0));
            if (ln.nsnap && !skip('s')) {
                k_h2_copy<<<ln.nsnap, 256, 0, ss>>>(P->cps.p + ln.snap0);
                FDE_CHECK_LAUNCH();
                ++nlaunch;
                dbg("snapshots");
            }
            delay('s', ss);
            FDE_CUDA(cudaEventRecord(evSnap, ss));
        }
        // sa: critical chain.  LU(k) ran on sl (k = 0: here), overlapping the
        // products and updates of step k-1; its only input from step k-1 is the
        // update of the diagonal tile, issued on sl right after the panels of step k-1.
        if (k == 0) {
            launch_lu(k, sl);
            FDE_CHECK_LAUNCH();
            ++nlaunch;
            FDE_CUDA(cudaEventRecord(evLU, sl));
        }
        FDE_CUDA(cudaStreamWaitEvent(sa, evLU, 0));
        if (np_subst) FDE_CUDA(cudaStreamWaitEvent(sa, evInv, 0));
        FDE_CUDA(cudaStreamWaitEvent(sa, evOp, 0));
        auto diag_lu = [&](cudaStream_t st) {   // tile (k+1, k+1), then LU(k+1) on sl
            if (!skip('d')) run_gemm(ln, 5, st);
            delay('d', st);
            mark(k, T_DIAG, st);
            if (k + 1 < kstop) {
                if (st != sl) {
                    FDE_CUDA(cudaEventRecord(evDg, st));
                    FDE_CUDA(cudaStreamWaitEvent(sl, evDg, 0));
                }
                launch_lu(k + 1, sl);
                FDE_CHECK_LAUNCH();
                ++nlaunch;
                dbg("lu");
                FDE_CUDA(cudaEventRecord(evLU, sl));
                mark(k, T_LU, sl);
            }
        };
        // (sa has captured evLU = LU(k) above; LU(k+1) may be recorded from here on)
        if (ln.nnp) {   // neighbour-tile panels, tile (k+1, k+1), LU(k+1): all on the LU stream
            FDE_CUDA(cudaStreamWaitEvent(sl, evCrit, 0));   // row / column k updated by step k-1
            if (!skip('n')) k_h2_panel<<<ln.nnp, 256, (pan_inv && !np_subst) ? pan_smem_inv : pan_smem, sl>>>(P->pan.p + ln.np0);
            FDE_CHECK_LAUNCH();
            delay('n', sl);
            ++nlaunch;
            dbg("neighbour panels");
            FDE_CUDA(cudaEventRecord(evNP, sl));
            diag_lu(sl);
        }
        if (!skip('p')) run_panel(ln);
        delay('p', sa);
        mark(k, T_PAN, sa);
        if (ln.nnp) {
            FDE_CUDA(cudaStreamWaitEvent(sa, evNP, 0));   // the products read the neighbour tiles too
        } else if (!ln.diag_scr) {   // dense x dense terms only: beside the products
            FDE_CUDA(cudaEventRecord(evPan, sa));
            FDE_CUDA(cudaStreamWaitEvent(sl, evPan, 0));
            diag_lu(sl);
        }
        if (!skip('g')) run_gemm(ln, 0, sa, !ln.nnp);   // (with neighbour panels an event wait precedes it)
        mark(k, T_G1, sa);
        if (!skip('g')) run_gemm(ln, 1, sa, ln.g_ntile[0] > 0);
        mark(k, T_G2, sa);
        if (!skip('g')) run_gemm(ln, 3, sa, ln.g_ntile[0] + ln.g_ntile[1] > 0);   // conversions to dense (after the products: a block may be
        delay('g', sa);
                               // an operand (row / column k) and a target (rows > k) at once)
        FDE_CUDA(cudaEventRecord(evP, sa));
        mark(k, T_PROD, sa);
        // snapshots of the operand factors for the dense updates (before the
        // truncations of step k+1 rewrite them: sb / se wait for evSnap)
        if (!snap_early) {
            if (ln.nsnap && !skip('s')) {
                k_h2_copy<<<ln.nsnap, 256, 0, sa>>>(P->cps.p + ln.snap0);
                FDE_CHECK_LAUNCH();
                ++nlaunch;
                dbg("snapshots");
            }
            delay('s', sa);
            FDE_CUDA(cudaEventRecord(evSnap, sa));
        } else {
            FDE_CUDA(cudaStreamWaitEvent(sa, evSnap, 0));   // (the updates below read the snapshots)
        }
        mark(k, T_SNAP, sa);
        if (ln.diag_scr) diag_lu(sa);
        FDE_CUDA(cudaStreamWaitEvent(sa, evC, 0));   // remaining updates of step k-1
        if (!skip('x')) run_gemm(ln, 2, sa);         // row / column k+1
        delay('x', sa);
        FDE_CUDA(cudaEventRecord(evCrit, sa));
        mark(k, T_CRIT, sa);
        // sb: new low-rank columns of step k (after the overflow truncations)
        FDE_CUDA(cudaStreamWaitEvent(sb, evP, 0));
        FDE_CUDA(cudaStreamWaitEvent(sb, evOv, 0));
        for (size_t r = 0; r < ln.cpr.size(); ++r) {
            if (ln.cpr[r].second && !skip('c')) {
                k_h2_copy<<<ln.cpr[r].second, 256, 0, sb>>>(P->cps.p + ln.cpr[r].first);
                FDE_CHECK_LAUNCH();
                ++nlaunch;
            }
            if (r < ln.trmid.size()) run_trunc(ln.trmid[r], sb, 0);
        }
        delay('c', sb);
        mark(k, T_CP, sb);
        // sc: the other dense updates of step k
        FDE_CUDA(cudaStreamWaitEvent(sc, evSnap, 0));
        FDE_CUDA(cudaStreamWaitEvent(sc, evP, 0));
        if (!skip_rest && !skip('r')) run_gemm(ln, 4, sc);   // (debug FDE_H2_SKIPREST: timing experiments only)
        delay('r', sc);
        FDE_CUDA(cudaEventRecord(evC, sc));
        mark(k, T_REST, sc);
        if (tline) thost.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count());
        if (tline) {
            const auto te3 = std::chrono::steady_clock::now();
            eq_us[0] += std::chrono::duration<double, std::micro>(te1 - te0).count();
            eq_us[1] += std::chrono::duration<double, std::micro>(te2 - te1).count();
            eq_us[2] += std::chrono::duration<double, std::micro>(te3 - te2).count();
        }
    }
    if (flat_worker.joinable()) flat_worker.join();
    if (flat_err) std::rethrow_exception(flat_err);
    if (tline) {
        FDE_CUDA(cudaDeviceSynchronize());
        const char* nm[T_N] = {"LU(k+1) end", "panel end", "products end", "crit end", "trunc_op end", "trunc_ov end",
                               "copies end", "rest end", "snap end", "diag end", "g1 end", "g2 end", "op gram end",
                               "op core end", "push done"};
        double prev[T_N] = {0};
        double sum[T_N] = {0};
        for (int k = 0; k < kstop; ++k)
            for (int w = 0; w < T_N; ++w) {
                float ms = 0;
                if (cudaEventElapsedTime(&ms, t0ev, tev[(size_t)k * T_N + w]) != cudaSuccess) continue;
                if (k > 0) sum[w] += ms - prev[w];
                prev[w] = ms;
            }
        fprintf(stderr, "hlu2 timeline (%d steps): per-step period of each mark (us):", kstop);
        for (int w = 0; w < T_N; ++w) fprintf(stderr, " %s %.1f |", nm[w], 1e3 * sum[w] / std::max(1, kstop - 1));
        if (kstop > 1)
            fprintf(stderr, " host enqueue %.1f (flatten %.1f [lists %.1f, expansion %.1f, split %.1f], push %.1f, launches %.1f) |",
                    (thost.back() - thost.front()) / (kstop - 1), eq_us[0] / kstop, fl_us[0] / kstop, fl_us[1] / kstop,
                    (eq_us[0] - fl_us[0] - fl_us[1]) / kstop, eq_us[1] / kstop, eq_us[2] / kstop);
        fprintf(stderr, "\n  step 10 marks (ms from start):");
        for (int w = 0; w < T_N && kstop > 10; ++w) {
            float ms = 0;
            cudaEventElapsedTime(&ms, t0ev, tev[(size_t)10 * T_N + w]);
            fprintf(stderr, " %s %.3f |", nm[w], ms);
        }
        fprintf(stderr, "\n  mean offset from the previous step's copies end (us):");
        for (int w = 0; w < T_N; ++w) {
            double acc = 0;
            int cnt = 0;
            for (int k = 4; k + 4 < kstop; ++k) {
                float a = 0, b = 0;
                if (cudaEventElapsedTime(&a, t0ev, tev[(size_t)(k - 1) * T_N + T_CP]) != cudaSuccess) continue;
                if (cudaEventElapsedTime(&b, t0ev, tev[(size_t)k * T_N + w]) != cudaSuccess) continue;
                acc += b - a;
                ++cnt;
            }
            if (cnt) fprintf(stderr, " %s %.1f |", nm[w], 1e3 * acc / cnt);
        }
        fprintf(stderr, "\n");
        for (auto& e : tev) cudaEventDestroy(e);
        cudaEventDestroy(t0ev);
        (void)cudaGetLastError();   // elapsed-time queries of unrecorded marks leave an error behind
    }
    FDE_CUDA(cudaEventRecord(evB, sb));
    FDE_CUDA(cudaStreamWaitEvent(sa, evB, 0));
    FDE_CUDA(cudaStreamWaitEvent(sa, evC, 0));
    if (kstop == nl) {
        if (!pan_inv) {
            put_copy(fin_cp, P->fin);
            put_panel(fin_pv, P->fin);
        }
        P->fin_lv.resize(fin_tt.size());
        for (size_t dd = 0; dd < fin_tt.size(); ++dd) {
            put_gemm(fin_tt[dd], P->fin_lv[dd], 0, 0);
            put_gemm(fin_tx[dd], P->fin_lv[dd], 1, 0);
        }
        push();
        FDE_CUDA(cudaStreamWaitEvent(sa, evD, 0));
        if (!pan_inv) {
            FDE_CUDA(cudaMemsetAsync(A + inv_lo, 0, (size_t)(inv_hi - inv_lo) * sizeof(double), sa));
            run_copy(P->fin, sa);
            run_panel(P->fin);
        }
        for (auto& lv : P->fin_lv) {
            run_gemm(lv, 0, sa);
            run_gemm(lv, 1, sa);
        }
    }
    FDE_CUDA(cudaEventRecord(evS, sa));
    FDE_CUDA(cudaStreamWaitEvent(s, evS, 0));
    if (getenv("FDE_H2_CHECK")) {
        FDE_CUDA(cudaDeviceSynchronize());
        H2Bad bad{};
        FDE_CUDA(cudaMemcpyFromSymbol(&bad, g_h2_bad, sizeof(H2Bad)));
        if (bad.tag)
            fprintf(stderr, "hlu2 bounds: tag %d (%d, %d) ptr %p bytes %lld arena [%p, %p)\n", bad.tag, bad.a, bad.b,
                    (void*)bad.p, bad.nbytes, (void*)A, (void*)(A + words));
        const int z = 0;
        FDE_CUDA(cudaMemcpyToSymbol(g_h2_bad_flag, &z, sizeof(int)));
        H2Bad zb{};
        FDE_CUDA(cudaMemcpyToSymbol(g_h2_bad, &zb, sizeof(H2Bad)));
    }
    if (getenv("FDE_DEBUG_PLAN")) {
        int nconv = 0;
        int64_t wconv = 0;
        for (int b = 0; b < nb; ++b)
            if (dyn[b]) {
                ++nconv;
                wconv += S.bl[b].m * S.bl[b].n;
            }
        fprintf(stderr, "hlu2 plan: %d low-rank blocks converted to dense (%.1f MB)\n", nconv, wconv * 8e-6);
    }
    if (getenv("FDE_DEBUG_PLAN"))
        fprintf(stderr, "hlu2 plan phases (ms): operands/panels %.2f pairs %.2f targets %.2f conversions %.2f "
                        "dense terms %.2f pretrunc %.2f slots/copies %.2f\n", psec[0], psec[1], psec[2], psec[3], psec[4],
                psec[5], psec[6]);
    if (getenv("FDE_DEBUG_PLAN")) {
        double gt[6] = {0}, gmx[6] = {0}, tr = 0, trk = 0, pn = 0, cp = 0;
        for (auto& ln : P->steps) {
            for (int w = 0; w < 6; ++w) { gt[w] += ln.g_ntile[w]; gmx[w] = std::max(gmx[w], (double)ln.g_ntile[w]); }
            tr += ln.tr.ne;
            trk += ln.tr.nc;
            pn += ln.npan;
            for (auto& c : ln.cpr) cp += c.second;
        }
        fprintf(stderr, "hlu2 plan: per step: gemm tiles (mean/max) cores %.1f/%g products %.1f/%g crit %.1f/%g "
                        "conv %.1f/%g rest %.1f/%g diag %.1f/%g | operand trunc entries %.1f chunks %.1f | panel CTAs %.1f "
                        "| copy CTAs %.1f\n", gt[0] / nl, gmx[0], gt[1] / nl, gmx[1], gt[2] / nl, gmx[2], gt[3] / nl, gmx[3],
                gt[4] / nl, gmx[4], gt[5] / nl, gmx[5], tr / nl, trk / nl, pn / nl, cp / nl);
        fprintf(stderr, "hlu2 plan: per step MFLOP / C MB: cores %.1f/%.1f products %.1f/%.1f crit %.1f/%.1f "
                        "rest %.1f/%.1f diag %.1f/%.1f\n", gstat_flop[0] / nl * 1e-6, gstat_cbytes[0] / nl * 1e-6,
                gstat_flop[1] / nl * 1e-6, gstat_cbytes[1] / nl * 1e-6, gstat_flop[2] / nl * 1e-6,
                gstat_cbytes[2] / nl * 1e-6, gstat_flop[4] / nl * 1e-6, gstat_cbytes[4] / nl * 1e-6,
                gstat_flop[5] / nl * 1e-6, gstat_cbytes[5] / nl * 1e-6);
    }
    if (getenv("FDE_DEBUG_PLAN"))
        fprintf(stderr, "hlu2 plan: nl %d blocks %d | simulate %.2f ms, layout+alloc %.2f ms, counts %.2f ms, "
                        "plan+launch total %.2f ms | tiles %zu terms %zu copies %zu panels %zu trunc %zu\n",
                nl, nb, ms_sim, ms_alloc, ms_flat0, ms_since(t_plan0), vtile.size(), vterm.size(), vcp.size(),
                vpan.size(), vte.size());
    L->nops = nlaunch;

    // ---- the blocks in the format of hlu.cu (substitutions, test helpers)
    L->max_rank = 0;
    for (int b = 0; b < nb; ++b) {
        const HBlock& hb = S.bl[b];
        LBlk& lb = L->B[b];
        lb.type = hb.type;
        lb.m = hb.m;
        lb.n = hb.n;
        lb.r0 = S.cl[hb.tau].r0;
        lb.c0 = S.cl[hb.sig].r0;
        for (int q = 0; q < 4; ++q) lb.child[q] = hb.child[q];
        if (dyn[b] && conv_step[b] < kstop) lb.type = HB_DENSE;
        if (lb.type == HB_DENSE) lb.D = A + offD[b];
        if (lb.type == HB_LR) {
            lb.U = A + offU[b];
            lb.V = A + offV[b];
            lb.k = kstop == nl ? kc[b] : kcap[b];   // partial sweep: unwritten columns are zero
            L->max_rank = std::max(L->max_rank, kc[b]);
        }
    }
    for (int f = 0; f < nleaf; ++f) {
        LBlk& d = L->B[own(lq0[f], lq0[f])];   // the dense diagonal block of leaf f
        d.Li = A + offLi[f];
        d.Ui = A + offUi[f];
    }
    return true;
}



// ------------------------------------------- many-RHS substitutions as GEMM tasks
// precond_apply with nrhs >= FDE_APPLY_GEMM_MIN right-hand sides (opt-in): the
// same leaf-sequential substitutions as k_apply, each leaf step as
// multi-term GEMM tasks on the FP64 tensor cores (k_h2_gemm):
//   x_k <- x_k - sum_d D_d x_{c_d} - sum_{l, chunk} U_l T_{l, chunk}   (in place, beta 1)
//   z   <- Inv_k x_k ;  x_k <- z                                          (strided copy)
//   T_{b, chunk} <- V_b[chunk]^T x_sigma[chunk]   for the blocks whose columns complete
//                                                 at leaf k (second stream)
// The projections of 256-row chunks enter the row task as separate terms (no
// reduction step).  A row task waits for the projections of two leaves back: a
// block whose columns end at leaf k-1 has no rows at leaf k (admissibility gap).
void apply_gemm_path(fde_ctx* h, ApplySched* A, double* x, int64_t ldx, int nrhs)
{
    cudaStream_t s = h->stream, sp = aux_stream6(h);
    if ((size_t)A->zmax * nrhs > A->zcap) {
        A->z.alloc((size_t)A->zmax * nrhs);
        A->zcap = (size_t)A->zmax * nrhs;
    }
    if ((size_t)A->tslots * nrhs > A->tcap) {
        A->t.alloc((size_t)A->tslots * nrhs);
        A->tcap = (size_t)A->tslots * nrhs;
    }
    const int nl = A->nleaf;
    if ((int)A->gev.size() < nl + 1) {
        for (auto e : A->gev)
            if (e) cudaEventDestroy(e);
        A->gev.assign(nl + 1, nullptr);
        for (auto& e : A->gev) FDE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    double* Tb = A->t.p;
    double* Z = A->z.p;
    // descriptors: per sweep and leaf, three launches (row task, inverse task, projections)
    std::vector<H2Task> tasks;
    std::vector<H2Term> terms;
    std::vector<H2Tile> tiles;
    struct Rng { int t0, nt; };
    std::vector<Rng> rrow, rinv, rproj;   // [sweep * nl + step]
    auto add_task = [&](double* C, long long ldc, int m, int n, double beta, int tm, int tn) {
        H2Task d;
        d.C = C;
        d.ldc = ldc;
        d.m = m;
        d.n = n;
        d.beta = beta;
        d.t_lo = (int)terms.size();
        d.t_hi = d.t_lo;
        tasks.push_back(d);
        (void)tm;
        (void)tn;
        return (int)tasks.size() - 1;
    };
    auto add_tiles = [&](int ti, int tm, int tn) {
        for (int m0 = 0; m0 < tasks[ti].m; m0 += tm)
            for (int n0 = 0; n0 < tasks[ti].n; n0 += tn) tiles.push_back({ti, m0, n0});
    };
    for (int w = 0; w < 2; ++w) {
        const std::vector<SLeaf>& LV = A->hleaf[w];
        const std::vector<SDense>& DV = A->hdense[w];
        const std::vector<SLRRow>& RV = A->hlrr[w];
        const std::vector<SProj>& PV = A->hproj[w];
        for (int st = 0; st < nl; ++st) {
            const int k = w ? nl - 1 - st : st;
            const SLeaf& L = LV[k];
            // row task (in place on the leaf's rows)
            {
                const int t0 = (int)tiles.size();
                const int ti = add_task(x + L.r0, ldx, L.m, nrhs, 1.0, 64, 64);
                for (int d = L.d_lo; d < L.d_hi; ++d) {
                    const SDense& D = DV[d];
                    terms.push_back({D.D + D.roff, x + D.c0, D.ldd, ldx, D.nc, 0, 0, -1.0});
                }
                for (int l = L.l_lo; l < L.l_hi; ++l) {
                    const SLRRow& R = RV[l];
                    for (int ch = 0; ch < R.nchunk; ++ch)
                        terms.push_back({R.U + R.roff, Tb + (long long)(R.tslot + ch * R.kc) * nrhs, R.ldu, R.kc,
                                         R.kc, 0, 0, -1.0});
                }
                tasks[ti].t_hi = (int)terms.size();
                add_tiles(ti, 32, 32);
                rrow.push_back({t0, (int)tiles.size() - t0});
            }
            // inverse task: z = Inv_k x_k
            {
                const int t0 = (int)tiles.size();
                const int ti = add_task(Z, L.m, L.m, nrhs, 0.0, 64, 64);
                terms.push_back({L.inv, x + L.r0, L.m, ldx, L.m, 0, 0, 1.0});
                tasks[ti].t_hi = (int)terms.size();
                add_tiles(ti, 32, 32);
                rinv.push_back({t0, (int)tiles.size() - t0});
            }
            // projections enabled by this leaf: T_{b, ch} = V_b[ch]^T x_sigma[ch]
            {
                const int t0 = (int)tiles.size();
                for (int p = L.p_lo; p < L.p_hi; ++p) {
                    const SProj& Pj = PV[p];
                    for (int ch = 0; ch < Pj.nchunk; ++ch) {
                        const int r0 = ch * PROJ_CHUNK, rows = std::min(PROJ_CHUNK, Pj.n - r0);
                        const int ti = add_task(Tb + (long long)(Pj.tslot + ch * Pj.kc) * nrhs, Pj.kc, Pj.kc, nrhs, 0.0,
                                                16, 16);
                        terms.push_back({Pj.V + r0, x + Pj.c0 + r0, Pj.ldv, ldx, rows, 1, 0, 1.0});
                        tasks[ti].t_hi = (int)terms.size();
                        add_tiles(ti, 16, 16);
                    }
                }
                rproj.push_back({t0, (int)tiles.size() - t0});
            }
        }
    }
    DBuf<H2Task> dtask;
    DBuf<H2Term> dterm;
    DBuf<H2Tile> dtile;
    dtask.upload(tasks.data(), tasks.size(), s);
    dterm.upload(terms.data(), terms.size(), s);
    dtile.upload(tiles.data(), tiles.size(), s);
    set_smem_once((const void*)k_h2_gemm<32, 32, true>, H2G_SMEM(32, 32));
    set_smem_once((const void*)k_h2_gemm<16, 16, true>, H2G_SMEM(16, 16));
    cudaEvent_t evx = h->ev_aux[14];   // (the H-LU's neighbour-panel event: free outside the factorisation)
    FDE_CUDA(cudaEventRecord(evx, s));
    FDE_CUDA(cudaStreamWaitEvent(sp, evx, 0));
    for (int w = 0; w < 2; ++w)
        for (int st = 0; st < nl; ++st) {
            const int q = w * nl + st;
            const int k = w ? nl - 1 - st : st;
            const SLeaf& L = A->hleaf[w][k];
            if (st >= 2) FDE_CUDA(cudaStreamWaitEvent(s, A->gev[st - 2], 0));
            if (rrow[q].nt)
                k_h2_gemm<32, 32, true><<<rrow[q].nt, 256, H2G_SMEM(32, 32), s>>>(dtile.p + rrow[q].t0, dtask.p, dterm.p,
                                                                                 rrow[q].nt);
            FDE_CHECK_LAUNCH();
            k_h2_gemm<32, 32, true><<<rinv[q].nt, 256, H2G_SMEM(32, 32), s>>>(dtile.p + rinv[q].t0, dtask.p, dterm.p,
                                                                             rinv[q].nt);
            FDE_CHECK_LAUNCH();
            FDE_CUDA(cudaMemcpy2DAsync(x + L.r0, (size_t)ldx * sizeof(double), Z, (size_t)L.m * sizeof(double),
                                       (size_t)L.m * sizeof(double), (size_t)nrhs, cudaMemcpyDeviceToDevice, s));
            FDE_CUDA(cudaEventRecord(evx, s));
            FDE_CUDA(cudaStreamWaitEvent(sp, evx, 0));
            if (rproj[q].nt) {
                k_h2_gemm<16, 16, true><<<rproj[q].nt, 256, H2G_SMEM(16, 16), sp>>>(dtile.p + rproj[q].t0, dtask.p,
                                                                                   dterm.p, rproj[q].nt);
                FDE_CHECK_LAUNCH();
            }
            FDE_CUDA(cudaEventRecord(A->gev[st], sp));
        }
    FDE_CUDA(cudaEventRecord(A->gev[nl], sp));
    FDE_CUDA(cudaStreamWaitEvent(s, A->gev[nl], 0));
}
