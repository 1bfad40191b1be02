// sem_assemble: batched dense fp64 assembly of A = rho M + theta S_l + (1-theta) S_l^T
// (Eq. (lsys)) on sm_100a.
//
// Two phases.
//  (1) Pair moments, one warp per element pair (i >= j):
//        K_ij[m][n] = gamma0 int_{-1}^{1} int_{-1}^{1} L_m(xi) L_n(eta) (t_i(xi) - s_j(eta))_+^{1-alpha}
//      (the derivatives of the local basis are Legendre series, psi_p' = -(2p+1) L_p,
//      hat' = +-1/2 L_0, so every S_l entry is a signed sum of these moments; the
//      Jacobians cancel).  With u = t - x_i, v = x_{j+1} - s and the gap
//      d = x_i - x_{j+1} >= 0 the kernel is (d + u + v)^{1-alpha}: no cancellation.
//        * i == j : K_ii = (h_i/2)^{1-alpha} Kself, Kself by nested Gauss-Jacobi (exact).
//        * d == 0 : Duffy split of the corner square [0,c0]^2 (radial Gauss-Jacobi with
//                   weight r^{2-alpha}, exact; angular Gauss-Legendre) + graded cells.
//        * d > 0  : graded composite tensor Gauss-Legendre; cells satisfy
//                   size <= c * distance to the singular point, c = 1/2; far pairs
//                   (h <= d/2) are a single cell.  Q per direction from the
//                   Bernstein-ellipse rate of the cell.
//  (2) Expansion of the moments into the dense rows of this rank (row-major,
//      element-interleaved order, padded to lda), adding rho M.
#include <cmath>

#include "fde_internal.h"
#include "hmatrix.h"

__constant__ double c_glx[FDE_GL_TOTAL];
__constant__ double c_glw[FDE_GL_TOTAL];
// Legendre recurrence coefficients L_{k+1} = a_k x L_k - b_k L_{k-1}, a_k = (2k+1)/(k+1),
// b_k = k/(k+1): multiplications instead of a division per step (the division was
// the largest single cost of the pair kernel)
#define FDE_LEG_K 64
__constant__ double c_leg_a[FDE_LEG_K];
__constant__ double c_leg_b[FDE_LEG_K];
// digits targeted by the quadrature order selection (FDE_ASM_DIGITS, default 17)
__constant__ float c_qdigits = 17.0f;

static bool g_gl_uploaded[64] = {};   // __constant__ memory is per device

static void upload_gl_tables(int dev)
{
    if (g_gl_uploaded[dev & 63]) return;
    std::vector<double> X(FDE_GL_TOTAL), W(FDE_GL_TOTAL);
    for (int q = 1; q <= FDE_QMAX; ++q) {
        std::vector<double> x, w;
        fdeq::gauss_legendre(q, x, w);
        for (int k = 0; k < q; ++k) {
            X[q * (q - 1) / 2 + k] = x[k];
            W[q * (q - 1) / 2 + k] = w[k];
        }
    }
    FDE_CUDA(cudaMemcpyToSymbol(c_glx, X.data(), sizeof(double) * FDE_GL_TOTAL));
    FDE_CUDA(cudaMemcpyToSymbol(c_glw, W.data(), sizeof(double) * FDE_GL_TOTAL));
    double la[FDE_LEG_K], lb[FDE_LEG_K];
    for (int k = 0; k < FDE_LEG_K; ++k) {
        la[k] = (2.0 * k + 1.0) / (k + 1.0);
        lb[k] = (double)k / (k + 1.0);
    }
    FDE_CUDA(cudaMemcpyToSymbol(c_leg_a, la, sizeof(la)));
    FDE_CUDA(cudaMemcpyToSymbol(c_leg_b, lb, sizeof(lb)));
    const float qd = getenv("FDE_ASM_DIGITS") ? (float)atof(getenv("FDE_ASM_DIGITS")) : 17.0f;
    FDE_CUDA(cudaMemcpyToSymbol(c_qdigits, &qd, sizeof(qd)));
    g_gl_uploaded[dev & 63] = true;
}

// --------------------------------------------------------------- device side
struct AsmDev {
    int N, P;
    double oma;      // 1 - alpha
    double g0;       // 1/Gamma(2-alpha)
    const double* nodes;
    const double* gjr_x;
    const double* gjr_w;
    int qr;
    const double* gji_x;
    const double* gji_w;
    int qi;
    const double* kself;
    int qm;          // per-direction capacity of the warp workspace
};

struct WarpWS {
    double *acc, *Lu, *Lv, *T, *kv, *ua, *wa, *vb, *wb;
};

// kernel values of a cell are produced ASM_KVC columns at a time (qm x ASM_KVC
// doubles instead of qm x qm: more warps per SM fit; same fma order, same bits)
#ifndef ASM_KVC
#define ASM_KVC 8
#endif
// rows of the per-point arrays: the Gauss-Legendre cap qm, and the P + 1 radial
// Gauss-Jacobi points of the Duffy corner (more than qm when P = FDE_MAX_P)
__host__ __device__ inline int ws_rows(int P, int qm) { return qm > P + 1 ? qm : P + 1; }
__host__ __device__ inline int ws_doubles(int P, int qm)
{
    const int q = ws_rows(P, qm);
    return P * P + 3 * q * P + q * ASM_KVC + 4 * q;
}

__device__ inline WarpWS carve_ws(double* base, int P, int qm)
{
    qm = ws_rows(P, qm);
    WarpWS w;
    w.acc = base;
    w.Lu = w.acc + P * P;
    w.Lv = w.Lu + qm * P;
    w.T = w.Lv + qm * P;
    w.kv = w.T + qm * P;
    w.ua = w.kv + qm * ASM_KVC;
    w.wa = w.ua + qm;
    w.vb = w.wa + qm;
    w.wb = w.vb + qm;
    return w;
}

// L_0..L_{P-1}(x) by the three-term recurrence
__device__ inline void leg_all(int P, double x, double* out)
{
    double p0 = 1.0, p1 = x;
    out[0] = 1.0;
    if (P > 1) out[1] = x;
    for (int k = 1; k + 1 < P; ++k) {
        double p2 = fma(c_leg_a[k] * x, p1, -c_leg_b[k] * p0);
        out[k + 1] = p2;
        p0 = p1;
        p1 = p2;
    }
}

// points per direction for a cell whose singular point lies at normalised
// distance eta (>1) from the cell centre line: Bernstein ellipse rho = eta +
// sqrt(eta^2-1); error ~ rho^{-(2Q - (P-1))} -> ~1e-17.
__device__ inline int q_select(double eta, int P, int qm)
{
    // (single precision suffices: the result is a point count; a count that differs
    // by one near a rounding boundary only moves the quadrature error around 1e-17)
    const float etaf = (float)fmin(eta, 1e30);
    // (explicit fmaf: the same rounding wherever the function is inlined -- a contraction
    // decided per call site moved counts at a rounding boundary between kernels)
    const float rho = etaf + sqrtf(fmaxf(fmaf(etaf, etaf, -1.0f), 0.0f));
    const float lr = __log10f(fmaxf(0.8f * rho, 1.05f));
    int q = (int)ceilf(__fmul_rn(__fadd_rn(__fdividef(c_qdigits, lr), (float)P), 0.5f));
    int qmin = P / 2 + 2;
    if (q < qmin) q = qmin;
    if (q > qm) q = qm;
    return q;
}

// One tensor Gauss-Legendre cell [u0,u1]x[v0,v1] of the (u,v) rectangle;
// accumulates sum w_a w_b L_m(xi_a) L_n(eta_b) (d+u_a+v_b)^{1-alpha} into acc.
template <int PT>
__device__ void warp_cell(const AsmDev& D, const WarpWS& ws, double d, double hi, double hj, double u0,
                          double u1, double v0, double v1, int lane)
{
    const int P = PT ? PT : D.P;
    const double du = u1 - u0, dv = v1 - v0;
    const double dist = d + u0 + v0;
    const int Qu = q_select(1.0 + 2.0 * dist / du, P, D.qm);
    const int Qv = q_select(1.0 + 2.0 * dist / dv, P, D.qm);
    const double* gxu = c_glx + Qu * (Qu - 1) / 2;
    const double* gwu = c_glw + Qu * (Qu - 1) / 2;
    const double* gxv = c_glx + Qv * (Qv - 1) / 2;
    const double* gwv = c_glw + Qv * (Qv - 1) / 2;
    for (int a = lane; a < Qu; a += 32) {
        double u = u0 + 0.5 * du * (gxu[a] + 1.0);
        ws.ua[a] = u;
        ws.wa[a] = 0.5 * du * gwu[a];
        leg_all(P, 2.0 * u / hi - 1.0, ws.Lu + a * P);
    }
    for (int b = lane; b < Qv; b += 32) {
        double v = v0 + 0.5 * dv * (gxv[b] + 1.0);
        ws.vb[b] = v;
        ws.wb[b] = 0.5 * dv * gwv[b];
        leg_all(P, 1.0 - 2.0 * v / hj, ws.Lv + b * P);
    }
    __syncwarp();
    const double uc = 0.5 * (u0 + u1), vc = 0.5 * (v0 + v1);
    const double zc = d + uc + vc;
    const double kc = pow(zc, D.oma), izc = 1.0 / zc;
    for (int b0 = 0; b0 < Qv; b0 += ASM_KVC) {
        const int nb = min(ASM_KVC, Qv - b0);
        for (int idx = lane; idx < Qu * nb; idx += 32) {
            const int a = idx / nb, bb = idx - a * nb, b = b0 + bb;
            double delta = ((ws.ua[a] - uc) + (ws.vb[b] - vc)) * izc;
            ws.kv[a * ASM_KVC + bb] = ws.wa[a] * ws.wb[b] * kc * exp(D.oma * log1p(delta));
        }
        __syncwarp();
        for (int idx = lane; idx < Qu * P; idx += 32) {
            int a = idx / P, nn = idx - a * P;
            const double* kr = ws.kv + a * ASM_KVC;
            double s = (b0 == 0) ? 0.0 : ws.T[idx];   // (the same fma sequence as one pass over b)
            for (int bb = 0; bb < nb; ++bb) s = fma(kr[bb], ws.Lv[(b0 + bb) * P + nn], s);
            ws.T[idx] = s;
        }
        __syncwarp();
    }
    for (int idx = lane; idx < P * P; idx += 32) {
        int m = idx / P, nn = idx - m * P;
        double s = 0.0;
        for (int a = 0; a < Qu; ++a) s = fma(ws.Lu[a * P + m], ws.T[a * P + nn], s);
        ws.acc[idx] += s;
    }
    __syncwarp();
}

// graded composite rule on the rectangle [u0,u1]x[v0,v1] (needs d+u0+v0 > 0)
template <int PT>
__device__ void warp_graded(const AsmDev& D, const WarpWS& ws, double d, double hi, double hj, double u0,
                            double u1, double v0, double v1, int lane)
{
    const double c = 0.5;
    double ua = u0;
    int guard = 0;
    while (ua < u1 && guard++ < 400) {
        double ub = fmin(u1, ua + c * (d + ua + v0));
        if (u1 - ub < 1e-3 * (ub - ua)) ub = u1;
        double va = v0;
        int g2 = 0;
        while (va < v1 && g2++ < 400) {
            double vb = fmin(v1, va + c * (d + u0 + va));
            if (v1 - vb < 1e-3 * (vb - va)) vb = v1;
            warp_cell<PT>(D, ws, d, hi, hj, ua, ub, va, vb, lane);
            va = vb;
        }
        ua = ub;
    }
}

// Duffy treatment of the corner square [0,c0]^2 of a touching pair (d = 0):
//  v <= u: v = u w:  int_0^c0 u^{2-a} L_m(xi(u)) int_0^1 (1+w)^{1-a} L_n(eta(u w)) dw du
//  u <= v: u = v w:  int_0^c0 v^{2-a} L_n(eta(v)) int_0^1 (1+w)^{1-a} L_m(xi(v w)) dw dv
template <int PT>
__device__ void warp_duffy(const AsmDev& D, const WarpWS& ws, double hi, double hj, double c0, int lane)
{
    const int P = PT ? PT : D.P;
    const int Qr = D.qr;
    const int Qw = q_select(3.0, P, D.qm);
    const double* gxw = c_glx + Qw * (Qw - 1) / 2;
    const double* gww = c_glw + Qw * (Qw - 1) / 2;
    const double rs = pow(0.5 * c0, 3.0 + D.oma - 1.0);   // (c0/2)^{3-alpha}
    double Lt[FDE_MAX_P];
    for (int tri = 0; tri < 2; ++tri) {
        // radial node k: r_k, weight; fixed-side Legendre values in Lu (tri 0) or Lv (tri 1)
        for (int k = lane; k < Qr; k += 32) {
            double r = 0.5 * c0 * (D.gjr_x[k] + 1.0);
            double wr = D.gjr_w[k] * rs;
            if (tri == 0)
                leg_all(P, 2.0 * r / hi - 1.0, ws.Lu + k * P);
            else
                leg_all(P, 1.0 - 2.0 * r / hj, ws.Lv + k * P);
            double* Trow = ws.T + k * P;
            for (int q = 0; q < P; ++q) Trow[q] = 0.0;
            for (int l = 0; l < Qw; ++l) {
                double w = 0.5 * (gxw[l] + 1.0);
                double W = wr * 0.5 * gww[l] * exp(D.oma * log1p(w));
                if (tri == 0)
                    leg_all(P, 1.0 - 2.0 * r * w / hj, Lt);
                else
                    leg_all(P, 2.0 * r * w / hi - 1.0, Lt);
                for (int q = 0; q < P; ++q) Trow[q] = fma(W, Lt[q], Trow[q]);
            }
        }
        __syncwarp();
        for (int idx = lane; idx < P * P; idx += 32) {
            int m = idx / P, nn = idx - m * P;
            double s = 0.0;
            if (tri == 0)
                for (int k = 0; k < Qr; ++k) s = fma(ws.Lu[k * P + m], ws.T[k * P + nn], s);
            else
                for (int k = 0; k < Qr; ++k) s = fma(ws.T[k * P + m], ws.Lv[k * P + nn], s);
            ws.acc[idx] += s;
        }
        __syncwarp();
    }
}

// compute the moment block of pair (i, j), i >= j, into out[P*P]
template <int PT>
__device__ void warp_pair(const AsmDev& D, const WarpWS& ws, int i, int j, double* out, int lane)
{
    const int P = PT ? PT : D.P;
    const double hi = D.nodes[i + 1] - D.nodes[i];
    if (i == j) {
        const double s = pow(0.5 * hi, D.oma);
        for (int idx = lane; idx < P * P; idx += 32) out[idx] = s * D.kself[idx];
        return;
    }
    const double hj = D.nodes[j + 1] - D.nodes[j];
    const double d = D.nodes[i] - D.nodes[j + 1];
    for (int idx = lane; idx < P * P; idx += 32) ws.acc[idx] = 0.0;
    __syncwarp();
    if (d > 0.0) {
        warp_graded<PT>(D, ws, d, hi, hj, 0.0, hi, 0.0, hj, lane);
    } else {
        const double c0 = fmin(hi, hj);
        warp_duffy<PT>(D, ws, hi, hj, c0, lane);
        if (hi > hj * (1.0 + 1e-12))
            warp_graded<PT>(D, ws, 0.0, hi, hj, c0, hi, 0.0, hj, lane);
        else if (hj > hi * (1.0 + 1e-12))
            warp_graded<PT>(D, ws, 0.0, hi, hj, 0.0, hi, c0, hj, lane);
    }
    const double sc = D.g0 * (2.0 / hi) * (2.0 / hj);
    for (int idx = lane; idx < P * P; idx += 32) out[idx] = sc * ws.acc[idx];
    __syncwarp();
}

#ifndef ASM_WARPS
#define ASM_WARPS 4
#endif

// mode 0: triangle rows [i0,i1): pair p -> (i, j<=i), slot p - T(i0)
// mode 1: rectangle i in [i0,i1) x j in [j0,j1)
// mode 2: explicit list
template <int PT>
__global__ void __launch_bounds__(32 * ASM_WARPS) k_pairs_kernel(AsmDev D, int mode, int i0, int i1, int j0,
                                                                int j1, const int* li, const int* lj,
                                                                const long long* lslot, long long count,
                                                                double* out)
{
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long p = (long long)blockIdx.x * ASM_WARPS + wid;
    if (p >= count) return;
    WarpWS ws = carve_ws(smem + (size_t)wid * ws_doubles(D.P, D.qm), D.P, D.qm);
    int i, j;
    long long slot;
    if (mode == 0) {
        long long T0 = (long long)i0 * (i0 + 1) / 2;
        long long g = T0 + p;
        long long ii = (long long)((sqrt(8.0 * (double)g + 1.0) - 1.0) * 0.5);
        while ((ii + 1) * (ii + 2) / 2 <= g) ++ii;
        while (ii * (ii + 1) / 2 > g) --ii;
        i = (int)ii;
        j = (int)(g - ii * (ii + 1) / 2);
        slot = p;
    } else if (mode == 1) {
        const int w = j1 - j0;
        i = i0 + (int)(p / w);
        j = j0 + (int)(p % w);
        slot = p;
    } else {
        i = li[p];
        j = lj[p];
        slot = lslot[p];
    }
    warp_pair<PT>(D, ws, i, j, out + slot * (long long)D.P * D.P, lane);
}

// Lane-per-pair path for P <= 8: almost every pair of a mesh is "far" -- gap d > 0
// and d >= 2 max(h_i, h_j), so warp_graded makes ONE cell of the whole rectangle --
// and a warp spent on one such pair leaves most lanes idle (6 x 6 kernel values,
// 6 + 6 Legendre rows, 64 moments over 32 lanes, warp barriers between the stages).
// Here lane L of warp w owns pair 32 w + L and runs the same one-cell rule alone:
// identical points, weights, kernel values and fma sequences (T[n] over b, then the
// moments over a), so the moments are bit-identical to warp_cell's; the pairs that
// are not single-cell far pairs (self, touching, near) are then done one by one by
// the whole warp with warp_pair, as before.
#ifndef ASM_LANE_UB
#define ASM_LANE_UB 2     // (b loop by two: also the unrolling that reproduces warp_cell's bits)
#endif
#ifndef ASM_LANE_WARPS
#define ASM_LANE_WARPS 2  // warps per CTA of the lane path
#endif
#ifndef ASM_LANE_UA
#define ASM_LANE_UA 1
#endif
constexpr int kLaneUB = ASM_LANE_UB, kLaneUA = ASM_LANE_UA;   // (loop unrolling of the lane path)
template <int PT>
__global__ void __launch_bounds__(32 * ASM_LANE_WARPS) k_pairs_lane(AsmDev D, int mode, int i0, int i1, int j0, int j1,
                                                              const int* li, const int* lj, const long long* lslot,
                                                              long long count, double* out)
{
    static_assert(PT >= 1 && PT <= 8, "lane path: P <= 8 (moments in registers)");
    constexpr int P = PT;
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long p = ((long long)blockIdx.x * ASM_LANE_WARPS + wid) * 32 + lane;
    const bool valid = p < count;
    int i = 0, j = 0;
    long long slot = 0;
    if (valid) {
        if (mode == 0) {
            const long long T0 = (long long)i0 * (i0 + 1) / 2;
            const long long g = T0 + p;
            long long ii = (long long)((sqrt(8.0 * (double)g + 1.0) - 1.0) * 0.5);
            while ((ii + 1) * (ii + 2) / 2 <= g) ++ii;
            while (ii * (ii + 1) / 2 > g) --ii;
            i = (int)ii;
            j = (int)(g - ii * (ii + 1) / 2);
            slot = p;
        } else if (mode == 1) {
            const int w = j1 - j0;
            i = i0 + (int)(p / w);
            j = j0 + (int)(p % w);
            slot = p;
        } else {
            i = li[p];
            j = lj[p];
            slot = lslot[p];
        }
    }
    bool far = false;
    double hi = 0.0, hj = 0.0, d = 0.0;
    if (valid && i != j) {
        hi = D.nodes[i + 1] - D.nodes[i];
        hj = D.nodes[j + 1] - D.nodes[j];
        d = D.nodes[i] - D.nodes[j + 1];
        if (d > 0.0) {   // warp_graded's first cell on (u0, v0) = (0, 0), c = 1/2
            double ub = fmin(hi, 0.5 * d);
            if (hi - ub < 1e-3 * ub) ub = hi;
            double vb = fmin(hj, 0.5 * d);
            if (hj - vb < 1e-3 * vb) vb = hj;
            far = (ub == hi) && (vb == hj);
        }
    }
    if (far) {   // warp_cell(d, hi, hj, 0, hi, 0, hj), one lane
        const int Qu = q_select(1.0 + 2.0 * d / hi, P, D.qm);
        const int Qv = q_select(1.0 + 2.0 * d / hj, P, D.qm);
        const double* gxu = c_glx + Qu * (Qu - 1) / 2;
        const double* gwu = c_glw + Qu * (Qu - 1) / 2;
        const double* gxv = c_glx + Qv * (Qv - 1) / 2;
        const double* gwv = c_glw + Qv * (Qv - 1) / 2;
        const double uc = 0.5 * hi, vc = 0.5 * hj;
        const double zc = d + uc + vc;
        const double kc = pow(zc, D.oma), izc = 1.0 / zc;
        double acc[P * P];
#pragma unroll
        for (int t = 0; t < P * P; ++t) acc[t] = 0.0;
#pragma unroll kLaneUA
        for (int a = 0; a < Qu; ++a) {
            const double u = 0.5 * hi * (gxu[a] + 1.0);
            const double wa = 0.5 * hi * gwu[a];
            double Lu[P];
            leg_all(P, 2.0 * u / hi - 1.0, Lu);
            double T[P];
#pragma unroll
            for (int n = 0; n < P; ++n) T[n] = 0.0;
#pragma unroll kLaneUB
            for (int b = 0; b < Qv; ++b) {
                const double v = 0.5 * hj * (gxv[b] + 1.0);
                const double wb = 0.5 * hj * gwv[b];
                double Lv[P];
                leg_all(P, 1.0 - 2.0 * v / hj, Lv);
                const double delta = ((u - uc) + (v - vc)) * izc;
                const double kv = wa * wb * kc * exp(D.oma * log1p(delta));
#pragma unroll
                for (int n = 0; n < P; ++n) T[n] = fma(kv, Lv[n], T[n]);
            }
#pragma unroll
            for (int m = 0; m < P; ++m)
#pragma unroll
                for (int n = 0; n < P; ++n) acc[m * P + n] = fma(Lu[m], T[n], acc[m * P + n]);
        }
        const double sc = D.g0 * (2.0 / hi) * (2.0 / hj);
        double* o = out + slot * (long long)(P * P);
#pragma unroll
        for (int t = 0; t < P * P; ++t) o[t] = sc * (0.0 + acc[t]);
    }
    // the other pairs of this warp: one at a time with the whole warp
    unsigned slow = __ballot_sync(0xffffffffu, valid && !far);
    if (!slow) return;
    WarpWS ws = carve_ws(smem + (size_t)wid * ws_doubles(P, D.qm), P, D.qm);
    while (slow) {
        const int L = __ffs(slow) - 1;
        slow &= slow - 1;
        const int ii = __shfl_sync(0xffffffffu, i, L), jj = __shfl_sync(0xffffffffu, j, L);
        const long long sl = __shfl_sync(0xffffffffu, slot, L);
        warp_pair<PT>(D, ws, ii, jj, out + sl * (long long)(P * P), lane);
    }
}

// Kself[m][n] = gamma0 2^{alpha-2} sum_k sum_l wo_k wi_l L_m(xi_k) L_n(xi_k - (1+xi_k)(1+y_l)/2)
// (nested Gauss-Jacobi, exact for polynomials); also the reference mass matrix
// Mref[a][b] = int_{-1}^{1} phi^_a phi^_b (hats and psi_p).
__global__ void k_selfref_kernel(AsmDev D, double* kself, double* mref)
{
    const int P = D.P;
    const int t = threadIdx.x;
    // the Gauss-Jacobi rules in shared memory (read 81 times per entry: from global
    // memory every inner step was a dependent L2 round trip)
    __shared__ double sgx[FDE_MAX_P + 2], sgw[FDE_MAX_P + 2], six[FDE_MAX_P + 2], siw[FDE_MAX_P + 2];
    for (int k = t; k < D.qr; k += blockDim.x) { sgx[k] = D.gjr_x[k]; sgw[k] = D.gjr_w[k]; }
    for (int k = t; k < D.qi; k += blockDim.x) { six[k] = D.gji_x[k]; siw[k] = D.gji_w[k]; }
    __syncthreads();
    double Lm[FDE_MAX_P + 2], Ln[FDE_MAX_P + 2];
    const double a2 = exp2(-1.0 - D.oma);   // 2^{alpha-2}
    const int M = P + 1;
    const int Q = (P + 2 < FDE_QMAX) ? P + 2 : FDE_QMAX;   // exact for degree 2P
    const double* gx = c_glx + Q * (Q - 1) / 2;
    const double* gw = c_glw + Q * (Q - 1) / 2;
    // small degrees: the Legendre values of every point pair in shared memory, each
    // computed once by its own thread, then the same fma sequences per entry from there
    // (one thread per entry re-evaluated them serially in local memory: ~30 us)
    constexpr int SR_CAP = 17 * 17 * 16;   // (P <= 16: qr, qi <= 17)
    __shared__ double sLn[SR_CAP], sLm[17 * 16], sIn[17 * 16], sLq[18 * 18];
    if (P <= 16 && D.qr <= 17 && D.qi <= 17 && D.qr * D.qi * P <= SR_CAP && Q <= 18) {
        for (int kl = t; kl < D.qr * D.qi; kl += blockDim.x) {
            const int k = kl / D.qi, l = kl - k * D.qi;
            const double xi = sgx[k];
            const double eta = xi - 0.5 * (1.0 + xi) * (1.0 + six[l]);
            leg_all(P, eta, Ln);
            for (int nn = 0; nn < P; ++nn) sLn[kl * P + nn] = Ln[nn];
        }
        for (int k = t; k < D.qr; k += blockDim.x) {
            leg_all(P, sgx[k], Lm);
            for (int m = 0; m < P; ++m) sLm[k * P + m] = Lm[m];
        }
        for (int k = t; k < Q; k += blockDim.x) {
            leg_all(P + 2 > 2 ? P + 2 : 2, gx[k], Lm);
            for (int a = 0; a < P + 2; ++a) sLq[k * (P + 2) + a] = Lm[a];
        }
        __syncthreads();
        for (int kn = t; kn < D.qr * P; kn += blockDim.x) {   // inner[k][nn]
            const int k = kn / P, nn = kn - k * P;
            double inner = 0.0;
            for (int l = 0; l < D.qi; ++l) inner = fma(siw[l], sLn[(k * D.qi + l) * P + nn], inner);
            sIn[kn] = inner;
        }
        __syncthreads();
        for (int idx = t; idx < P * P; idx += blockDim.x) {
            const int m = idx / P, nn = idx - m * P;
            double s = 0.0;
            for (int k = 0; k < D.qr; ++k) s = fma(sgw[k] * sLm[k * P + m], sIn[k * P + nn], s);
            kself[idx] = D.g0 * a2 * s;
        }
        for (int idx = t; idx < M * M; idx += blockDim.x) {
            const int a = idx / M, b = idx - a * M;
            double s = 0.0;
            for (int k = 0; k < Q; ++k) {
                const double xi = gx[k];
                const double* Lq = sLq + k * (P + 2);
                double fa = (a == 0) ? 0.5 * (1 - xi) : (a == P ? 0.5 * (1 + xi) : Lq[a - 1] - Lq[a + 1]);
                double fb = (b == 0) ? 0.5 * (1 - xi) : (b == P ? 0.5 * (1 + xi) : Lq[b - 1] - Lq[b + 1]);
                s = fma(gw[k], fa * fb, s);
            }
            mref[idx] = s;
        }
        return;
    }
    for (int idx = t; idx < P * P; idx += blockDim.x) {
        int m = idx / P, nn = idx - m * P;
        double s = 0.0;
        for (int k = 0; k < D.qr; ++k) {
            double xi = sgx[k];
            leg_all(P, xi, Lm);
            double inner = 0.0;
            for (int l = 0; l < D.qi; ++l) {
                double eta = xi - 0.5 * (1.0 + xi) * (1.0 + six[l]);
                leg_all(P, eta, Ln);
                inner = fma(siw[l], Ln[nn], inner);
            }
            s = fma(sgw[k] * Lm[m], inner, s);
        }
        kself[idx] = D.g0 * a2 * s;
    }
    for (int idx = t; idx < M * M; idx += blockDim.x) {
        int a = idx / M, b = idx - a * M;
        double s = 0.0;
        for (int k = 0; k < Q; ++k) {
            double xi = gx[k];
            leg_all(P + 2 > 2 ? P + 2 : 2, xi, Lm);
            double fa = (a == 0) ? 0.5 * (1 - xi) : (a == P ? 0.5 * (1 + xi) : Lm[a - 1] - Lm[a + 1]);
            double fb = (b == 0) ? 0.5 * (1 - xi) : (b == P ? 0.5 * (1 + xi) : Lm[b - 1] - Lm[b + 1]);
            s = fma(gw[k], fa * fb, s);
        }
        mref[idx] = s;
    }
}

// ----------------------------------------------------------------- dof terms
// internal (element-interleaved) dof r: element e = r / P, q = r % P;
//   q < P-1 : modal psi_{q+1} of element e
//   q = P-1 : hat of node e+1 (elements e and e+1)
// r == n : boundary hat of node 0 ; r == n+1 : boundary hat of node N.
struct DofTerms {
    int cnt;
    int e[2];
    int m[2];      // Legendre index of the derivative term
    double c[2];   // coefficient of L_m in d/dxi (phi restricted to e)
    int ml[2];     // local function index for the mass matrix (0 left hat, P right hat)
};

template <int PT = 0>
__device__ inline DofTerms dof_terms(long long r, long long n, int N, int Prt)
{
    const int P = PT ? PT : Prt;   // (compile-time P: the division below becomes a multiply)
    DofTerms t;
    if (r == n) {
        t.cnt = 1; t.e[0] = 0; t.m[0] = 0; t.c[0] = -0.5; t.ml[0] = 0;
        return t;
    }
    if (r == n + 1) {
        t.cnt = 1; t.e[0] = N - 1; t.m[0] = 0; t.c[0] = 0.5; t.ml[0] = P;
        return t;
    }
    const int ri = (int)r;   // r < 2^31 (n = N P - 1)
    int e = ri / P, q = ri - e * P;
    if (q < P - 1) {
        int p = q + 1;
        t.cnt = 1; t.e[0] = e; t.m[0] = p; t.c[0] = -(2.0 * p + 1.0); t.ml[0] = p;
    } else {
        t.cnt = 2;
        t.e[0] = e; t.m[0] = 0; t.c[0] = 0.5; t.ml[0] = P;
        t.e[1] = e + 1; t.m[1] = 0; t.c[1] = -0.5; t.ml[1] = 0;
    }
    return t;
}

// K lookups -------------------------------------------------------------
// Band storage: rows i in [b0,b1] with j <= i (packed), plus K_{i,j} for
// i > b1, j in [b0,b1] (dense).
struct KBand {
    const double* row;
    const double* col;
    int b0, b1, N, P2;
    __device__ const double* get(int i, int j) const
    {
        if (i >= b0 && i <= b1)   // (i < 2^16: the triangle index fits 32 bits)
            return row + (long long)((unsigned)i * (unsigned)(i + 1) / 2u - (unsigned)b0 * (unsigned)(b0 + 1) / 2u + (unsigned)j) * P2;
        return col + ((long long)(i - b1 - 1) * (b1 - b0 + 1) + (j - b0)) * P2;
    }
};

// Boundary table: slot i = K_{i,0}, slot N+i = K_{N-1,i}
struct KBnd {
    const double* t;
    int N, P2;
    __device__ const double* get(int i, int j) const
    {
        if (j == 0) return t + (long long)i * P2;
        return t + (long long)(N + j) * P2;   // i == N-1
    }
};

// Per-leaf rectangle table: K for element pairs (i,j) with i in [i0, i0+ni),
// j in [j0, j0+nj), stored for i>=j as K_{i,j} and for i<j as K_{j,i}
// (the lookup is symmetric in its slot choice).
struct KRect {
    const double* t;
    int i0, ni, j0, nj, P2;
    __device__ const double* get(int i, int j) const   // i >= j, one of them in each range
    {
        // (i,j) stored at [i - i0][j - j0] if i in row range and j in col range, else at [j-i0][i-j0]
        if (i >= i0 && i < i0 + ni && j >= j0 && j < j0 + nj)
            return t + ((long long)(i - i0) * nj + (j - j0)) * P2;
        return t + ((long long)(j - i0) * nj + (i - j0)) * P2;
    }
};

template <class KL, int PT = 0>
__device__ inline double a_entry(const KL& K, long long r, long long c, long long n, int N, int Prt, double theta,
                                 double rho, const double* nodes, const double* mref)
{
    const int P = PT ? PT : Prt;
    DofTerms tr = dof_terms<PT>(r, n, N, P), tc = dof_terms<PT>(c, n, N, P);
    const int P2 = P * P;
    (void)P2;
    double sl = 0.0, slt = 0.0, mass = 0.0;
    for (int x = 0; x < tr.cnt; ++x) {
        int ei = tr.e[x];
        if (ei < 0 || ei >= N) continue;
        for (int y = 0; y < tc.cnt; ++y) {
            int ej = tc.e[y];
            if (ej < 0 || ej >= N) continue;
            double cc = tr.c[x] * tc.c[y];
            if (ej <= ei) sl = fma(cc, K.get(ei, ej)[tr.m[x] * P + tc.m[y]], sl);
            if (ei <= ej) slt = fma(cc, K.get(ej, ei)[tc.m[y] * P + tr.m[x]], slt);
            if (ei == ej) mass = fma(0.5 * (nodes[ei + 1] - nodes[ei]), mref[tr.ml[x] * (P + 1) + tc.ml[y]], mass);
        }
    }
    return rho * mass + theta * sl + (1.0 - theta) * slt;
}

// Expansion per element pair: thread (ei, ej) writes the P x P entries A[rows of
// element ei][columns of element ej] (8 contiguous doubles per row: a warp writes
// 32 consecutive segments, coalesced).  The index arithmetic of dof_terms /
// K.get is done once per pair (base pointers of the <= 4 neighbouring pair blocks
// in both orientations) instead of once per entry.  Same terms in the same order
// as a_entry: bit-identical entries.
template <int PT>
__global__ void __launch_bounds__(128) k_expand_pairs(KBand K, long long r0, long long r1, long long n, long long lda,
                                                      int N, int Prt, double theta, double rho, const double* nodes,
                                                      const double* mref, double* A)
{
    const int P = PT ? PT : Prt;
    const int ej = blockIdx.x * blockDim.x + threadIdx.x;
    const int ei = (int)(r0 / P) + blockIdx.y;
    const long long c0 = (long long)ej * P;
    if (c0 >= lda) return;
    // pair blocks: lower K(a, b) (b <= a) and upper K(b, a) (a <= b), a in {ei, ei+1}, b in {ej, ej+1}
    const double* kl[2][2];
    const double* ku[2][2];
#pragma unroll
    for (int da = 0; da < 2; ++da)
#pragma unroll
        for (int db = 0; db < 2; ++db) {
            const int a = ei + da, b = ej + db;
            const bool ok = a < N && b < N;
            kl[da][db] = (ok && b <= a) ? K.get(a, b) : nullptr;
            ku[da][db] = (ok && a <= b) ? K.get(b, a) : nullptr;
        }
    const double hi = ei < N ? 0.5 * (nodes[ei + 1] - nodes[ei]) : 0.0;
    const double hi1 = ei + 1 < N ? 0.5 * (nodes[ei + 2] - nodes[ei + 1]) : 0.0;
    for (int qr = 0; qr < P; ++qr) {
        const long long r = (long long)ei * P + qr;
        if (r < r0 || r >= r1) continue;
        const DofTerms tr = dof_terms<PT>(r, n, N, P);
        double* Ar = A + (r - r0) * lda + c0;
        for (int qc = 0; qc < P; ++qc) {
            const long long c = c0 + qc;
            if (c >= lda) break;
            double v = 0.0;
            if (c < n && ej < N) {
                const DofTerms tc = dof_terms<PT>(c, n, N, P);
                double sl = 0.0, slt = 0.0, mass = 0.0;
                for (int x = 0; x < tr.cnt; ++x) {
                    const int eiX = tr.e[x];
                    if (eiX < 0 || eiX >= N) continue;
                    for (int y = 0; y < tc.cnt; ++y) {
                        const int ejY = tc.e[y];
                        if (ejY < 0 || ejY >= N) continue;
                        const double cc = tr.c[x] * tc.c[y];
                        const int da = eiX - ei, db = ejY - ej;
                        if (ejY <= eiX) sl = fma(cc, kl[da][db][tr.m[x] * P + tc.m[y]], sl);
                        if (eiX <= ejY) slt = fma(cc, ku[da][db][tc.m[y] * P + tr.m[x]], slt);
                        if (eiX == ejY) mass = fma(da ? hi1 : hi, mref[tr.ml[x] * (P + 1) + tc.ml[y]], mass);
                    }
                }
                v = rho * mass + theta * sl + (1.0 - theta) * slt;
            }
            Ar[qc] = v;
        }
    }
}

// Expansion by tiles of 8 x 8 element pairs (world 1: the whole triangle K table).
// A tile (I, J), J <= I, needs the pair blocks K(max(a,b), min(a,b)) for a in
// I + {next element}, b in J + {next element} (the hats of an element's right
// node reach into the next element): 9 x 9 blocks staged ONCE in shared memory
// with 16-byte copies, from which the CTA writes both A[rows of I][cols of J]
// (S_l part theta, S_l^T part 1-theta, mass) and the mirrored A[rows of J][cols
// of I] -- each pair block is read about 1.27 times instead of once per use (the
// per-pair kernel re-read the table 2.2 times), and every row segment is written
// by consecutive threads.  Same terms in the same order as a_entry (bit-identical).
#define EX_TE 8
template <int PT>
__global__ void __launch_bounds__(256) k_expand_tiles(const double* Ktri, long long n, long long lda, int N, double theta,
                                                      double rho, const double* nodes, const double* mref_g, double* A)
{
    // slot rows padded to P + 1 doubles: the S_l^T reads kb[n (P+1) + m] of 16 consecutive
    // columns (two elements) then hit 16 distinct bank pairs (stride P: 8-way conflicts,
    // half of all shared-memory wavefronts of the kernel were replays)
    constexpr int P = PT, P2 = PT * PT, NB = EX_TE + 1, SP = PT + 1, PS = PT * SP;
    extern __shared__ __align__(16) double ksm[];   // [a][b] slots of P2 doubles
    __shared__ double mref[(PT + 1) * (PT + 1)];
    __shared__ double hh[2 * EX_TE + 2];
    // tile index -> (ti, tj), tj <= ti (lower triangle, row by row)
    const long long bidx = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)bidx + 1.0) - 1.0) * 0.5);
    while ((long long)ti * (ti + 1) / 2 > bidx) --ti;
    while ((long long)(ti + 1) * (ti + 2) / 2 <= bidx) ++ti;
    const int tj = (int)(bidx - (long long)ti * (ti + 1) / 2);
    const int I0 = ti * EX_TE, J0 = tj * EX_TE;
    for (int e = threadIdx.x; e < (P + 1) * (P + 1); e += 256) mref[e] = mref_g[e];
    for (int e = threadIdx.x; e < 2 * NB; e += 256) {
        const int el = e < NB ? I0 + e : J0 + e - NB;
        hh[e] = el < N ? 0.5 * (nodes[el + 1] - nodes[el]) : 0.0;
    }
    // stage the slots (16-byte copies; P2 even)
    for (int e = threadIdx.x; e < NB * NB * (P2 / 2); e += 256) {
        const int slot = e / (P2 / 2), w = e - slot * (P2 / 2);
        const int a = I0 + slot / NB, b = J0 + slot % NB;
        const int hi = a > b ? a : b, lo = a > b ? b : a;
        double2 v = make_double2(0.0, 0.0);
        if (hi < N) v = reinterpret_cast<const double2*>(Ktri + ((long long)hi * (hi + 1) / 2 + lo) * P2)[w];
        const int m = (2 * w) / P, nn = 2 * w - m * P;   // (P even: a pair never straddles a row)
        double* d = ksm + (long long)slot * PS + m * SP + nn;
        d[0] = v.x;
        d[1] = v.y;
    }
    __syncthreads();
    // the two blocks: (rows I, cols J) and, off the diagonal, (rows J, cols I)
    for (int blk = 0; blk < (ti == tj ? 1 : 2); ++blk) {
        const int R0 = blk ? J0 : I0, C0 = blk ? I0 : J0;
        constexpr int nr = EX_TE * P, nc = EX_TE * P, nph = 256 / nc;   // (nc divides 256 for P = 4, 8, 16)
        const int cc2 = threadIdx.x % nc;
        const long long c = (long long)C0 * P + cc2;   // this thread's column: its terms once
        const DofTerms tc = dof_terms<PT>(c < n ? c : 0, n, N, P);
        for (int rr = threadIdx.x / nc; rr < nr; rr += nph) {
            const long long r = (long long)R0 * P + rr;
            if (r >= n || c >= n) continue;
            const DofTerms tr = dof_terms<PT>(r, n, N, P);
            double sl = 0.0, slt = 0.0, mass = 0.0;
            for (int x = 0; x < tr.cnt; ++x) {
                const int ei = tr.e[x];
                if (ei < 0 || ei >= N) continue;
                for (int y = 0; y < tc.cnt; ++y) {
                    const int ej = tc.e[y];
                    if (ej < 0 || ej >= N) continue;
                    const double cf = tr.c[x] * tc.c[y];
                    // slot of the pair (ei, ej): row index from I, column from J (or mirrored)
                    const int sa = blk ? ej - I0 : ei - I0, sb = blk ? ei - J0 : ej - J0;
                    const double* kb = ksm + (sa * NB + sb) * PS;   // K(max(ei,ej), min(ei,ej))
                    if (ej <= ei) sl = fma(cf, kb[tr.m[x] * SP + tc.m[y]], sl);
                    if (ei <= ej) slt = fma(cf, kb[tc.m[y] * SP + tr.m[x]], slt);
                    if (ei == ej)
                        mass = fma(hh[blk ? NB + (ei - J0) : (ei - I0)], mref[tr.ml[x] * (P + 1) + tc.ml[y]], mass);
                }
            }
            A[r * lda + c] = rho * mass + theta * sl + (1.0 - theta) * slt;
        }
    }
}

template <int PT>
__global__ void __launch_bounds__(256) k_expand_dense(KBand K, long long r0, long long r1, long long n, long long lda,
                                                      int N, int P, double theta, double rho, const double* nodes,
                                                      const double* mref, double* A)
{
    const long long r = r0 + blockIdx.y;
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1 || c >= lda) return;
    double v = 0.0;
    if (c < n) v = a_entry<KBand, PT>(K, r, c, n, N, P, theta, rho, nodes, mref);
    A[(r - r0) * lda + c] = v;
}

template <class KL>
__global__ void k_boundary_cols(KL K, long long n, int N, int P, double theta, double rho,
                                const double* nodes, const double* mref, double* bnd)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    bnd[r] = a_entry(K, r, n, n, N, P, theta, rho, nodes, mref);
    bnd[n + r] = a_entry(K, r, n + 1, n, N, P, theta, rho, nodes, mref);
}

// dense block of A for rows [ra, ra+m) x cols [ca, ca+nc) (internal order),
// column-major with ldb; lookups through a per-leaf rectangle table
__global__ void k_expand_block(KRect K, long long ra, int m, long long ca, int nc, long long n, int N, int P,
                               double theta, double rho, const double* nodes, const double* mref, double* B,
                               long long ldb)
{
    const int rr = blockIdx.x * blockDim.x + threadIdx.x;
    const int cc = blockIdx.y;
    if (rr >= m || cc >= nc) return;
    B[(long long)cc * ldb + rr] = a_entry(K, ra + rr, ca + cc, n, N, P, theta, rho, nodes, mref);
}

// ------------------------------------------------------------------- RHS
struct ForcingDev {
    int nleg;
    const double* leg;
    int nterm;
    const int* side;
    const double* pw;
    const double* coef;
    const double* gj_x;   // per term Gauss-Jacobi rule with its endpoint weight
    const double* gj_w;
    int qj;
};

__device__ inline double forcing_smooth(const ForcingDev& F, double offa, double offb, double ab, int skip_term_e,
                                        int e, int N)
{
    double fx = 0.0;
    if (F.nleg > 0) {
        double z = 2.0 * offa / ab - 1.0;
        double p0 = 1.0, p1 = z;
        fx = F.leg[0];
        if (F.nleg > 1) fx = fma(F.leg[1], z, fx);
        for (int k = 1; k + 1 < F.nleg; ++k) {
            double p2 = ((2 * k + 1) * z * p1 - k * p0) / (k + 1);
            fx = fma(F.leg[k + 1], p2, fx);
            p0 = p1;
            p1 = p2;
        }
    }
    (void)skip_term_e;
    (void)e;
    (void)N;
    return fx;
}

// local load vector of element e for one forcing: loc[a] = (h/2) int f(x(xi)) phi^_a(xi) dxi
__global__ void k_element_loads(const double* nodes, int N, int P, double a, double b, ForcingDev F,
                                double* loc /* N x (P+1) */)
{
    const int e = blockIdx.x;
    const int lane = threadIdx.x;   // one warp
    const int M = P + 1;
    const double xl = nodes[e], h = nodes[e + 1] - nodes[e];
    const double ab = b - a;
    double acc[FDE_MAX_P + 1];
    for (int k = 0; k < M; ++k) acc[k] = 0.0;
    double Lb[FDE_MAX_P + 2];
    // (1) Legendre series: exact Gauss-Legendre
    if (F.nleg > 0) {
        int Q = (F.nleg + P) / 2 + 2;
        if (Q > FDE_QMAX) Q = FDE_QMAX;
        const double* gx = c_glx + Q * (Q - 1) / 2;
        const double* gw = c_glw + Q * (Q - 1) / 2;
        for (int k = lane; k < Q; k += 32) {
            double xi = gx[k];
            double offa = (xl - nodes[0]) + 0.5 * h * (xi + 1.0);
            double offb = (nodes[N] - nodes[e + 1]) + 0.5 * h * (1.0 - xi);
            double fx = forcing_smooth(F, offa, offb, ab, -1, e, N) * 0.5 * h * gw[k];
            leg_all(P + 1, xi, Lb);
            for (int q = 0; q < M; ++q) {
                double ph = (q == 0) ? 0.5 * (1 - xi) : (q == P ? 0.5 * (1 + xi) : Lb[q - 1] - Lb[q + 1]);
                acc[q] = fma(fx, ph, acc[q]);
            }
        }
    }
    // (2) power terms
    for (int t = 0; t < F.nterm; ++t) {
        const int side = F.side[t];
        const double pw = F.pw[t], cf = F.coef[t];
        const bool touches = (side == 0) ? (e == 0) : (e == N - 1);
        if (touches) {
            // Gauss-Jacobi with the endpoint weight: exact for the polynomial basis
            const double* jx = F.gj_x + t * F.qj;
            const double* jw = F.gj_w + t * F.qj;
            for (int k = lane; k < F.qj; k += 32) {
                double xi = jx[k];
                double w = jw[k] * pow(0.5 * h, pw) * 0.5 * h * cf;
                leg_all(P + 1, xi, Lb);
                for (int q = 0; q < M; ++q) {
                    double ph = (q == 0) ? 0.5 * (1 - xi) : (q == P ? 0.5 * (1 + xi) : Lb[q - 1] - Lb[q + 1]);
                    acc[q] = fma(w, ph, acc[q]);
                }
            }
        } else {
            // graded Gauss-Legendre cells toward the base point (cell size <= distance)
            const double o0 = (side == 0) ? (xl - nodes[0]) : (nodes[N] - nodes[e + 1]);
            const int Q = 24;
            const double* gx = c_glx + Q * (Q - 1) / 2;
            const double* gw = c_glw + Q * (Q - 1) / 2;
            double oa = o0;
            const double oend = o0 + h;
            int guard = 0;
            while (oa < oend && guard++ < 200) {
                double ob = fmin(oend, 2.0 * oa);
                for (int k = lane; k < Q; k += 32) {
                    double o = oa + 0.5 * (ob - oa) * (gx[k] + 1.0);
                    double w = 0.5 * (ob - oa) * gw[k] * cf * pow(o, pw);
                    // reference coordinate of this point in the element
                    double xi = (side == 0) ? (2.0 * (o - o0) / h - 1.0) : (1.0 - 2.0 * (o - o0) / h);
                    leg_all(P + 1, xi, Lb);
                    for (int q = 0; q < M; ++q) {
                        double ph = (q == 0) ? 0.5 * (1 - xi) : (q == P ? 0.5 * (1 + xi) : Lb[q - 1] - Lb[q + 1]);
                        acc[q] = fma(w, ph, acc[q]);
                    }
                }
                oa = ob;
            }
        }
    }
    // warp reduction (fixed order)
    for (int q = 0; q < M; ++q) {
        double v = acc[q];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) loc[(long long)e * M + q] = v;
    }
}

// G[r] (internal order) from element loads, minus the lifting c1 A[:,0] + c2 A[:,N]
__global__ void k_gather_loads(const double* loc, long long n, int N, int P, double c1, double c2,
                               const double* bnd, double* G)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int M = P + 1;
    DofTerms t = dof_terms(r, n, N, P);
    double g = 0.0;
    for (int x = 0; x < t.cnt; ++x) g += loc[(long long)t.e[x] * M + t.ml[x]];
    g -= c1 * bnd[r] + c2 * bnd[n + r];
    G[r] = g;
}

// ------------------------------------------------------------------ host side
static AsmDev make_dev(fde_op* op, int qm)
{
    AsmDev D;
    D.N = op->N;
    D.P = op->P;
    D.oma = 1.0 - op->prob.alpha;
    D.g0 = op->g0;
    D.nodes = op->tab.nodes.p;
    D.gjr_x = op->tab.gjr_x.p;
    D.gjr_w = op->tab.gjr_w.p;
    D.qr = op->tab.qr;
    D.gji_x = op->tab.gji_x.p;
    D.gji_w = op->tab.gji_w.p;
    D.qi = op->tab.qi;
    D.kself = op->tab.kself.p;
    D.qm = qm;
    return D;
}

static int qm_for(int P)
{
    // per-direction point capacity of the warp workspace (FDE_ASM_QM overrides)
    static const int env = getenv("FDE_ASM_QM") ? atoi(getenv("FDE_ASM_QM")) : 0;
    int q = P + 2;
    if (q < (env ? env : 24)) q = env ? env : 24;
    if (q > FDE_QMAX) q = FDE_QMAX;
    return q;
}

void asm_prepare_tables(fde_ctx* h, fde_op* op)
{
    upload_gl_tables(h->device);
    const int P = op->P;
    const double alpha = op->prob.alpha;
    op->tab.nodes.upload(op->nodes_h.data(), op->nodes_h.size(), h->stream);
    std::vector<double> x, w;
    op->tab.qr = P + 1;
    fdeq::gauss_jacobi(op->tab.qr, 0.0, 2.0 - alpha, x, w);
    op->tab.gjr_x.upload(x.data(), x.size(), h->stream);
    op->tab.gjr_w.upload(w.data(), w.size(), h->stream);
    op->tab.qi = P + 1;
    fdeq::gauss_jacobi(op->tab.qi, 0.0, 1.0 - alpha, x, w);
    op->tab.gji_x.upload(x.data(), x.size(), h->stream);
    op->tab.gji_w.upload(w.data(), w.size(), h->stream);
    op->tab.kself.alloc((size_t)P * P);
    op->tab.mref.alloc((size_t)(P + 1) * (P + 1));
    AsmDev D = make_dev(op, qm_for(P));
    k_selfref_kernel<<<1, 256, 0, h->stream>>>(D, op->tab.kself.p, op->tab.mref.p);
    FDE_CHECK_LAUNCH();
}

static void launch_pairs(fde_ctx* h, fde_op* op, int mode, int i0, int i1, int j0, int j1, const int* li,
                         const int* lj, const long long* ls, long long count, double* out)
{
    if (count <= 0) return;
    const int qm = qm_for(op->P);
    AsmDev D = make_dev(op, qm);
    size_t smem = (size_t)ASM_WARPS * ws_doubles(op->P, qm) * sizeof(double);
    long long blocks = ceil_div(count, ASM_WARPS);
    // grid.x limit is 2^31-1: fine for the sizes we handle; the common degrees with a compile-time P
#define FDE_PAIRS(PT_)                                                                                          \
    do {                                                                                                        \
        FDE_CUDA(cudaFuncSetAttribute(k_pairs_kernel<PT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        k_pairs_kernel<PT_><<<(unsigned)blocks, 32 * ASM_WARPS, smem, h->stream>>>(D, mode, i0, i1, j0, j1, li, lj, ls, \
                                                                                  count, out);                   \
    } while (0)
    // lane-per-pair far-field path for P = 4, 8 (FDE_ASM_LANE=0: one warp per pair)
    static const bool lane_path = !(getenv("FDE_ASM_LANE") && atoi(getenv("FDE_ASM_LANE")) == 0);
    const size_t lsmem = (size_t)ASM_LANE_WARPS * ws_doubles(op->P, qm) * sizeof(double);
#define FDE_PAIRS_LANE(PT_)                                                                                     \
    do {                                                                                                        \
        FDE_CUDA(cudaFuncSetAttribute(k_pairs_lane<PT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsmem)); \
        k_pairs_lane<PT_><<<(unsigned)ceil_div(count, 32LL * ASM_LANE_WARPS), 32 * ASM_LANE_WARPS, lsmem, h->stream>>>( \
            D, mode, i0, i1, j0, j1, li, lj, ls, count, out);                                                   \
    } while (0)
    // (only for large all-pairs launches -- the triangle or a rectangle of a dense assembly --
    // where nearly every pair is far: near-field lists and the few lag pairs of a Toeplitz
    // operator are mostly near pairs, which the lane path would serialise 32 to a warp)
    if (lane_path && (op->P == 8 || op->P == 4) && mode != 2 && count >= 32LL * 1024) {
        if (op->P == 8) FDE_PAIRS_LANE(8);
        else FDE_PAIRS_LANE(4);
    } else {
        switch (op->P) {
            case 4: FDE_PAIRS(4); break;
            case 8: FDE_PAIRS(8); break;
            case 16: FDE_PAIRS(16); break;
            default: FDE_PAIRS(0);
        }
    }
#undef FDE_PAIRS_LANE
#undef FDE_PAIRS
    FDE_CHECK_LAUNCH();
}

void asm_k_triangle(fde_ctx* h, fde_op* op, int i0, int i1, double* out)
{
    long long count = (long long)i1 * (i1 + 1) / 2 - (long long)i0 * (i0 + 1) / 2;
    launch_pairs(h, op, 0, i0, i1, 0, 0, nullptr, nullptr, nullptr, count, out);
}

void asm_k_rect(fde_ctx* h, fde_op* op, int i0, int i1, int j0, int j1, double* out)
{
    long long count = (long long)(i1 - i0) * (j1 - j0);
    launch_pairs(h, op, 1, i0, i1, j0, j1, nullptr, nullptr, nullptr, count, out);
}

void asm_k_list(fde_ctx* h, fde_op* op, const int* di, const int* dj, const long long* dslot, int64_t count,
                double* out)
{
    launch_pairs(h, op, 2, 0, 0, 0, 0, di, dj, dslot, count, out);
}

void asm_expand_dense(fde_ctx* h, fde_op* op, const double* Krow, const double* Kcol)
{
    KBand K;
    K.row = Krow;
    K.col = Kcol;
    K.b0 = op->e_lo;
    K.b1 = std::min(op->e_hi, op->N - 1);
    K.N = op->N;
    K.P2 = op->P * op->P;
    const long long rows = op->r1 - op->r0;
    if (rows <= 0) return;
    dim3 grid((unsigned)ceil_div(op->lda, 256), (unsigned)rows);
#define FDE_EXPAND(PT_)                                                                                           \
    k_expand_dense<PT_><<<grid, 256, 0, h->stream>>>(K, op->r0, op->r1, op->n, op->lda, op->N, op->P, op->prob.theta, \
                                                     op->prob.rho, op->tab.nodes.p, op->tab.mref.p, op->A.p)
    static const bool per_entry = getenv("FDE_EXPAND_ENTRY") != nullptr;   // (the previous per-entry kernel)
    static const bool per_pair = getenv("FDE_EXPAND_PAIRS") != nullptr;   // (round 1's per-pair kernel)
    const bool whole = op->r0 == 0 && op->r1 == op->n && K.b0 == 0 && K.b1 == op->N - 1;
    if (!per_entry && !per_pair && whole && (op->P == 4 || op->P == 8 || op->P == 16)) {
        // tiles of 8 x 8 element pairs over the whole triangle (world 1)
        const long long nt = ceil_div(op->N, EX_TE);
        const unsigned ntiles = (unsigned)(nt * (nt + 1) / 2);
        if (op->lda > op->n)   // padding columns [n, lda) of every row
            FDE_CUDA(cudaMemset2DAsync(op->A.p + op->n, op->lda * sizeof(double), 0, (op->lda - op->n) * sizeof(double),
                                       op->n, h->stream));
        const size_t smem = (size_t)(EX_TE + 1) * (EX_TE + 1) * op->P * (op->P + 1) * sizeof(double);
#define FDE_EXPAND_T(PT_)                                                                                              do {                                                                                                                   FDE_CUDA(cudaFuncSetAttribute(k_expand_tiles<PT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));         k_expand_tiles<PT_><<<ntiles, 256, smem, h->stream>>>(Krow, op->n, op->lda, op->N, op->prob.theta,                                                                     op->prob.rho, op->tab.nodes.p, op->tab.mref.p, op->A.p);     } while (0)
        switch (op->P) {
            case 4: FDE_EXPAND_T(4); break;
            case 8: FDE_EXPAND_T(8); break;
            default: FDE_EXPAND_T(16);
        }
#undef FDE_EXPAND_T
        FDE_CHECK_LAUNCH();
        return;
    }
    if (per_entry) {
        switch (op->P) {   // the common degrees with a compile-time P
            case 4: FDE_EXPAND(4); break;
            case 8: FDE_EXPAND(8); break;
            case 16: FDE_EXPAND(16); break;
            default: FDE_EXPAND(0);
        }
    } else {
        const long long e_first = op->r0 / op->P, e_last = (op->r1 - 1) / op->P;
        const long long col_elems = ceil_div(op->lda, (long long)op->P);
        dim3 pg((unsigned)ceil_div(col_elems, 128LL), (unsigned)(e_last - e_first + 1));
#define FDE_EXPAND_P(PT_)                                                                                       \
    k_expand_pairs<PT_><<<pg, 128, 0, h->stream>>>(K, op->r0, op->r1, op->n, op->lda, op->N, op->P, op->prob.theta, \
                                                    op->prob.rho, op->tab.nodes.p, op->tab.mref.p, op->A.p)
        switch (op->P) {
            case 4: FDE_EXPAND_P(4); break;
            case 8: FDE_EXPAND_P(8); break;
            case 16: FDE_EXPAND_P(16); break;
            default: FDE_EXPAND_P(0);
        }
#undef FDE_EXPAND_P
    }
#undef FDE_EXPAND
    FDE_CHECK_LAUNCH();
}

void asm_boundary_columns(fde_ctx* h, fde_op* op)
{
    const int N = op->N, P2 = op->P * op->P;
    op->bnd.alloc((size_t)2 * op->n);
    if (op->kb_row && op->e_lo == 0 && op->e_hi >= N) {
        // one GPU, dense path: every pair (i, 0) and (N-1, i) is already in the band of
        // pair moments the dense expansion read (same moments, same bits)
        KBand K;
        K.row = op->kb_row;
        K.col = op->kb_col;
        K.b0 = 0;
        K.b1 = N - 1;
        K.N = N;
        K.P2 = P2;
        k_boundary_cols<<<(unsigned)ceil_div(op->n, 256), 256, 0, h->stream>>>(
            K, op->n, N, op->P, op->prob.theta, op->prob.rho, op->tab.nodes.p, op->tab.mref.p, op->bnd.p);
        FDE_CHECK_LAUNCH();
        return;
    }
    // pair list: (i,0) -> slot i ; (N-1, i) -> slot N+i
    std::vector<int> li(2 * N), lj(2 * N);
    std::vector<long long> ls(2 * N);
    for (int i = 0; i < N; ++i) {
        li[i] = i; lj[i] = 0; ls[i] = i;
        li[N + i] = N - 1; lj[N + i] = i; ls[N + i] = N + i;
    }
    DBuf<int> di, dj;
    DBuf<long long> dsl;
    DBuf<double> tab;
    di.upload(li.data(), li.size(), h->stream);
    dj.upload(lj.data(), lj.size(), h->stream);
    dsl.upload(ls.data(), ls.size(), h->stream);
    tab.alloc((size_t)2 * N * P2);
    asm_k_list(h, op, di.p, dj.p, dsl.p, 2 * N, tab.p);
    KBnd K{tab.p, N, P2};
    k_boundary_cols<<<(unsigned)ceil_div(op->n, 256), 256, 0, h->stream>>>(
        K, op->n, N, op->P, op->prob.theta, op->prob.rho, op->tab.nodes.p, op->tab.mref.p, op->bnd.p);
    FDE_CHECK_LAUNCH();
}

void asm_rhs(fde_ctx* h, fde_op* op, const fde_forcing* f, int nrhs, double* G, int64_t ld)
{
    const int N = op->N, P = op->P, M = P + 1;
    DBuf<double> loc;
    loc.alloc((size_t)N * M);
    for (int r = 0; r < nrhs; ++r) {
        const fde_forcing& F = f[r];
        DBuf<double> leg, pw, cf, gjx, gjw;
        DBuf<int> side;
        ForcingDev FD{};
        FD.nleg = F.nleg;
        if (F.nleg > 0) {
            if (F.nleg > 64) fde_fail(FDE_EINVAL_PARAM, "forcing: at most 64 Legendre coefficients");
            leg.upload(F.leg, F.nleg, h->stream);
            FD.leg = leg.p;
        }
        FD.nterm = F.nterm;
        std::vector<double> jx, jw;
        const int qj = P / 2 + 3;
        if (F.nterm > 0) {
            side.upload(F.side, F.nterm, h->stream);
            pw.upload(F.power, F.nterm, h->stream);
            cf.upload(F.coef, F.nterm, h->stream);
            for (int t = 0; t < F.nterm; ++t) {
                if (!(F.power[t] > -1.0)) fde_fail(FDE_EINVAL_PARAM, "forcing: power terms need power > -1");
                std::vector<double> x, w;
                if (F.side[t] == 0)
                    fdeq::gauss_jacobi(qj, 0.0, F.power[t], x, w);
                else
                    fdeq::gauss_jacobi(qj, F.power[t], 0.0, x, w);
                jx.insert(jx.end(), x.begin(), x.end());
                jw.insert(jw.end(), w.begin(), w.end());
            }
            gjx.upload(jx.data(), jx.size(), h->stream);
            gjw.upload(jw.data(), jw.size(), h->stream);
            FD.side = side.p;
            FD.pw = pw.p;
            FD.coef = cf.p;
            FD.gj_x = gjx.p;
            FD.gj_w = gjw.p;
            FD.qj = qj;
        }
        k_element_loads<<<N, 32, 0, h->stream>>>(op->tab.nodes.p, N, P, op->prob.a, op->prob.b, FD, loc.p);
        FDE_CHECK_LAUNCH();
        k_gather_loads<<<(unsigned)ceil_div(op->n, 256), 256, 0, h->stream>>>(
            loc.p, op->n, N, P, op->prob.c1, op->prob.c2, op->bnd.p, G + (long long)r * ld);
        FDE_CHECK_LAUNCH();
    }
}

// ------------------------------------------------------ H-matrix leaf blocks
__global__ void k_expand_leaves(const double* Ktab, const LeafDesc* d, long long n, int N, int P, double theta,
                                double rho, const double* nodes, const double* mref, double* arena)
{
    const LeafDesc L = d[blockIdx.y];
    const int P2 = P * P;
    KRect K{Ktab + L.ktab * P2, L.i0, L.ni, L.j0, L.nj, P2};
    const long long tot = (long long)L.m * L.nc;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
         idx += (long long)gridDim.x * blockDim.x) {
        const int rr = (int)(idx % L.m), cc = (int)(idx / L.m);
        arena[L.out + (long long)cc * L.m + rr] = a_entry(K, L.ra + rr, L.ca + cc, n, N, P, theta, rho, nodes, mref);
    }
}

// the same leaves straight from the assembly's pair-moment band (world 1: every
// pair j <= i), while the dense expansion of A still runs: identical a_entry terms
__global__ void k_expand_leaves_band(KBand K, const LeafDesc* d, long long n, int N, int P, double theta, double rho,
                                     const double* nodes, const double* mref, double* arena)
{
    const LeafDesc L = d[blockIdx.y];
    const long long tot = (long long)L.m * L.nc;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
         idx += (long long)gridDim.x * blockDim.x) {
        const int rr = (int)(idx % L.m), cc = (int)(idx / L.m);
        arena[L.out + (long long)cc * L.m + rr] = a_entry(K, L.ra + rr, L.ca + cc, n, N, P, theta, rho, nodes, mref);
    }
}

void asm_expand_leaves_band(fde_ctx* h, fde_op* op, const LeafDesc* d, int nleaves, int maxentries, double* arena)
{
    KBand K;
    K.row = op->kb_row;
    K.col = op->kb_col;
    K.b0 = 0;
    K.b1 = op->N - 1;
    K.N = op->N;
    K.P2 = op->P * op->P;
    const unsigned gx = (unsigned)std::min<long long>(ceil_div(maxentries, 256), 64);
    for (int base = 0; base < nleaves; base += 65535) {
        unsigned cnt = (unsigned)std::min(65535, nleaves - base);
        k_expand_leaves_band<<<dim3(gx, cnt), 256, 0, h->stream>>>(K, d + base, op->n, op->N, op->P, op->prob.theta,
                                                                   op->prob.rho, op->tab.nodes.p, op->tab.mref.p, arena);
        FDE_CHECK_LAUNCH();
    }
}

void asm_expand_leaves(fde_ctx* h, fde_op* op, const double* Ktab, const LeafDesc* d, int nleaves, int maxentries,
                       double* arena)
{
    const unsigned gx = (unsigned)std::min<long long>(ceil_div(maxentries, 256), 64);
    for (int base = 0; base < nleaves; base += 65535) {
        unsigned cnt = (unsigned)std::min(65535, nleaves - base);
        k_expand_leaves<<<dim3(gx, cnt), 256, 0, h->stream>>>(Ktab, d + base, op->n, op->N, op->P, op->prob.theta,
                                                              op->prob.rho, op->tab.nodes.p, op->tab.mref.p, arena);
        FDE_CHECK_LAUNCH();
    }
}
