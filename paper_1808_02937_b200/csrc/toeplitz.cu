// stiffness_matvec, Toeplitz path (uniform meshes).
//
// On a uniform mesh t - s = (h/2)(xi - eta + 2k) for trial element j = i - k, so
// the pair moments K_ij = K_{k,0} depend only on the lag k (block-Toeplitz with
// P x P blocks, cf. Eq. (eq420)).  With d_e[n] the Legendre coefficients of
// du/dxi on element e (d_e[0] = (u~_{e+1} - u~_e)/2, d_e[p] = -(2p+1) u^p_e):
//     z_i[m]  = sum_{k>=0} sum_n K_k[m][n] d_{i-k}[n]      (S_l part, convolution)
//     z'_i[m] = sum_{k>=0} sum_n K_k[n][m] d_{i+k}[n]      (S_l^T part, correlation)
// Both are diagonalised by one 2N-point circulant embedding:
//     W^_m(w) = sum_n [theta K^_mn(w) + (1-theta) conj(K^_nm(w))] D^_n(w).
// Cost per matvec: P forward + P inverse FFTs of length L >= 2N and P^2 complex
// multiply-adds per frequency: O(P N log N + P^2 N) -- below the paper's
// O(P^2 N log N) for the same product.  Rows are then scattered back
// (modal: -(2p+1) w_e[p]; hat of node J: (w_{J-1}[0] - w_J[0])/2) and rho M x
// is added from the element mass matrices.
//
// Geometric meshes (h_{e+1} = q h_e for every element, the
// paper's second structured case): the nodes are x_e = o + c q^e for a virtual
// origin o, so t_i - s_j = q^j (t_{i-j} - s_0) and K_ij = w_j K_{i-j,0} with
// w_j = (h_j / h_0)^{1-alpha}: still Toeplitz after a diagonal scaling (the
// moment form needs only column scales, the Jacobians having cancelled):
//     z_i  = sum_k K_k (w d)_{i-k}              (S_l part: scale the input)
//     z'_i = w_i sum_k K_k^T d_{i+k}            (S_l^T part: scale the output)
// -- two spectral products (theta K^ on FFT(w d), (1-theta) K^H on FFT(d)).
#include <cmath>

#include "fde_internal.h"

#define FFT_THREADS 512

// in-place radix-2 FFT of L complex values in shared memory (bit-reversed input
// order handled by the loader); sign = -1 forward, +1 inverse (unnormalised)
__device__ void smem_fft(double2* a, int L, int logL, const double2* tw, int inverse)
{
    for (int len = 2; len <= L; len <<= 1) {
        const int half = len >> 1, step = L / len;
        for (int t = threadIdx.x; t < (L >> 1); t += blockDim.x) {
            const int grp = t / half, pos = t - grp * half;
            const int i = grp * len + pos, j = i + half;
            double2 w = tw[pos * step];
            if (inverse) w.y = -w.y;
            const double2 u = a[i], v = a[j];
            const double2 vw = make_double2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
            a[i] = make_double2(u.x + vw.x, u.y + vw.y);
            a[j] = make_double2(u.x - vw.x, u.y - vw.y);
        }
        __syncthreads();
    }
}

__device__ inline int bitrev(int x, int logL) { return (int)(__brev((unsigned)x) >> (32 - logL)); }

__global__ void k_twiddles(double2* tw, int L)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= L / 2) return;
    double s, c;
    sincospi(-2.0 * (double)k / (double)L, &s, &c);   // exp(-2 pi i k / L)
    tw[k] = make_double2(c, s);
}

// forward FFT of the lag sequences sym[k][mn], k < N, zero padded to L -> Khat[mn][w]
__global__ void k_symbol_fft(const double* sym, int N, int P2, int L, int logL, const double2* tw, double2* Khat)
{
    extern __shared__ double2 sbuf[];
    const int mn = blockIdx.x;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        const int src = bitrev(k, logL);
        sbuf[k] = make_double2(src < N ? sym[(long long)src * P2 + mn] : 0.0, 0.0);
    }
    __syncthreads();
    smem_fft(sbuf, L, logL, tw, 0);
    for (int k = threadIdx.x; k < L; k += blockDim.x) Khat[(long long)mn * L + k] = sbuf[k];
}

// spec[w][m][n] = theta Khat[m][n](w) + (1-theta) conj(Khat[n][m](w))
// (mode 1: theta Khat[m][n] only; mode 2: (1-theta) conj(Khat[n][m]) only)
__global__ void k_symbol_combine(const double2* Khat, int P, int L, double theta, double2* spec, int mode = 0)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long tot = (long long)L * P * P;
    if (idx >= tot) return;
    const int w = (int)(idx / (P * P));
    const int mn = (int)(idx - (long long)w * P * P);
    const int m = mn / P, n = mn - m * P;
    const double2 a = Khat[(long long)(m * P + n) * L + w];
    const double2 b = Khat[(long long)(n * P + m) * L + w];
    const double ta = mode == 2 ? 0.0 : theta, tb = mode == 1 ? 0.0 : 1.0 - theta;
    spec[idx] = make_double2(ta * a.x + tb * b.x, ta * a.y - tb * b.y);
}

// gather d_e[n] (internal-order x, column c) and forward FFT -> Dhat[c][n][w]
__global__ void k_gather_fft(const double* x, long long ldx, int N, int P, int L, int logL, const double2* tw,
                             double2* Dhat, const double* wsc)   // wsc: per-element input scales (or null)
{
    extern __shared__ double2 sbuf[];
    const int nn = blockIdx.x, c = blockIdx.y;
    const double* xc = x + c * ldx;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
        const int e = bitrev(k, logL);
        double v = 0.0;
        if (e < N) {
            if (nn == 0) {
                const double ur = (e + 1 <= N - 1) ? xc[(long long)(e + 1) * P - 1] : 0.0;   // hat node e+1
                const double ul = (e >= 1) ? xc[(long long)e * P - 1] : 0.0;                // hat node e
                v = 0.5 * (ur - ul);
            } else {
                v = -(2.0 * nn + 1.0) * xc[(long long)e * P + nn - 1];
            }
            if (wsc) v *= wsc[e];
        }
        sbuf[k] = make_double2(v, 0.0);
    }
    __syncthreads();
    smem_fft(sbuf, L, logL, tw, 0);
    double2* out = Dhat + ((long long)c * P + nn) * L;
    for (int k = threadIdx.x; k < L; k += blockDim.x) out[k] = sbuf[k];
}

// W^[c][m][w] = sum_n spec[w][m][n] D^[c][n][w]
__global__ void k_symbol_apply(const double2* spec, const double2* Dhat, int P, int L, int nrhs, double2* What)
{
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long tot = (long long)L * P;
    const int c = blockIdx.y;
    if (idx >= tot) return;
    const int m = (int)(idx / L), w = (int)(idx - (long long)m * L);
    const double2* D = Dhat + (long long)c * P * L;
    const double2* S = spec + ((long long)w * P + m) * P;
    double re = 0.0, im = 0.0;
    for (int n = 0; n < P; ++n) {
        const double2 s = S[n], d = D[(long long)n * L + w];
        re = fma(s.x, d.x, fma(-s.y, d.y, re));
        im = fma(s.x, d.y, fma(s.y, d.x, im));
    }
    What[((long long)c * P + m) * L + w] = make_double2(re, im);
}

// inverse FFT of W^[c][m] -> wout[c][m][e] = Re(.)/L, e < N
// (wsc: per-element output scales, accumulated into wout; null: wout overwritten)
__global__ void k_ifft(const double2* What, int N, int P, int L, int logL, const double2* tw, double* wout,
                       const double* wsc)
{
    extern __shared__ double2 sbuf[];
    const int m = blockIdx.x, c = blockIdx.y;
    const double2* in = What + ((long long)c * P + m) * L;
    for (int k = threadIdx.x; k < L; k += blockDim.x) sbuf[k] = in[bitrev(k, logL)];
    __syncthreads();
    smem_fft(sbuf, L, logL, tw, 1);
    const double invL = 1.0 / (double)L;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
        double* o = wout + ((long long)c * P + m) * N + e;
        if (wsc) *o = fma(wsc[e], sbuf[e].x * invL, *o);
        else *o = sbuf[e].x * invL;
    }
}

// y rows (internal order): sum of test terms + rho (M x)
__global__ void k_toeplitz_scatter(const double* wv, const double* x, long long ldx, const double* nodes,
                                   const double* mref, int N, int P, long long n, double rho, double* y,
                                   long long ldy)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= n) return;
    const double* w = wv + (long long)c * P * N;
    const double* xc = x + c * ldx;
    const int e = (int)(r / P), q = (int)(r - (long long)e * P);
    const int M = P + 1;
    double v = 0.0, mass = 0.0;
    // element-local coefficient of local function b in element el
    auto xloc = [&](int el, int b) -> double {
        if (b == 0) return el >= 1 ? xc[(long long)el * P - 1] : 0.0;
        if (b == P) return (el + 1 <= N - 1) ? xc[(long long)(el + 1) * P - 1] : 0.0;
        return xc[(long long)el * P + b - 1];
    };
    if (q < P - 1) {
        const int p = q + 1;
        v = -(2.0 * p + 1.0) * w[(long long)p * N + e];
        const double hh = 0.5 * (nodes[e + 1] - nodes[e]);
        for (int b = 0; b < M; ++b) mass = fma(hh * mref[p * M + b], xloc(e, b), mass);
    } else {
        v = 0.5 * (w[e] - w[e + 1]);
        const double h0 = 0.5 * (nodes[e + 1] - nodes[e]);
        const double h1 = 0.5 * (nodes[e + 2] - nodes[e + 1]);
        for (int b = 0; b < M; ++b) {
            mass = fma(h0 * mref[P * M + b], xloc(e, b), mass);
            mass = fma(h1 * mref[0 * M + b], xloc(e + 1, b), mass);
        }
    }
    y[c * ldy + r] = v + rho * mass;
}

static int ilog2(int L)
{
    int k = 0;
    while ((1 << k) < L) ++k;
    return k;
}

void toeplitz_prepare(fde_ctx* h, fde_op* op)
{
    const int N = op->N, P = op->P, P2 = P * P;
    int L = 2;
    while (L < 2 * N) L <<= 1;
    if ((size_t)L * sizeof(double2) > 200 * 1024)
        fde_fail(FDE_EUNSUPPORTED_MESH, "Toeplitz path: 2N exceeds the single-CTA FFT size (N <= 6400)");
    op->L = L;
    const int logL = ilog2(L);
    // lag symbols K_{k,0}, k < N
    std::vector<int> li(N), lj(N, 0);
    std::vector<long long> ls(N);
    for (int k = 0; k < N; ++k) {
        li[k] = k;
        ls[k] = k;
    }
    DBuf<int> di, dj;
    DBuf<long long> dsl;
    di.upload(li.data(), N, h->stream);
    dj.upload(lj.data(), N, h->stream);
    dsl.upload(ls.data(), N, h->stream);
    op->sym.alloc((size_t)N * P2);
    asm_k_list(h, op, di.p, dj.p, dsl.p, N, op->sym.p);
    op->twid.alloc((size_t)L);   // L/2 double2 = L doubles
    double2* tw = reinterpret_cast<double2*>(op->twid.p);
    k_twiddles<<<(unsigned)ceil_div(L / 2, 256), 256, 0, h->stream>>>(tw, L);
    FDE_CHECK_LAUNCH();
    DBuf<double2> Khat;
    Khat.alloc((size_t)P2 * L);
    const size_t smem = (size_t)L * sizeof(double2);
    FDE_CUDA(cudaFuncSetAttribute(k_symbol_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FDE_CUDA(cudaFuncSetAttribute(k_gather_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FDE_CUDA(cudaFuncSetAttribute(k_ifft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_symbol_fft<<<P2, FFT_THREADS, smem, h->stream>>>(op->sym.p, N, P2, L, logL, tw, Khat.p);
    FDE_CHECK_LAUNCH();
    op->spec.alloc((size_t)(op->geometric ? 4 : 2) * L * P2);
    double2* spec = reinterpret_cast<double2*>(op->spec.p);
    const unsigned gb = (unsigned)ceil_div((long long)L * P2, 256);
    if (!op->geometric) {
        k_symbol_combine<<<gb, 256, 0, h->stream>>>(Khat.p, P, L, op->prob.theta, spec);
        FDE_CHECK_LAUNCH();
    } else {
        k_symbol_combine<<<gb, 256, 0, h->stream>>>(Khat.p, P, L, op->prob.theta, spec, 1);
        FDE_CHECK_LAUNCH();
        k_symbol_combine<<<gb, 256, 0, h->stream>>>(Khat.p, P, L, op->prob.theta, spec + (size_t)L * P2, 2);
        FDE_CHECK_LAUNCH();
        std::vector<double> w(N);
        const double h0 = op->nodes_h[1] - op->nodes_h[0];
        for (int e = 0; e < N; ++e) w[e] = std::pow((op->nodes_h[e + 1] - op->nodes_h[e]) / h0, 1.0 - op->prob.alpha);
        op->wsc.upload(w.data(), N, h->stream);
    }
    FDE_CUDA(cudaStreamSynchronize(h->stream));
}

void toeplitz_matvec(fde_ctx* h, fde_op* op, const double* x, int64_t ldx, double* y, int64_t ldy, int nrhs)
{
    const int N = op->N, P = op->P, L = op->L, logL = ilog2(L);
    // (handle-owned scratch: the spectra of x and of the product, the inverse transforms)
    DBuf<double2>& Dhat = h->t_Dhat;
    DBuf<double2>& What = h->t_What;
    DBuf<double>& wv = h->t_wv;
    const size_t need = (size_t)nrhs * P * L;
    if (Dhat.n < need) Dhat.alloc(need);
    if (What.n < need) What.alloc(need);
    if (wv.n < (size_t)nrhs * P * N) wv.alloc((size_t)nrhs * P * N);
    const double2* tw = reinterpret_cast<const double2*>(op->twid.p);
    const size_t smem = (size_t)L * sizeof(double2);
    const double2* spec = reinterpret_cast<const double2*>(op->spec.p);
    // uniform: one pass with the combined symbol; geometric: the S_l pass on the
    // scaled input, then the S_l^T pass with scaled, accumulated output
    for (int pass = 0; pass < (op->geometric ? 2 : 1); ++pass) {
        const double* win = (op->geometric && pass == 0) ? op->wsc.p : nullptr;
        const double* wout = (op->geometric && pass == 1) ? op->wsc.p : nullptr;
        k_gather_fft<<<dim3(P, nrhs), FFT_THREADS, smem, h->stream>>>(x, ldx, N, P, L, logL, tw, Dhat.p, win);
        FDE_CHECK_LAUNCH();
        k_symbol_apply<<<dim3((unsigned)ceil_div((long long)L * P, 256), nrhs), 256, 0, h->stream>>>(
            spec + (size_t)pass * L * P * P, Dhat.p, P, L, nrhs, What.p);
        FDE_CHECK_LAUNCH();
        k_ifft<<<dim3(P, nrhs), FFT_THREADS, smem, h->stream>>>(What.p, N, P, L, logL, tw, wv.p, wout);
        FDE_CHECK_LAUNCH();
    }
    k_toeplitz_scatter<<<dim3((unsigned)ceil_div(op->n, 256), nrhs), 256, 0, h->stream>>>(
        wv.p, x, ldx, op->tab.nodes.p, op->tab.mref.p, N, P, op->n, op->prob.rho, y, ldy);
    FDE_CHECK_LAUNCH();
}
