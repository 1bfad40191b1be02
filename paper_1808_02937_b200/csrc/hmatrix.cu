#include <chrono>
// hmatrix_build: H-matrix approximation A~ = rho M + theta H + (1-theta) H^T of
// the SEM stiffness (Eq. (approxmat)/(approxsys); reading A2).
//
//  * cluster tree: binary median split of element ranges down to n_min elements
//    (reading A9); a cluster carries the modal dofs of its elements and the hats
//    of their right nodes (element-interleaved order => contiguous dof range);
//    its support is the union of the supports, [x_e0, x_{e1+1}].
//  * partition: a block is an admissible leaf if max(diam) <= lambda dist
//    (Eq. (admis)), a dense leaf if not and one cluster is a leaf,
//    otherwise it is subdivided 2 x 2.
//  * admissible leaves carry the Taylor factors of Lemma 3.2:
//    Q = gamma0 int h_nu phi', W = int g_nu phi',
//    expanded in s about the column-cluster midpoint, or in t about the row
//    midpoint when the column cluster is larger (Remark).
//    Lower blocks (row cluster right of column cluster) store
//    U = theta Q, V = W; upper blocks U = (1-theta) W, V = Q of the mirrored pair.
//  * inadmissible leaves hold exact entries of A, computed from
//    the pair moments K_ij of assemble.cu for the element pairs of the leaf.
//  All arithmetic runs on the device; the host only builds the tree.
#include <algorithm>
#include <cmath>

#include "hmatrix.h"


// ------------------------------------------------------------ structure
static int build_cluster(HStruct& S, const std::vector<double>& x, int e0, int e1, int n_min)
{
    HCluster c;
    c.e0 = e0;
    c.e1 = e1;
    c.r0 = (int64_t)e0 * S.P;
    c.r1 = std::min((int64_t)e1 * S.P, S.n);
    c.child[0] = c.child[1] = -1;
    c.lo = x[e0];
    c.hi = x[std::min(e1 + 1, S.N)];
    c.nlo = e0;
    c.nhi = std::min(e1 + 1, S.N);
    c.kind = HC_INTERLEAVED;
    int id = (int)S.cl.size();
    S.cl.push_back(c);
    if (e1 - e0 > n_min) {
        int mid = (e0 + e1) / 2;
        int a = build_cluster(S, x, e0, mid, n_min);
        int b = build_cluster(S, x, mid, e1, n_min);
        S.cl[id].child[0] = a;
        S.cl[id].child[1] = b;
    }
    return id;
}

// the paper's partition: a modal tree over elements (a cluster
// [e0, e1) holds the dofs (e, p) in the paper order e (P-1) + p - 1, support
// [x_e0, x_e1]) and a nodal tree over the interior nodes (a cluster [j0, j1) holds
// the hats of nodes j0..j1-1, paper dofs N (P-1) + j - 1, support [x_{j0-1}, x_{j1}])
static int build_modal(HStruct& S, const std::vector<double>& x, int e0, int e1, int n_min)
{
    HCluster c;
    c.kind = HC_MODAL;
    c.e0 = e0;
    c.e1 = e1;
    c.r0 = (int64_t)e0 * (S.P - 1);
    c.r1 = (int64_t)e1 * (S.P - 1);
    c.child[0] = c.child[1] = -1;
    c.lo = x[e0];
    c.hi = x[e1];
    c.nlo = e0;
    c.nhi = e1;
    const int id = (int)S.cl.size();
    S.cl.push_back(c);
    if (e1 - e0 > n_min) {
        const int mid = (e0 + e1) / 2;
        const int a = build_modal(S, x, e0, mid, n_min);
        const int b = build_modal(S, x, mid, e1, n_min);
        S.cl[id].child[0] = a;
        S.cl[id].child[1] = b;
    }
    return id;
}
static int build_nodal(HStruct& S, const std::vector<double>& x, int j0, int j1, int n_min)
{
    HCluster c;
    c.kind = HC_NODAL;
    c.e0 = j0;
    c.e1 = j1;
    const int64_t nm = (int64_t)S.N * (S.P - 1);
    c.r0 = nm + j0 - 1;
    c.r1 = nm + j1 - 1;
    c.child[0] = c.child[1] = -1;
    c.lo = x[j0 - 1];
    c.hi = x[j1];
    c.nlo = j0 - 1;
    c.nhi = j1;
    const int id = (int)S.cl.size();
    S.cl.push_back(c);
    if (j1 - j0 > n_min) {
        const int mid = (j0 + j1) / 2;
        const int a = build_nodal(S, x, j0, mid, n_min);
        const int b = build_nodal(S, x, mid, j1, n_min);
        S.cl[id].child[0] = a;
        S.cl[id].child[1] = b;
    }
    return id;
}

static bool admissible(const HCluster& t, const HCluster& s, double lam)
{
    const double diam = std::max(t.hi - t.lo, s.hi - s.lo);
    const double dist = std::max(std::max(s.lo - t.hi, t.lo - s.hi), 0.0);
    return dist > 0.0 && diam <= lam * dist;
}

static int build_block(HStruct& S, int t, int s, double lam, int level)
{
    HBlock b;
    b.tau = t;
    b.sig = s;
    b.m = S.cl[t].r1 - S.cl[t].r0;
    b.n = S.cl[s].r1 - S.cl[s].r0;
    for (int k = 0; k < 4; ++k) b.child[k] = -1;
    b.off = 0;
    b.kcap = 0;
    b.lower = 0;
    S.depth = std::max(S.depth, level);
    const HCluster &T = S.cl[t], &Sg = S.cl[s];
    if (admissible(T, Sg, lam)) {
        b.type = HB_LR;
        b.lower = (T.lo >= Sg.hi) ? 1 : 0;   // row cluster right of column cluster
    } else if (T.child[0] < 0 || Sg.child[0] < 0) {
        b.type = HB_DENSE;
    } else {
        b.type = HB_HIER;
    }
    int id = (int)S.bl.size();
    S.bl.push_back(b);
    if (b.type == HB_HIER) {
        int k = 0;
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 2; ++c) {
                int ch = build_block(S, T.child[a], Sg.child[c], lam, level + 1);
                S.bl[id].child[k++] = ch;
            }
    }
    return id;
}

void hstruct_build(HStruct& S, const std::vector<double>& nodes, int P, int n_min, double lam, int partition)
{
    S.N = (int)nodes.size() - 1;
    S.P = P;
    S.n = (int64_t)S.N * P - 1;
    S.cl.clear();
    S.bl.clear();
    S.depth = 0;
    S.paper = partition;
    int root;
    if (!partition) {
        root = build_cluster(S, nodes, 0, S.N, std::max(1, n_min));
    } else {
        // virtual root [modal | nodal] (never admissible: its supports overlap), so the
        // block tree's first level is the 2 x 2 superblock [B F; E C] of PAPER.md:168-172
        const bool has_modal = P > 1, has_nodal = S.N > 1;
        if (has_modal && has_nodal) {
            HCluster c;
            c.kind = HC_ROOT;
            c.e0 = 0;
            c.e1 = S.N;
            c.r0 = 0;
            c.r1 = S.n;
            c.lo = nodes[0];
            c.hi = nodes[S.N];
            c.nlo = 0;
            c.nhi = S.N;
            root = (int)S.cl.size();
            S.cl.push_back(c);
            const int a = build_modal(S, nodes, 0, S.N, std::max(1, n_min));
            const int b = build_nodal(S, nodes, 1, S.N, std::max(1, n_min));
            S.cl[root].child[0] = a;
            S.cl[root].child[1] = b;
        } else if (has_modal) {
            root = build_modal(S, nodes, 0, S.N, std::max(1, n_min));
        } else {
            root = build_nodal(S, nodes, 1, S.N, std::max(1, n_min));
        }
    }
    S.root = build_block(S, root, root, lam, 0);
}

// ------------------------------------------------------------- device side
struct FDesc {
    int mode;          // cluster kind: HC_INTERLEAVED, HC_MODAL, HC_NODAL (dof of a row)
    int e0;            // first element of the cluster (first node for HC_NODAL)
    int rows;          // dof rows
    int64_t out;       // arena offset of the factor (rows x kcap col-major, ld rows)
    int kind;          // 0: power  pref * alt^nu * c_nu * z^{1-alpha-nu},  1: polynomial pref * (x-x0)^nu
    int sgn;           // power: z = sgn * (x - x0)
    int alt;           // power: multiply by (-1)^nu
    double pref;
    int ea;            // x0 = x_ea + oa  (anchor node + offset, avoids cancellation)
    double oa;
};

__global__ void k_factors(const FDesc* fd, const double* nodes, int N, int P, int R, double alpha, double g0,
                          double* arena)
{
    __shared__ double red[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const FDesc D = fd[blockIdx.y];
    const int row = blockIdx.x * 8 + wid;
    if (row >= D.rows) return;
    // the row's dof as (element e, q): q < P - 1 modal psi_{q+1} of e, q = P - 1 hat of node e + 1
    int e, q;
    if (D.mode == HC_MODAL) {
        e = D.e0 + row / (P - 1);
        q = row - (row / (P - 1)) * (P - 1);
    } else if (D.mode == HC_NODAL) {
        e = D.e0 + row - 1;
        q = P - 1;
    } else {
        e = D.e0 + row / P;
        q = row - (row / P) * P;
    }
    double acc[32];
    for (int nu = 0; nu < R; ++nu) acc[nu] = 0.0;
    // 32-point Gauss-Legendre, one point per lane, over the 1 or 2 elements of the dof
    const int npass = (q < P - 1) ? 1 : 2;
    for (int pass = 0; pass < npass; ++pass) {
        const int el = (q < P - 1) ? e : (pass == 0 ? e : e + 1);
        if (el >= N) continue;
        const double xl = nodes[el], h = nodes[el + 1] - nodes[el];
        // Gauss-Legendre 32 from constant memory (assemble.cu)
        const int Q = 32;
        const double xi = c_glx[Q * (Q - 1) / 2 + lane];
        const double wq = c_glw[Q * (Q - 1) / 2 + lane];
        double dphi;
        if (q < P - 1) {
            const int p = q + 1;
            double p0 = 1.0, p1 = xi, Lp = (p == 0) ? 1.0 : xi;
            for (int k = 1; k < p; ++k) {
                double p2 = ((2 * k + 1) * xi * p1 - k * p0) / (k + 1);
                p0 = p1;
                p1 = p2;
                Lp = p2;
            }
            dphi = (2.0 / h) * (-(2.0 * p + 1.0)) * Lp;
        } else {
            dphi = (pass == 0) ? 1.0 / h : -1.0 / h;
        }
        // x - x0 from node differences
        const double dx = (xl - nodes[D.ea]) + 0.5 * h * (xi + 1.0) - D.oa;
        const double w = wq * 0.5 * h * dphi;
        if (D.kind == 0) {
            const double z = D.sgn * dx;
            const double lz = log(z);
            double c = 1.0;
            for (int nu = 0; nu < R; ++nu) {
                double term = c * exp((1.0 - alpha - nu) * lz);
                if (D.alt && (nu & 1)) term = -term;
                acc[nu] = fma(w, term, acc[nu]);
                c *= (alpha - 1.0 + nu) / (nu + 1.0);
            }
        } else {
            double pw = 1.0;
            for (int nu = 0; nu < R; ++nu) {
                acc[nu] = fma(w, pw, acc[nu]);
                pw *= dx;
            }
        }
    }
    for (int nu = 0; nu < R; ++nu) {
        double v = acc[nu];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[wid][nu] = v;
    }
    __syncwarp();
    if (lane < R) arena[D.out + (int64_t)lane * D.rows + row] = D.pref * red[wid][lane];
    (void)g0;
}


struct DenseDesc {
    int type;
    int64_t r0, c0;
    int m, n;
    int64_t off;
    int kcap;
    int blk;
};

__global__ void k_blocks_to_dense(const DenseDesc* dd, const double* dense, const double* lr, const int* rank,
                                  double* out, int64_t ldo)
{
    const DenseDesc D = dd[blockIdx.y];
    const int64_t tot = (int64_t)D.m * D.n;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % D.m), j = (int)(idx / D.m);
        double v;
        if (D.type == HB_DENSE) {
            v = dense[D.off + (int64_t)j * D.m + i];
        } else {
            const int k = rank[D.blk];
            const double* U = lr + D.off;
            const double* V = U + (int64_t)D.m * D.kcap;
            v = 0.0;
            for (int t = 0; t < k; ++t) v = fma(U[(int64_t)t * D.m + i], V[(int64_t)t * D.n + j], v);
        }
        out[(D.c0 + j) * ldo + D.r0 + i] = v;
    }
}

// ------------------------------------------------------------------ host
void hm_leaves(const HStruct& S, int b, std::vector<int>& out)
{
    const HBlock& B = S.bl[b];
    if (B.type == HB_HIER) {
        for (int k = 0; k < 4; ++k) hm_leaves(S, B.child[k], out);
    } else {
        out.push_back(b);
    }
}

// one 32 x 32 tile of a dense leaf copied from the row-major dense operator
struct LeafTile {
    int64_t r, c;      // first row / column (internal order)
    int64_t out;       // arena offset of the tile's first element
    int64_t ldo;       // leaf rows (column-major ld)
    int m, n;          // tile extent
};

__global__ void k_leaf_from_dense(const LeafTile* T, const double* __restrict__ A, long long lda, double* arena)
{
    __shared__ double t[32][33];
    const LeafTile d = T[blockIdx.x];
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int r = ty; r < d.m; r += 8)   // coalesced along the row of A
        if (tx < d.n) t[r][tx] = A[(d.r + r) * lda + d.c + tx];
    __syncthreads();
    for (int c = ty; c < d.n; c += 8)   // coalesced along the leaf column
        if (tx < d.m) arena[d.out + (int64_t)c * d.ldo + tx] = t[tx][c];
}

// the same for leaves in the paper order (paper partition): dof i of the paper order
// is internal dof e P + p - 1 (modal (e, p)) or (j - 1) P + P - 1 (hat of node j)
__device__ __forceinline__ long long internal_of_paper_dof(long long i, int N, int P)
{
    const long long nm = (long long)N * (P - 1);
    if (i < nm) {
        const long long e = i / (P - 1);
        return e * P + (i - e * (P - 1));
    }
    return (i - nm) * P + (P - 1);
}
__global__ void k_leaf_from_dense_paper(const LeafTile* T, const double* __restrict__ A, long long lda, double* arena,
                                        int N, int P)
{
    __shared__ double t[32][33];
    const LeafTile d = T[blockIdx.x];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long ci = tx < d.n ? internal_of_paper_dof(d.c + tx, N, P) : 0;
    for (int r = ty; r < d.m; r += 8)
        if (tx < d.n) t[r][tx] = A[internal_of_paper_dof(d.r + r, N, P) * lda + ci];
    __syncthreads();
    for (int c = ty; c < d.n; c += 8)
        if (tx < d.m) arena[d.out + (int64_t)c * d.ldo + tx] = t[tx][c];
}

fde_hm* hm_build(fde_ctx* h, fde_op* op, int R, double lam, int n_min, bool recompute, bool from_band, int partition)
{
    if (R < 1 || R > 32) fde_fail(FDE_EINVAL_PARAM, "hmatrix_build: R must be in [1, 32]");
    if (!(lam > 0)) fde_fail(FDE_EINVAL_PARAM, "hmatrix_build: lambda must be > 0");
    if (n_min < 1) fde_fail(FDE_EINVAL_PARAM, "hmatrix_build: n_min must be >= 1");
    fde_hm* hm = new fde_hm();
    hm->tm.start(h->stream);   // (returns without waiting; see LazyTimer)
    static const bool dbg_t = getenv("FDE_DEBUG_HBUILD") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto tick = [&](const char* what) {
        if (!dbg_t) return;
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "hbuild host %-12s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    try {
        hm->op = op;
        hm->R = R;
        hm->lam = lam;
        hm->n_min = n_min;
        HStruct& S = hm->S;
        hstruct_build(S, op->nodes_h, op->P, n_min, lam, partition);
        if (partition && !(op->A.p && op->r0 == 0 && op->r1 == op->n))
            fde_fail(FDE_EINVAL_PARAM, "hmatrix_build: the paper partition needs the resident dense operator (world 1, FDE_OP_DENSE)");
        tick("structure");
        const int N = op->N, P = op->P;
        const std::vector<double>& x = op->nodes_h;
        std::vector<int> lv;
        hm_leaves(S, S.root, lv);
        // arenas
        int64_t doff = 0, loff = 0;
        for (int b : lv) {
            HBlock& B = S.bl[b];
            if (B.type == HB_DENSE) {
                B.off = doff;
                doff += B.m * B.n;
                hm->n_dense++;
            } else {
                B.kcap = R;
                B.off = loff;
                loff += (B.m + B.n) * R;
                hm->n_lr++;
            }
        }
        hm->dense_words = doff;
        hm->lr_words = loff;
        hm->dense.alloc(std::max<int64_t>(doff, 1));
        hm->lr.alloc(std::max<int64_t>(loff, 1));
        tick("arenas");
        std::vector<int> rank_h(S.bl.size(), 0);
        // ---- low-rank factors
        std::vector<FDesc> fd;
        const double theta = op->prob.theta, g0 = op->g0;
        for (int b : lv) {
            HBlock& B = S.bl[b];
            if (B.type != HB_LR) continue;
            rank_h[b] = R;
            // expansion pair: test cluster T (right), trial cluster Sg (left)
            const int tcl = B.lower ? B.tau : B.sig;
            const int scl = B.lower ? B.sig : B.tau;
            const HCluster &T = S.cl[tcl], &Sg = S.cl[scl];
            const bool s_exp = (Sg.hi - Sg.lo) <= (T.hi - T.lo);
            FDesc q{}, w{};
            // Q on the test cluster, W on the trial cluster
            q.mode = T.kind;
            q.e0 = T.e0;
            q.rows = (int)(T.r1 - T.r0);
            w.mode = Sg.kind;
            w.e0 = Sg.e0;
            w.rows = (int)(Sg.r1 - Sg.r0);
            const double scale = B.lower ? theta : (1.0 - theta);
            if (s_exp) {
                // s0 = mid(support of Sg): anchor at its left node
                const int ea = Sg.nlo;
                const double oa = 0.5 * (x[Sg.nhi] - x[Sg.nlo]);
                q.kind = 0; q.sgn = 1; q.alt = 0; q.pref = g0; q.ea = ea; q.oa = oa;
                w.kind = 1; w.sgn = 1; w.alt = 0; w.pref = 1.0; w.ea = ea; w.oa = oa;
            } else {
                const int ea = T.nlo;
                const double oa = 0.5 * (x[T.nhi] - x[T.nlo]);
                q.kind = 1; q.sgn = 1; q.alt = 0; q.pref = g0; q.ea = ea; q.oa = oa;
                w.kind = 0; w.sgn = -1; w.alt = 1; w.pref = 1.0; w.ea = ea; w.oa = oa;
            }
            // lower: U = theta Q (rows tau = T), V = W (rows sigma = Sg)
            // upper: U = (1-theta) W (rows tau = Sg), V = Q (rows sigma = T)
            const int64_t Uoff = B.off, Voff = B.off + B.m * R;
            if (B.lower) {
                q.pref *= scale;
                q.out = Uoff;
                w.out = Voff;
            } else {
                w.pref *= scale;
                w.out = Uoff;
                q.out = Voff;
            }
            fd.push_back(q);
            fd.push_back(w);
        }
        DBuf<FDesc> dfd;
        if (!fd.empty()) {
            dfd.upload(fd.data(), fd.size(), h->stream);
            int maxrows = 0;
            for (auto& f : fd) maxrows = std::max(maxrows, f.rows);
            // grid.y limit 65535: chunk the descriptor list
            for (size_t base = 0; base < fd.size(); base += 65535) {
                unsigned cnt = (unsigned)std::min<size_t>(65535, fd.size() - base);
                k_factors<<<dim3((unsigned)ceil_div(maxrows, 8), cnt), 256, 0, h->stream>>>(
                    dfd.p + base, op->tab.nodes.p, N, P, R, op->prob.alpha, g0, hm->lr.p);
                FDE_CHECK_LAUNCH();
            }
        }
        tick("factors");
        // ---- dense leaves: K tables + expansion
        std::vector<LeafDesc> ld;
        std::vector<int> li, lj;
        std::vector<long long> ls;
        int64_t kslot = 0;
        int maxent = 0;
        for (int b : lv) {
            HBlock& B = S.bl[b];
            if (B.type != HB_DENSE) continue;
            const HCluster &T = S.cl[B.tau], &Sg = S.cl[B.sig];
            LeafDesc L;
            L.ra = T.r0;
            L.ca = Sg.r0;
            L.m = (int)B.m;
            L.nc = (int)B.n;
            L.i0 = T.e0;
            L.ni = std::min(T.e1 + 1, N) - T.e0;
            L.j0 = Sg.e0;
            L.nj = std::min(Sg.e1 + 1, N) - Sg.e0;
            L.ktab = kslot;
            L.out = B.off;
            kslot += (int64_t)L.ni * L.nj;
            maxent = std::max(maxent, L.m * L.nc);
            ld.push_back(L);
        }
        if (!ld.empty() && partition) {
            // paper partition: leaves in the paper order, gathered from the internal-order A
            std::vector<LeafTile> lt;
            for (auto& L : ld)
                for (int c0 = 0; c0 < L.nc; c0 += 32)
                    for (int r0 = 0; r0 < L.m; r0 += 32)
                        lt.push_back(LeafTile{L.ra + r0, L.ca + c0, L.out + (int64_t)c0 * L.m + r0, L.m,
                                              std::min(32, L.m - r0), std::min(32, L.nc - c0)});
            DBuf<LeafTile> dlt;
            dlt.upload(lt.data(), lt.size(), h->stream);
            for (size_t base = 0; base < lt.size(); base += 65535u * 8) {
                const unsigned cnt = (unsigned)std::min<size_t>(65535u * 8, lt.size() - base);
                k_leaf_from_dense_paper<<<cnt, dim3(32, 8), 0, h->stream>>>(dlt.p + base, op->A.p, op->lda, hm->dense.p,
                                                                            N, P);
                FDE_CHECK_LAUNCH();
            }
        } else if (!ld.empty() && from_band) {
            // the assembly's pair-moment band (all pairs j <= i, world 1) is complete:
            // the leaves are expanded from it while A's expansion still runs
            DBuf<LeafDesc> dld;
            dld.upload(ld.data(), ld.size(), h->stream);
            asm_expand_leaves_band(h, op, dld.p, (int)ld.size(), maxent, hm->dense.p);
        } else if (!ld.empty() && !recompute && op->A.p && op->r0 == 0 && op->r1 == op->n) {
            // the dense operator is resident with all rows: the exact entries of the
            // inadmissible leaves are its sub-blocks -- one batched
            // transposing copy (row-major A -> column-major leaves) instead of
            // recomputing their pair moments
            std::vector<LeafTile> lt;
            for (auto& L : ld)
                for (int c0 = 0; c0 < L.nc; c0 += 32)
                    for (int r0 = 0; r0 < L.m; r0 += 32)
                        lt.push_back(LeafTile{L.ra + r0, L.ca + c0, L.out + (int64_t)c0 * L.m + r0, L.m,
                                              std::min(32, L.m - r0), std::min(32, L.nc - c0)});
            DBuf<LeafTile> dlt;
            dlt.upload(lt.data(), lt.size(), h->stream);
            for (size_t base = 0; base < lt.size(); base += 65535u * 8) {
                const unsigned cnt = (unsigned)std::min<size_t>(65535u * 8, lt.size() - base);
                k_leaf_from_dense<<<cnt, dim3(32, 8), 0, h->stream>>>(dlt.p + base, op->A.p, op->lda, hm->dense.p);
                FDE_CHECK_LAUNCH();
            }
        } else if (!ld.empty()) {
            // element pairs of the dense leaves (only needed when they are recomputed)
            for (const LeafDesc& L : ld)
                for (int a = 0; a < L.ni; ++a)
                    for (int c = 0; c < L.nj; ++c) {
                        const int i = L.i0 + a, j = L.j0 + c;
                        li.push_back(std::max(i, j));
                        lj.push_back(std::min(i, j));
                        ls.push_back(L.ktab + (int64_t)a * L.nj + c);
                    }
            DBuf<int> di, dj;
            DBuf<long long> dsl;
            DBuf<double> ktab;
            DBuf<LeafDesc> dld;
            di.upload(li.data(), li.size(), h->stream);
            dj.upload(lj.data(), lj.size(), h->stream);
            dsl.upload(ls.data(), ls.size(), h->stream);
            ktab.alloc((size_t)kslot * P * P);
            asm_k_list(h, op, di.p, dj.p, dsl.p, (int64_t)li.size(), ktab.p);
            dld.upload(ld.data(), ld.size(), h->stream);
            asm_expand_leaves(h, op, ktab.p, dld.p, (int)ld.size(), maxent, hm->dense.p);
        }
        tick("leaves");
        hm->rank.upload(rank_h.data(), rank_h.size(), h->stream);
        hm->tm.stop(h->stream);
        tick("end");
    } catch (...) {
        delete hm;
        throw;
    }
    return hm;
}

void hm_to_dense_internal(fde_ctx* h, fde_hm* hm, double* out, int64_t ldo)
{
    std::vector<int> lv;
    hm_leaves(hm->S, hm->S.root, lv);
    std::vector<DenseDesc> dd;
    for (int b : lv) {
        const HBlock& B = hm->S.bl[b];
        DenseDesc d;
        d.type = B.type;
        d.r0 = hm->S.cl[B.tau].r0;
        d.c0 = hm->S.cl[B.sig].r0;
        d.m = (int)B.m;
        d.n = (int)B.n;
        d.off = B.off;
        d.kcap = B.kcap;
        d.blk = b;
        dd.push_back(d);
    }
    DBuf<DenseDesc> ddd;
    ddd.upload(dd.data(), dd.size(), h->stream);
    for (size_t base = 0; base < dd.size(); base += 65535) {
        unsigned cnt = (unsigned)std::min<size_t>(65535, dd.size() - base);
        k_blocks_to_dense<<<dim3(64, cnt), 256, 0, h->stream>>>(ddd.p + base, hm->dense.p, hm->lr.p, hm->rank.p, out,
                                                               ldo);
        FDE_CHECK_LAUNCH();
    }
    FDE_CUDA(cudaStreamSynchronize(h->stream));
}
