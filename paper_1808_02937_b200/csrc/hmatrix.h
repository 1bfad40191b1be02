// H-matrix structures shared by hmatrix.cu and hlu.cu.
#pragma once

#include "fde_internal.h"

enum { HB_DENSE = 0, HB_LR = 1, HB_HIER = 2 };

// Cluster kinds: the element-interleaved tree (reading A9: a cluster holds the
// modal dofs of its elements and the hats of their right nodes, dofs in the
// internal order), or the paper's partition (Fig. fig200):
// separate modal and nodal trees under a virtual root, dofs in the paper order.
enum { HC_INTERLEAVED = 0, HC_MODAL = 1, HC_NODAL = 2, HC_ROOT = 3 };

struct HCluster {
    int e0, e1;          // element range [e0, e1) (interleaved / modal), interior node range [j0, j1) (nodal)
    int64_t r0, r1;      // dof range (the H-matrix's order: internal, or paper for the paper partition)
    int child[2];        // -1 for leaves
    double lo, hi;       // support
    int nlo = 0, nhi = 0;   // node indices of the support ends (expansion points: x_nlo + (x_nhi - x_nlo)/2)
    int kind = HC_INTERLEAVED;
};

struct HBlock {
    int tau, sig;        // row / column cluster
    int type;
    int child[4];        // hier: (t0,s0) (t0,s1) (t1,s0) (t1,s1)
    int64_t m, n;        // rows, cols
    int64_t off;         // dense: offset of the m x n col-major block (ld = m)
                         // lr: offset of U (m x kcap col-major), V follows (n x kcap)
    int kcap;            // rank capacity (lr)
    int lower;           // lr: tau right of sigma
};

struct HStruct {
    int N = 0, P = 0;
    int64_t n = 0;
    int paper = 0;           // 1: the paper's modal / nodal partition, dofs in the paper order
    std::vector<HCluster> cl;
    std::vector<HBlock> bl;
    int root = 0;
    int depth = 0;
};

struct fde_hm {
    LazyTimer tm;        // device time of the build (read lazily)
    fde_op* op = nullptr;
    int R = 0;
    double lam = 1.0;
    int n_min = 16;
    HStruct S;
    DBuf<double> dense;      // dense leaf arena
    DBuf<double> lr;         // low-rank arena (kcap = R)
    DBuf<int> rank;          // per block (device), R for LR blocks of A~
    int64_t dense_words = 0, lr_words = 0;
    int n_dense = 0, n_lr = 0;
    double build_ms = 0;
    cudaStream_t st = nullptr;   // stream the build was enqueued on (the handle's build stream)
};

struct LeafDesc {
    int64_t ra, ca;    // first row / column dof
    int m, nc;
    int i0, ni, j0, nj;
    int64_t ktab;      // first K block of the leaf table
    int64_t out;       // dense arena offset
};

void hm_leaves(const HStruct& S, int b, std::vector<int>& out);
// exact entries of the dense leaves from their K tables (assemble.cu)
void asm_expand_leaves_band(fde_ctx* h, fde_op* op, const LeafDesc* d, int nleaves, int maxentries, double* arena);
void asm_expand_leaves(fde_ctx* h, fde_op* op, const double* Ktab, const LeafDesc* d, int nleaves, int maxentries,
                       double* arena);

// build the cluster tree and block partition (host, structure only)
void hstruct_build(HStruct& S, const std::vector<double>& nodes, int P, int n_min, double lam, int partition = 0);

// recompute: build the inadmissible leaves from pair moments even when the dense
// operator is resident (the build then does not wait for the dense assembly)
fde_hm* hm_build(fde_ctx* h, fde_op* op, int R, double lam, int n_min, bool recompute = false, bool from_band = false,
                 int partition = 0);
void hm_to_dense_internal(fde_ctx* h, fde_hm* hm, double* out, int64_t ldo);   // out col-major n x n
