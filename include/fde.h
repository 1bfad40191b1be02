/*
 * fde.h -- C-ABI of the B200-native hot path of arXiv 1808.02937
 * ("H-matrix preconditioned SEM solver for the 1-D two-sided Riemann-Liouville
 * fractional diffusion equation").  Library: paper_1808_02937_b200/libfde.so.
 *
 * Problem (Eq. (Model)):
 *   -D^2( theta aI_x^{2-alpha} u + (1-theta) xI_b^{2-alpha} u ) + rho u = f on (a,b),
 *   u(a) = c1, u(b) = c2,  1 < alpha < 2, 0 <= theta <= 1, rho >= 0.
 * Discretisation: spectral elements on the partition
 * a = x_0 < ... < x_N = b with N-1 nodal hats and P-1 modal functions
 * psi_p = L_{p-1} - L_{p+1} per element; n = N*P - 1 unknowns.
 *
 * Conventions shared by every entry point
 *  - Vectors at this boundary are in the paper's X ordering:
 *      [u^1_1..u^{P-1}_1; ...; u^1_N..u^{P-1}_N; u~_1..u~_{N-1}].
 *    Multi-RHS blocks are column-major with leading dimension `ld` (>= n).
 *  - Vector pointers are DEVICE pointers owned by the caller (e.g. torch
 *    tensors); the library never frees them.  Host pointers are marked (host).
 *  - Every call is ordered on the handle's CUDA stream; nothing synchronises
 *    the host except solve (returns after convergence), hlu_factor (returns
 *    once the factorisation has finished, so that a zero pivot or a rank
 *    overflow is its return value) and calls that return host data.
 *  - Opaque objects are created by the library and released with the
 *    matching fde_free_* call.  Mesh nodes are copied.  Lifetimes: an
 *    fde_hmatrix keeps a pointer to the fde_operator it was built from, and an
 *    fde_hlu to that operator too (precond_apply / solve read its sizes and
 *    work vectors): free an operator only after every H-matrix and H-LU built
 *    from it.  All objects must be used with the handle that created them.
 *  - Return value: FDE_OK (0) or a negative FDE_E* code; fde_last_error()
 *    gives the message.  No entry point falls back to the CPU: without a
 *    usable CUDA device fde_create returns FDE_ECUDA.
 */
#ifndef FDE_H
#define FDE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ error codes */
enum {
    FDE_OK = 0,
    FDE_EINVAL_DOMAIN = -1,      /* a >= b, or a / b not finite                      */
    FDE_EINVAL_SIZE = -2,        /* N < 1, nrhs < 1, ld < n                          */
    FDE_EINVAL_PARAM = -3,       /* alpha not in (1,2), theta not in [0,1], rho < 0,
                                    R < 1, lambda <= 0, n_min < 1, tol < 0           */
    FDE_EINVAL_MESH = -4,        /* nodes not strictly increasing / ends != a,b      */
    FDE_EDEGREE = -5,            /* P < 1 or P > FDE_MAX_P                           */
    FDE_EUNSUPPORTED_MESH = -6,  /* Toeplitz path requested on a non-uniform mesh    */
    FDE_EDIM = -7,               /* objects of different problems mixed              */
    FDE_ESINGULAR_PIVOT = -8,    /* zero/NaN pivot in an H-LU leaf                   */
    FDE_EBREAKDOWN = -9,         /* Krylov breakdown, or non-finite right-hand side  */
    FDE_EMAXITER = -10,          /* Krylov did not converge within maxiter           */
    FDE_ECUDA = -11,
    FDE_ENCCL = -12,
    FDE_ENOMEM = -13,
    FDE_ERANK = -14              /* a low-rank block exceeded its rank capacity      */
};

#define FDE_MAX_P 32

/* ------------------------------------------------------------- problem */
typedef struct {
    double a, b;          /* interval                       */
    double alpha;         /* 1 < alpha < 2                                 */
    double theta;         /* 0 <= theta <= 1                               */
    double rho;           /* reaction coefficient >= 0                     */
    double c1, c2;        /* Dirichlet data u(a)=c1, u(b)=c2               */
} fde_problem;

enum { FDE_MESH_CUSTOM = 0, FDE_MESH_UNIFORM = 1 };

typedef struct {
    int32_t N;              /* elements                                      */
    const double* nodes;    /* (host) N+1 strictly increasing, [0]=a, [N]=b  */
    int32_t P;              /* uniform polynomial degree, 1 <= P <= FDE_MAX_P */
    int32_t kind;           /* FDE_MESH_*; UNIFORM is verified, not trusted  */
} fde_mesh;

/* Forcing f(x) = sum_k leg[k] L_k(2(x-a)/(b-a)-1)
 *             + sum_t coef[t] (x-a)^power[t]  (side[t]==0)
 *             + sum_t coef[t] (b-x)^power[t]  (side[t]==1).   All host arrays. */
typedef struct {
    int32_t nleg;  const double* leg;
    int32_t nterm; const int32_t* side; const double* power; const double* coef;
} fde_forcing;

typedef struct fde_ctx* fde_handle;
typedef struct fde_op* fde_operator;
typedef struct fde_hm* fde_hmatrix;
typedef struct fde_lu* fde_hlu;

/* ------------------------------------------------------------- context */
/* device: CUDA ordinal; cuda_stream: cudaStream_t to order work on (NULL =
 * the legacy default stream, as in the CUDA runtime); nccl_unique_id: 128-byte ncclUniqueId shared by all
 * ranks (NULL => world must be 1); rank/world: this process in the job. */
int fde_create(fde_handle* out, int device, void* cuda_stream, const void* nccl_unique_id,
               int rank, int world);
void fde_destroy(fde_handle h);
/* Test / diagnostics: a handle that BEHAVES as rank `rank` of `world` ranks
 * without a communicator, so one process on one GPU can run each rank's local
 * work of the row-sharded path (sharded assembly, the near-field recompute of
 * hmatrix_build, fde_shard_matvec, the all-gather compaction through
 * fde_debug_compact_gather).  Calls that need the collective (the dense
 * stiffness_matvec and solve at world > 1) fail with FDE_ENCCL. */
int fde_create_virtual_rank(fde_handle* out, int device, void* cuda_stream, int rank, int world);
const char* fde_last_error(fde_handle h);
int fde_sync(fde_handle h);                   /* cudaStreamSynchronize(stream)    */
int fde_nccl_unique_id(void* out128);          /* ncclGetUniqueId, for rank 0     */

/* Live kernel timing with CUDA events recorded on the handle's stream around
 * the dense GEMV launches (class 0), the Toeplitz FFT matvec (class 1) and the
 * preconditioner application (class 2).  fde_profile_collect synchronises the
 * stream and writes, per class c, out9[3c] = launches, out9[3c+1] = total ms,
 * out9[3c+2] = algorithmic bytes (GEMV: 8 * rows * n per 4-RHS pass + vectors). */
int fde_profile(fde_handle h, int enable);
int fde_profile_collect(fde_handle h, double* out9, int reset);
/* Number of kernels this library has launched in the process so far. */
long long fde_launch_count(void);
/* Diagnostics: H-LU truncation statistics since load: out4 = {calls, sum of
 * compacted widths, sum of Jacobi sweeps, max width}; counted only when the
 * process runs with FDE_TRUNC_STATS=1 (no atomics on the hot path otherwise). */
int fde_debug_trunc_stats(unsigned long long* out4);
/* Diagnostics (FDE_TRUNC_STATS=1): out32[0..3] as above; out32[4 + i] = SM
 * cycles of phase i of the truncation core k_bcore summed over its CTAs (0 column
 * mask, 1 Gram reduction, 2 index / zeroing, 3 scaling, 4 pivoted Cholesky,
 * 5 core product, 6 Jacobi, 7 ordering, 8 output); out32[16..19] = sum / max of
 * the nonzero width and of the chunk count per entry; out32[20] = max cycles of
 * one CTA.  The rest is zero. */
int fde_debug_trunc_profile(unsigned long long* out32);
/* Test entry: the H-LU's batched formatted truncation (the
 * "prescribed tolerance" Tol_HLU of the H-LU, Boerm's truncation of a low-rank sum
 * to the singular values sigma_i > tol * sigma_1) applied to nb independent sums
 * U_q V_q^T, q < nb.  U: device, nb consecutive column-major m x k blocks; V: nb
 * n x k blocks; Uo / Vo: device outputs, nb m x kc / n x kc blocks (columns >= the
 * kept rank are zero; Uo_q Vo_q^T is the truncated sum).  1 <= k, kc <= 64,
 * tol > 0.  *overflow = 1 when some sum kept more than kc singular values (then
 * the first kc are kept).  Runs on the handle's stream and synchronises it.
 * Errors: FDE_EINVAL_SIZE, FDE_EINVAL_PARAM, FDE_ECUDA. */
int fde_debug_truncate(fde_handle h, const double* U, const double* V, int64_t m, int64_t n, int k, int nb, double tol,
                       int kc, double* Uo, double* Vo, int* overflow);
/* Diagnostics: H-LU algorithm selection for later hlu_factor calls (process
 * wide).  mode 0 (default): the leaf-ordered batched factorisation whenever the
 * partition allows it (leaves <= 128 dofs), else the recursive one; mode 1: the
 * recursive formatted H-LU only; mode 2 + s: leaf-ordered, stopped after s leaf
 * steps (test helper: fde_hlu_dense_internal then shows the partial state; the
 * factor is not usable for precond_apply).  Both compute the H-LU of
 * PAPER.md:598-606; FDE_EINVAL_PARAM for negative modes. */
int fde_debug_hlu_mode(int mode);
/* Diagnostics: reserved / used bytes of the device's default stream-ordered
 * memory pool (every library buffer comes from it). */
int fde_debug_pool_bytes(int device, unsigned long long* reserved, unsigned long long* used);

/* Row-block sharding of the dense operator over `world` GPUs (host function,
 * usable without a device): rank owns internal rows [*r0, *r1) = the dofs of
 * elements [N*rank/world, N*(rank+1)/world); *rows_max = largest shard (the
 * all-gather pads every shard to it). */
int fde_shard_rows(int N, int P, int world, int rank, int64_t* r0, int64_t* r1, int64_t* rows_max);

/* --------------------------------------------------------- sem_assemble */
enum { FDE_OP_DENSE = 1, FDE_OP_TOEPLITZ = 2 };

/* Builds the operator A = rho M + theta S_l + (1-theta) S_l^T of Eq. (lsys)
 * on the device.  FDE_OP_DENSE stores this rank's row shard
 * of the dense fp64 matrix (element-interleaved internal order, row-major);
 * FDE_OP_TOEPLITZ stores the P x P block-Toeplitz lag symbols and their
 * 2N-point circulant spectra: on uniform meshes, and on
 * single-ratio geometric meshes (h_{e+1} = q h_e for every element to 1e-10,
 * PAPER.md:632-735; there K_ij = (h_j/h_0)^{1-alpha} K_{i-j,0}, two spectral
 * passes); any other mesh fails with FDE_EUNSUPPORTED_MESH.  Both may be
 * requested together.  Entries are computed by Gauss quadrature of the pair
 * moments K_ij[m][n] = gamma0 int int L_m L_n (t-s)_+^{1-alpha} with
 * Gauss-Jacobi / Duffy treatment of the diagonal and touching pairs and graded
 * composite rules on near pairs. */
int sem_assemble(fde_handle h, const fde_problem* prob, const fde_mesh* mesh, int flags,
                 fde_operator* out);

typedef struct {
    int64_t n;            /* unknowns NP-1                                      */
    int32_t N, P;
    int64_t row_begin, row_end;   /* this rank's rows (internal order)          */
    int64_t lda;          /* leading dimension of the dense shard               */
    int32_t flags;
    int32_t uniform;      /* mesh verified uniform                               */
    double assemble_ms;   /* device time of the assembly; -1 while it still runs */
} fde_operator_info;
/* sem_assemble and hmatrix_build return as soon as their device work is
 * enqueued on the handle's stream (results are stream-ordered: later calls and
 * stream work see them complete); get_info never waits, *_wait blocks until the
 * object's device work is done (then the timing fields are final). */
int fde_operator_get_info(fde_operator op, fde_operator_info* info);
int fde_operator_wait(fde_operator op);

/* Copy the dense operator rows [r0,r1) x all columns, PAPER order, into the
 * device buffer out (row-major, ldo >= n).  World==1 only (test helper). */
int fde_operator_dense_paper(fde_handle h, fde_operator op, double* out, int64_t ldo);
/* Columns of the boundary hats (node 0, node N) of the full operator, length n
 * each, paper order, into device buffer out[2*n] (used for the lifting). */
int fde_operator_boundary_columns(fde_handle h, fde_operator op, double* out);
/* This rank's dense rows [row_begin, row_end) x n in the INTERNAL
 * element-interleaved order (fde_hlu_dense_internal's convention), row-major
 * into device buffer out with ldo >= n; any world (test helper). */
int fde_operator_rows_internal(fde_handle h, fde_operator op, double* out, int64_t ldo);

/* -------------------------------------------------------------- sem_rhs */
/* G[:, r] = (f_r, phi_I) - A[:, {0,N}] [c1, c2]  (lifting
 * by the boundary hats).  f: host array of nrhs forcings; G device, paper
 * order, column-major ld. */
int sem_rhs(fde_handle h, fde_operator op, const fde_forcing* f, int nrhs, double* G, int64_t ld);

/* ----------------------------------------------------- stiffness_matvec */
enum { FDE_PATH_AUTO = 0, FDE_PATH_DENSE = 1, FDE_PATH_TOEPLITZ = 2 };
/* y = A x for nrhs columns (PAPER.md:629 dense O(N_d^2); PAPER.md:632-735 FFT on
 * uniform meshes).  x, y device, paper order, full length n on every rank;
 * with world > 1 the dense path multiplies the local row shard and all-gathers
 * y over NCCL. */
int stiffness_matvec(fde_handle h, fde_operator op, const double* x, double* y, int nrhs,
                     int64_t ld, int path);
/* The local half of the sharded dense matvec: y_loc = A[r0:r1, :] x for this
 * rank's rows only (no all-gather).  x device, paper order, ld ldx >= n; y_loc
 * device, internal order, rows r0..r1 of column c at y_loc + c * ldy,
 * ldy >= the largest shard (fde_shard_rows' rows_max). */
int fde_shard_matvec(fde_handle h, fde_operator op, const double* x, int64_t ldx, double* y_loc, int64_t ldy,
                     int nrhs);
/* The step after ncclAllGather in the sharded matvec, on a caller-supplied
 * buffer in the all-gather layout: gathered[(g * nrhs + c) * rows_max + r] =
 * row r0(g) + r of column c from rank g.  Writes y (device, paper order, ld). */
int fde_debug_compact_gather(fde_handle h, fde_operator op, const double* gathered, double* y, int64_t ld,
                             int nrhs);
/* Test entry: the sharded matvec's communication path on one GPU.  On a world-1
 * handle, creates a one-rank NCCL communicator (libnccl.so.2 resolved with
 * dlopen, ncclGetUniqueId, ncclCommInitRank), computes the local rows of A x
 * (x: nrhs paper-order columns, stride ld), passes them through ncclAllGather and
 * the post-all-gather compaction exactly as every Krylov iteration of a world > 1
 * run does, writes y (paper order, stride ld) and destroys the communicator.
 * Synchronises the handle's stream.  Errors: FDE_EINVAL_PARAM (world != 1, a
 * handle that already has a communicator, or no dense form), FDE_EINVAL_SIZE,
 * FDE_ENCCL (library or call failure), FDE_ECUDA. */
int fde_debug_comm_selftest(fde_handle h, fde_operator op, const double* x, double* y, int64_t ld, int nrhs);

/* -------------------------------------------------------- hmatrix_build */
/* H-matrix H ~ S_l on the element-cluster block tree with admissibility
 * max(diam) <= lambda dist (Eq. (admis)), Taylor factors of rank
 * R (Lemma 3.2; Q,W, Qbar, Wbar of PAPER.md:365-388) on
 * admissible leaves, exact entries on inadmissible leaves,
 * and the preconditioner operator A~ = rho M + theta H + (1-theta) H^T
 * (Eq. (approxsys), reading A2).  Replicated on every rank. */
int hmatrix_build(fde_handle h, fde_operator op, int R, double lambda, int n_min, fde_hmatrix* out);

/* The same with a choice of cluster partition:
 *  FDE_PARTITION_INTERLEAVED (the default of hmatrix_build, reading A9):
 *    one binary tree over element ranges, a cluster holding the modal functions
 *    of its elements and the hats of their right nodes;
 *  FDE_PARTITION_PAPER (Fig. fig200, Eq. (approxmat)): separate
 *    trees for the modal functions (clusters of elements, support = their union)
 *    and the nodal hats (clusters of interior nodes, support = union of
 *    [x_{j-1}, x_{j+1}]), under a root whose first block level is the 2 x 2
 *    superblock [B F; E C] of S_l; the H-matrix, its H-LU and precond_apply then
 *    work in the paper's dof order internally.  Needs the resident dense
 *    operator (world 1, FDE_OP_DENSE): FDE_EINVAL_PARAM otherwise. */
enum { FDE_PARTITION_INTERLEAVED = 0, FDE_PARTITION_PAPER = 1 };
int hmatrix_build_partition(fde_handle h, fde_operator op, int R, double lambda, int n_min, int partition,
                            fde_hmatrix* out);

typedef struct {
    int32_t nblocks_dense, nblocks_lr, depth, nclusters;
    int64_t dense_entries, lr_entries;   /* stored fp64 words              */
    double build_ms;      /* device time of the build; -1 while it still runs    */
} fde_hmatrix_info;
int fde_hmatrix_get_info(fde_hmatrix hm, fde_hmatrix_info* info);
int fde_hmatrix_wait(fde_hmatrix hm);
/* Expand A~ into a dense n x n matrix, paper order, column-major with ldo >= n,
 * device buffer (test / diagnostics helper; O(n^2) memory). */
int fde_hmatrix_dense_paper(fde_handle h, fde_hmatrix hm, double* out, int64_t ldo);

/* ----------------------------------------------------------- hlu_factor */
/* A~ ~= L_H U_H, L_H unit lower, both in H format on the same block tree
 * (Fig. fig:HLU); formatted arithmetic with per-block
 * truncation sigma_i <= tol sigma_1 (reading A12); tol = 0 keeps every rank
 * (exact up to rounding; rank capacity permitting).  No pivoting
 * (coercivity, Theorem 2.1).  Does not modify hm.  Returns after the device
 * work: FDE_ESINGULAR_PIVOT for a zero / non-finite pivot of a diagonal tile,
 * FDE_ERANK when a truncated rank exceeds the block capacity (the host-side
 * planning overlaps the device work queued before the call). */
int hlu_factor(fde_handle h, fde_hmatrix hm, double tol, fde_hlu* out);

typedef struct {
    int32_t max_rank;
    int64_t stored_entries;
    double factor_ms;
    int32_t nops;          /* device operations issued                      */
    int32_t algorithm;     /* 0 recursive formatted H-LU, 1 leaf-ordered    */
    double plan_ms;        /* host time of the leaf-ordered schedule (ms)   */
} fde_hlu_info;
int fde_hlu_get_info(fde_hlu lu, fde_hlu_info* info);

/* Test helper: the packed factors (strict lower part L_H, upper part U_H) as a
 * dense n x n column-major device matrix in the INTERNAL element-interleaved
 * order (dof r: element r/P; r%P < P-1 modal psi_{r%P+1}, r%P = P-1 hat of
 * node r/P+1). */
int fde_hlu_dense_internal(fde_handle h, fde_hlu lu, double* out, int64_t ldo);

/* -------------------------------------------------------- precond_apply */
/* z = U_H^{-1} L_H^{-1} r: hierarchical forward and backward substitution
 * (PAPER.md:605).  r, z device, paper order; r may equal z. */
int precond_apply(fde_handle h, fde_hlu lu, const double* r, double* z, int nrhs, int64_t ld);

/* ---------------------------------------------------------------- solve */
enum { FDE_GMRES = 0, FDE_BICGSTAB = 1 };
typedef struct {
    int32_t method;       /* FDE_GMRES (BASELINE) | FDE_BICGSTAB */
    double tol;           /* relative residual of the preconditioned system     */
    int32_t maxiter;      /* total iterations                                    */
    int32_t restart;      /* GMRES(m)                                            */
    int32_t path;         /* FDE_PATH_* for the matvec                           */
    int32_t verify;       /* GMRES: 1 = at convergence recompute the true
                             preconditioned residual ||A~^{-1}(G - A X)|| and restart
                             the columns still above tol (one more matvec + apply);
                             0 = trust the Givens estimate                         */
} fde_solve_opts;

typedef struct {
    int32_t iterations;   /* max over RHS                                       */
    int32_t matvecs;      /* operator applications per RHS column               */
    int32_t converged;    /* number of converged RHS columns                    */
    double relres;        /* max final preconditioned relative residual          */
    double solve_ms;
    double relres_true;   /* max recomputed ||A~^{-1}(G-AX)||/||A~^{-1}G|| (verify=1), else -1 */
} fde_solve_report;

/* Solve A~^{-1} A X = A~^{-1} G (Eq. (precondsys)) from
 * X0 = 0; lu may be NULL (unpreconditioned).  G, X device, paper order. */
int solve(fde_handle h, fde_operator op, fde_hlu lu, const double* G, double* X, int nrhs,
          int64_t ld, const fde_solve_opts* opts, fde_solve_report* rep);
/* same entry point under a prefixed name */
int fde_solve(fde_handle h, fde_operator op, fde_hlu lu, const double* G, double* X, int nrhs,
              int64_t ld, const fde_solve_opts* opts, fde_solve_report* rep);

/* ------------------------------------------------------------- cleanup */
void fde_free_operator(fde_operator op);
void fde_free_hmatrix(fde_hmatrix hm);
void fde_free_hlu(fde_hlu lu);

#ifdef __cplusplus
}
#endif
#endif /* FDE_H */
