// H-LU factorisation and hierarchical forward/backward substitution.
#pragma once
#include "fde_internal.h"
#include "hmatrix.h"

fde_lu* hlu_build(fde_ctx* h, fde_hm* hm, double tol);
void hlu_info(fde_lu* lu, fde_hlu_info* info);
fde_op* hlu_operator(fde_lu* lu);
void hlu_destroy(fde_lu* lu);
void precond_apply_internal(fde_ctx* h, fde_lu* lu, const double* r, int64_t ldr, double* z, int64_t ldz, int nrhs);
void hlu_dense_internal(fde_ctx* h, fde_lu* L, double* out, int64_t ldo);
void hlu_solve_debug(fde_ctx* h, fde_lu* L, double* X, int64_t ldx, int nrhs, int which);
