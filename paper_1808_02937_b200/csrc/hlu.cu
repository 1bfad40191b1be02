// H-LU (placeholder until the formatted factorisation lands)
#include "hlu.h"

struct fde_lu {
    fde_op* op = nullptr;
};

fde_lu* hlu_build(fde_ctx*, fde_hm*, double) { fde_fail(FDE_EINVAL_PARAM, "hlu_factor: not built yet"); return nullptr; }
void hlu_info(fde_lu*, fde_hlu_info* info) { memset(info, 0, sizeof(*info)); }
fde_op* hlu_operator(fde_lu* lu) { return lu->op; }
void hlu_destroy(fde_lu* lu) { delete lu; }
void precond_apply_internal(fde_ctx*, fde_lu*, const double*, int64_t, double*, int64_t, int)
{
    fde_fail(FDE_EINVAL_PARAM, "precond_apply: not built yet");
}
