// V(nu1,nu2) cycle composition -- see hhg.h.
#include "hhg_internal.h"

using namespace hhg;

extern "C" hhg_status hhg_vcycle(hhg_ctx ctx, int L, int nu1, int nu2, int L_coarse, int coarse_cg_iters,
                                 hhg_op op, double* u, const double* f, int n_cycles, double* res_hist) {
  Ctx* c = (Ctx*)ctx;
  (void)L; (void)nu1; (void)nu2; (void)L_coarse; (void)coarse_cg_iters; (void)op; (void)u; (void)f;
  (void)n_cycles; (void)res_hist;
  return set_err(c, HHG_ERR_STATE, "hhg_vcycle: not implemented yet");
}
