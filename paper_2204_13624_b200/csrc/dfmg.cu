// Doubly-fine material grid (DFMG) -- placeholder until the DFMG kernels land.
#include "context.hpp"

extern "C" {

int combo_dfmg_stress(combo_ctx* c, const double*, double*, combo_sweep_stats*, int) {
  if (c) c->err = "dfmg: not implemented yet";
  return COMBO_ERR_STATE;
}

int combo_dfmg_tangent_matvec(combo_ctx* c, const double*, const double*, double*, int) {
  if (c) c->err = "dfmg: not implemented yet";
  return COMBO_ERR_STATE;
}

int combo_dfmg_get_warm_starts(combo_ctx* c, double*, int) {
  if (c) c->err = "dfmg: not implemented yet";
  return COMBO_ERR_STATE;
}

}  // extern "C"
