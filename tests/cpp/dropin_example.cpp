// Drop-in usage of the C++ layer (include/combo_b200.hpp): the reference's
// acceptance criterion 9 (2x1x1 laminate RVE, acceptance.cpp:407-434) written
// against combo::b200. Built by tests/test_capi.py (compile + link) and run by
// tests/test_gpu_dropin.py on the GPU.
#include <cmath>
#include <cstdio>

#include "combo_b200.hpp"

int main() {
  using namespace combo::b200;
  Device dev(0);
  PhaseImage img;
  img.dims = {2, 1, 1};
  img.lengths = {1, 1, 1};
  img.data = {1, 0};
  ComboGrid g = coarsen(dev, img, {1, 1, 1});
  g.normal = {1, 0, 0, 1, 0, 0};
  CellMaterials cm(dev, g, neo_hookean_enu(1.0, 0.0), neo_hookean_enu(10.0, 0.3), true);
  SolverConfig cfg;
  cfg.green = GreenKind::rotated;
  cfg.tol_equilibrium = 1e-12;
  const Mat3 fbar = {1, 0.5, 0, 0, 1, 0, 0, 0, 1};
  const SolveResult r = solve(cm, fbar, cfg);
  std::printf("{\"success\": %s, \"pbar\": [%.17g, %.17g, %.17g, %.17g], \"steps\": %zu, \"ls\": %lld}\n",
              r.report.success ? "true" : "false", r.pbar[0], r.pbar[1], r.pbar[3], r.pbar[4],
              r.report.steps.size(), (long long)r.report.ls_iterations);
  // all-pure grid (factors 1): no laminate states to recover
  if (!recover_composites(r.f, cm).empty()) return 3;
  try {
    SolverConfig bad = cfg;
    bad.eval = MaterialEval::dfmg;  // requires staggered (solver.cpp:277-280)
    solve(cm, fbar, bad);
    return 2;
  } catch (const ConfigInvalid&) {
  }
  return r.report.success ? 0 : 1;
}
