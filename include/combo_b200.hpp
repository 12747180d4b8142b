// combo_b200.hpp -- C++17 layer over the C-ABI (combo_cuda.h) with the
// reference library's names and semantics (namespace combo::b200):
//
//   CellMaterials(grid, matrix, inclusion, combo, lam)  cell_material.hpp:22-23
//   SweepStats stress_sweep(cm, F, P)                    cell_material.hpp:90-92
//   GreenOperator(kind, grid).project(in, out)           green.hpp:30-40
//   ComboGrid coarsen(img, factors)                      combo_grid.hpp:62-63
//   NormalStats compute_normals(img, grid, method, opt)  normals.hpp:55-57
//   SolveResult solve(cm, fbar, cfg)                     solver.hpp:68-69
//   PhaseAverages phase_averages(f, cm)                  postprocess.hpp:20-35
//
// Differences from the reference API, all forced by the boundary:
//   * plain std::array / std::vector instead of Eigen types;
//   * exceptions carry the reference type names (ConfigInvalid, ...) and are
//     thrown from the C status codes; LoadPathFailed stays in the report
//     (solver.cpp:332-336);
//   * fields stay on the device between calls of one solve; host Field9
//     copies happen only at entry and exit.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "combo_cuda.h"

namespace combo {
namespace b200 {

using Mat3 = std::array<double, 9>;  // row major (tensor.hpp:14-16)
using Vec3 = std::array<double, 3>;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct ConfigInvalid : Error { using Error::Error; };
struct InadmissibleMacroState : Error { using Error::Error; };
struct SingularMatrix : Error { using Error::Error; };
struct NonDividingFactor : Error { using Error::Error; };
struct BadShapeSpec : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(int rc, const combo_ctx* c) {
  if (rc == COMBO_OK) return;
  const std::string msg = combo_last_error(c);
  switch (rc) {
    case COMBO_ERR_CONFIG_INVALID: throw ConfigInvalid(rc, msg);
    case COMBO_ERR_INADMISSIBLE_MACRO: throw InadmissibleMacroState(rc, msg);
    case COMBO_ERR_SINGULAR: throw SingularMatrix(rc, msg);
    case COMBO_ERR_NON_DIVIDING_FACTOR: throw NonDividingFactor(rc, msg);
    case COMBO_ERR_BAD_SHAPE: throw BadShapeSpec(rc, msg);
    case COMBO_ERR_CUDA:
    case COMBO_ERR_NCCL:
    case COMBO_ERR_OOM: throw DeviceError(rc, msg);
    default: throw Error(rc, msg);
  }
}

/// One device + stream; shared by the objects below.
class Device {
 public:
  explicit Device(int device = 0) {
    combo_ctx* c = nullptr;
    check(combo_ctx_create(device, &c), nullptr);
    ctx_.reset(c, [](combo_ctx* p) { combo_ctx_destroy(p); });
  }
  combo_ctx* get() const { return ctx_.get(); }

 private:
  std::shared_ptr<combo_ctx> ctx_;
};

struct PhaseImage {  // image.hpp:17-44
  std::array<int64_t, 3> dims{0, 0, 0};
  std::array<double, 3> lengths{1.0, 1.0, 1.0};
  std::vector<uint8_t> data;
};

struct ComboGrid {  // combo_grid.hpp:29-59
  std::array<int64_t, 3> dims{0, 0, 0};
  std::array<int64_t, 3> factors{1, 1, 1};
  std::array<double, 3> lengths{1.0, 1.0, 1.0};
  std::vector<uint8_t> kind;  // 0 matrix, 1 inclusion, 2 composite
  std::vector<double> c_plus;
  std::vector<int64_t> count_plus;
  std::vector<double> normal;  // 3 per boxel
  std::vector<uint8_t> normal_flag;
  int64_t boxel_count() const { return dims[0] * dims[1] * dims[2]; }
};

inline ComboGrid coarsen(const Device& d, const PhaseImage& img, const std::array<int64_t, 3>& factors) {
  ComboGrid g;
  g.factors = factors;
  g.lengths = img.lengths;
  for (int a = 0; a < 3; ++a) g.dims[a] = factors[a] > 0 ? img.dims[a] / factors[a] : 0;
  const size_t nb = size_t(g.boxel_count());
  g.kind.resize(nb);
  g.c_plus.resize(nb);
  g.count_plus.resize(nb);
  g.normal.assign(3 * nb, 0.0);
  g.normal_flag.assign(nb, 0);
  check(combo_coarsen(d.get(), img.data.data(), img.dims.data(), factors.data(), g.kind.data(), g.c_plus.data(),
                      g.count_plus.data(), COMBO_MEM_HOST),
        d.get());
  return g;
}

enum class NormalMethod { barycenter = COMBO_NORMAL_BARYCENTER, second_moment = COMBO_NORMAL_SECOND_MOMENT };

struct NormalOptions {  // normals.hpp:33-37
  int centering = COMBO_CENTER_WEIGHTED_CENTROID;
  int min_interface_voxels = 3;
};

inline combo_normal_stats compute_normals(const Device& d, const PhaseImage& img, ComboGrid& g,
                                          NormalMethod m = NormalMethod::second_moment,
                                          const NormalOptions& opt = {}) {
  combo_normal_stats st{};
  check(combo_normals(d.get(), img.data.data(), img.dims.data(), img.lengths.data(), g.factors.data(), g.kind.data(),
                      int(m), opt.centering, opt.min_interface_voxels, g.normal.data(), g.normal_flag.data(), &st,
                      COMBO_MEM_HOST),
        d.get());
  return st;
}

/// NeoHookeanParams (materials.hpp:14-21) set directly by (lambda, mu).
inline combo_law neo_hookean(double lambda, double mu) {
  combo_law l{};
  l.kind = COMBO_LAW_NEO_HOOKEAN;
  l.lambda = lambda;
  l.mu = mu;
  return l;
}
/// NeoHookeanParams::from_enu (materials.cpp:11-20)
inline combo_law neo_hookean_enu(double e, double nu) {
  return neo_hookean(e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), e / (2.0 * (1.0 + nu)));
}

struct LaminateOptions {  // laminate.hpp:72-79
  double tol_abs = 0.0, tol_rel = 1e-10, stress_floor = 0.0;
  int max_iter = 50;
  bool back_projection = true;
  double c_min = 0.0;
  combo_laminate_opts c() const {
    return {tol_abs, tol_rel, stress_floor, max_iter, back_projection ? 1 : 0, c_min};
  }
};

/// Field9 (field.hpp:32-70): component-major, component c = 3i+J.
struct Field9 {
  std::array<int64_t, 3> dims{1, 1, 1};
  std::vector<double> data;
  int64_t cells() const { return dims[0] * dims[1] * dims[2]; }
};

/// CellMaterials bound on the device (cell_material.cpp:12-55).
class CellMaterials {
 public:
  CellMaterials(const Device& d, const ComboGrid& g, const combo_law& matrix, const combo_law& inclusion,
                bool combo = true, const LaminateOptions& lam = {})
      : dev_(d), dims_(g.dims) {
    const combo_laminate_opts o = lam.c();
    check(combo_bind_materials(d.get(), g.dims.data(), g.lengths.data(), g.kind.data(), g.c_plus.data(),
                               g.normal.data(), &matrix, &inclusion, combo ? 1 : 0, &o, COMBO_MEM_HOST),
          d.get());
  }
  int64_t composite_cells() const {
    int64_t n = 0;
    check(combo_composite_cells(dev_.get(), &n), dev_.get());
    return n;
  }
  void reset_warm_starts() { check(combo_reset_warm_starts(dev_.get()), dev_.get()); }
  const Device& device() const { return dev_; }
  const std::array<int64_t, 3>& dims() const { return dims_; }

 private:
  Device dev_;
  std::array<int64_t, 3> dims_;
};

/// stress_sweep (cell_material.cpp:104-168): P(F), warm starts updated.
inline combo_sweep_stats stress_sweep(CellMaterials& cm, const Field9& f, Field9& p) {
  p.dims = f.dims;
  p.data.resize(f.data.size());
  combo_sweep_stats st{};
  check(combo_stress_sweep(cm.device().get(), f.data.data(), p.data.data(), &st, COMBO_MEM_HOST), cm.device().get());
  return st;
}

/// recover_phase_fields + phase_averages (postprocess.cpp:13-106) in one
/// call: composite laminates re-solved at f from the warm starts (read only).
struct PhaseAverages {  // postprocess.hpp:27-35
  Mat3 pbar{}, pbar_plus{}, pbar_minus{};
  bool has_plus = false, has_minus = false;
  double c_plus = 0.0;
  int max_resolve_iterations = 0;
};
inline PhaseAverages phase_averages(const Field9& f, CellMaterials& cm) {
  combo_phase_avg a{};
  check(combo_phase_averages(cm.device().get(), f.data.data(), &a, COMBO_MEM_HOST), cm.device().get());
  PhaseAverages o;
  for (int q = 0; q < 9; ++q) {
    o.pbar[q] = a.pbar[q];
    o.pbar_plus[q] = a.pbar_plus[q];
    o.pbar_minus[q] = a.pbar_minus[q];
  }
  o.has_plus = a.has_plus != 0;
  o.has_minus = a.has_minus != 0;
  o.c_plus = a.c_plus;
  o.max_resolve_iterations = a.max_resolve_iterations;
  return o;
}

/// recover_phase_fields per composite (postprocess.cpp:13-36): the
/// LaminateResult fields interface_tractions() consumes, by composite id.
struct RecoveredComposite {
  int64_t cell = 0;
  Mat3 f_plus{}, f_minus{};
  double traction[3] = {0.0, 0.0, 0.0};
};
inline std::vector<RecoveredComposite> recover_composites(const Field9& f, CellMaterials& cm) {
  int64_t nc = 0;
  check(combo_composite_cells(cm.device().get(), &nc), cm.device().get());
  const size_t n = size_t(nc > 0 ? nc : 1);
  std::vector<int64_t> cell(n);
  std::vector<double> fp(9 * n), fm(9 * n), tr(3 * n);
  check(combo_recover_composites(cm.device().get(), f.data.data(), cell.data(), fp.data(), fm.data(), tr.data(),
                                 COMBO_MEM_HOST),
        cm.device().get());
  std::vector<RecoveredComposite> out(static_cast<size_t>(nc));
  for (size_t q = 0; q < out.size(); ++q) {
    out[q].cell = cell[q];
    for (int c = 0; c < 9; ++c) {
      out[q].f_plus[c] = fp[size_t(c) * n + q];
      out[q].f_minus[c] = fm[size_t(c) * n + q];
    }
    for (int i = 0; i < 3; ++i) out[q].traction[i] = tr[size_t(i) * n + q];
  }
  return out;
}

/// y = A(F) : x with the tangent of the last sweep's states (matrix free;
/// replaces stress_sweep(tangents45) + tangent_matvec, cell_material.cpp:170-194).
inline void tangent_matvec(CellMaterials& cm, const Field9& f, const Field9& x, Field9& y) {
  y.dims = x.dims;
  y.data.resize(x.data.size());
  check(combo_tangent_matvec(cm.device().get(), f.data.data(), x.data.data(), y.data.data(), COMBO_MEM_HOST),
        cm.device().get());
}

enum class GreenKind { continuous = COMBO_GREEN_CONTINUOUS, rotated = COMBO_GREEN_ROTATED,
                       staggered = COMBO_GREEN_STAGGERED };

class GreenOperator {  // green.hpp:30-59
 public:
  GreenOperator(const Device& d, GreenKind kind, const std::array<int64_t, 3>& dims,
                const std::array<double, 3>& lengths)
      : dev_(d), kind_(kind), dims_(dims), lengths_(lengths) {}
  void project(const Field9& in, Field9& out) const {
    check(combo_set_grid(dev_.get(), dims_.data(), lengths_.data()), dev_.get());
    out.dims = in.dims;
    out.data.resize(in.data.size());
    check(combo_project(dev_.get(), int(kind_), in.data.data(), out.data.data(), COMBO_MEM_HOST), dev_.get());
  }

 private:
  Device dev_;
  GreenKind kind_;
  std::array<int64_t, 3> dims_;
  std::array<double, 3> lengths_;
};

enum class Scheme { basic = COMBO_SCHEME_BASIC, newton_cg = COMBO_SCHEME_NEWTON_CG };
enum class MaterialEval { per_cell = COMBO_EVAL_PER_CELL, dfmg = COMBO_EVAL_DFMG };

struct SolverConfig {  // solver.hpp:18-32
  Scheme scheme = Scheme::newton_cg;
  GreenKind green = GreenKind::rotated;
  MaterialEval eval = MaterialEval::per_cell;
  double tol_equilibrium = 1e-8;
  int max_outer = 200;
  double cg_tol = 1e-2;
  int cg_max = 2000;
  int load_steps = 1;
  int max_bisections = 5;
  int threads = 0;
  bool verbose = false;
  combo_solver_cfg c() const {
    return {int(scheme), int(green), int(eval), tol_equilibrium, max_outer, cg_tol, cg_max, load_steps,
            max_bisections, threads, verbose ? 1 : 0, 0};
  }
};

struct StepReport {  // solver.hpp:34-46
  combo_step_info info{};
  std::vector<double> residuals;
  std::vector<int> cg_iters;
  std::vector<Mat3> pbar_history;
};

struct ConvergenceReport {  // solver.hpp:48-55
  std::vector<StepReport> steps;
  bool success = false;
  int bisections = 0;
  double alpha = 0.0, seconds_total = 0.0;
  int64_t ls_iterations = 0;
  std::string json;
};

struct SolveResult {  // solver.hpp:57-62
  Field9 f, p;
  Mat3 pbar{};
  ConvergenceReport report;
};

/// solve (solver.cpp:286-346)
inline SolveResult solve(CellMaterials& cm, const Mat3& fbar, const SolverConfig& cfg, bool want_fields = true) {
  SolveResult out;
  combo_ctx* c = cm.device().get();
  const int64_t n = cm.dims()[0] * cm.dims()[1] * cm.dims()[2];
  if (want_fields) {
    out.f.dims = out.p.dims = cm.dims();
    out.f.data.resize(size_t(9 * n));
    out.p.data.resize(size_t(9 * n));
  }
  const combo_solver_cfg cc = cfg.c();
  combo_report* rep = nullptr;
  check(combo_solve(c, fbar.data(), &cc, want_fields ? out.f.data.data() : nullptr,
                    want_fields ? out.p.data.data() : nullptr, out.pbar.data(), &rep, COMBO_MEM_HOST),
        c);
  std::unique_ptr<combo_report, int (*)(combo_report*)> guard(rep, combo_report_free);
  int success = 0, nsteps = 0;
  check(combo_report_summary(rep, &success, &out.report.bisections, &nsteps, &out.report.alpha,
                             &out.report.seconds_total, &out.report.ls_iterations),
        c);
  out.report.success = success != 0;
  for (int s = 0; s < nsteps; ++s) {
    StepReport sr;
    check(combo_report_step(rep, s, &sr.info), c);
    sr.residuals.resize(size_t(sr.info.n_residuals));
    sr.cg_iters.resize(size_t(sr.info.n_residuals));
    sr.pbar_history.resize(size_t(sr.info.n_residuals));
    if (sr.info.n_residuals > 0)
      check(combo_report_step_history(rep, s, sr.residuals.data(), sr.pbar_history[0].data(), sr.cg_iters.data()),
            c);
    out.report.steps.push_back(std::move(sr));
  }
  out.report.json = combo_report_json(rep);
  return out;
}

}  // namespace b200
}  // namespace combo
