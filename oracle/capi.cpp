// TEST INFRASTRUCTURE ONLY (see oracle.hpp): flat C entry points so that
// tests/ (ctypes) and bench.py's cpu_baseline leg can drive the oracle.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "oracle.hpp"

using namespace oracle;

extern "C" {

struct oracle_law {
  int kind;       // 0 neo-hookean, 1 linear
  double lambda;  // neo-hookean
  double mu;
  double c6[36];  // linear: Mandel stiffness
};

struct oracle_lam_opts {
  double tol_abs, tol_rel, stress_floor;
  int max_iter;
  int back_projection;
  double c_min;
};

struct oracle_solver_cfg {
  int scheme, green, eval;
  double tol_equilibrium;
  int max_outer;
  double cg_tol;
  int cg_max, load_steps, max_bisections, threads, verbose;
  long long max_ls_iterations;
};

}  // extern "C"

namespace {
Law to_law(const oracle_law* l) {
  if (l->kind == kLinear) {
    Mat6 c;
    std::memcpy(c.a, l->c6, sizeof(c.a));
    return Law::linear(c);
  }
  return Law::neo_hookean(l->lambda, l->mu);
}
LaminateOptions to_opts(const oracle_lam_opts* o) {
  LaminateOptions r;
  if (!o) return r;
  r.tol_abs = o->tol_abs;
  r.tol_rel = o->tol_rel;
  r.stress_floor = o->stress_floor;
  r.max_iter = o->max_iter;
  r.back_projection = o->back_projection != 0;
  r.c_min = o->c_min;
  return r;
}
PhaseImage make_image(const std::uint8_t* img, const std::int64_t* dims, const double* lengths) {
  PhaseImage p;
  p.dims = {dims[0], dims[1], dims[2]};
  p.lengths = {lengths[0], lengths[1], lengths[2]};
  p.data.assign(img, img + p.size());
  return p;
}
thread_local std::string g_err;

struct CmHandle {
  CellMaterials cm;
  DfmgState dfmg;
};

std::string fmt(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_generate(int shape, const std::int64_t* dims, const double* lengths,
                    const double* params, std::uint8_t* out) {
  try {
    const std::array<std::int64_t, 3> d{dims[0], dims[1], dims[2]};
    const std::array<double, 3> l{lengths[0], lengths[1], lengths[2]};
    PhaseImage img;
    switch (shape) {
      case 0: img = generate_sphere(d, l, params[0]); break;
      case 1: img = generate_octahedron(d, l, params[0]); break;
      case 2: img = generate_fiber(d, l, int(params[0]), params[1], params[2]); break;
      case 3: img = generate_cross_ply(d, l, params[0], params[1], int(params[2])); break;
      case 4:
        img = generate_fiber_pack(d, l, std::uint64_t(params[0]), int(params[1]), params[2],
                                  params[3], params[4]);
        break;
      case 5: img = generate_slab(d, l, int(params[0]), params[1]); break;
      case 10:
      case 11:
      case 12: img = generate_config(shape, d, l, params); break;
      default: g_err = "unknown shape"; return -13;
    }
    std::memcpy(out, img.data.data(), img.data.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int oracle_mirror(const std::uint8_t* img, const std::int64_t* dims, int axis, std::uint8_t* out) {
  const double l[3] = {1, 1, 1};
  const PhaseImage m = mirrored(make_image(img, dims, l), axis);
  std::memcpy(out, m.data.data(), m.data.size());
  return 0;
}

int oracle_coarsen(const std::uint8_t* img, const std::int64_t* dims, const double* lengths,
                   const std::int64_t* factors, std::uint8_t* kind, double* c_plus,
                   std::int64_t* count_plus) {
  try {
    const ComboGrid g = coarsen(make_image(img, dims, lengths), {factors[0], factors[1], factors[2]});
    std::memcpy(kind, g.kind.data(), g.kind.size());
    std::memcpy(c_plus, g.c_plus.data(), g.c_plus.size() * sizeof(double));
    std::memcpy(count_plus, g.count_plus.data(), g.count_plus.size() * sizeof(std::int64_t));
    return 0;
  } catch (const NonDividingFactor& e) {
    g_err = e.what();
    return -5;
  }
}

int oracle_laplace_weights(const std::uint8_t* img, const std::int64_t* dims,
                           const double* lengths, double* w) {
  const auto v = laplace_weights(make_image(img, dims, lengths));
  std::memcpy(w, v.data(), v.size() * sizeof(double));
  return 0;
}

int oracle_normals(const std::uint8_t* img, const std::int64_t* dims, const double* lengths,
                   const std::int64_t* factors, int method, int centering, int min_support,
                   double* normal3, std::uint8_t* flags, std::int64_t* stats3) {
  try {
    const PhaseImage im = make_image(img, dims, lengths);
    ComboGrid g = coarsen(im, {factors[0], factors[1], factors[2]});
    const NormalStats st = compute_normals(im, g, method, centering, min_support);
    for (std::size_t i = 0; i < g.normal.size(); ++i)
      for (int d = 0; d < 3; ++d) normal3[3 * i + std::size_t(d)] = g.normal[i][d];
    std::memcpy(flags, g.normal_flag.data(), g.normal_flag.size());
    stats3[0] = st.composite;
    stats3[1] = st.degenerate_fallbacks;
    stats3[2] = st.too_few_fallbacks;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -5;
  }
}

int oracle_sym_eig3(const double* m, double* lam, double* vec) {
  sym_eig3_jacobi(m, lam, vec);
  return 0;
}

int oracle_law_eval(const oracle_law* law, const double* f9, double* p9, double* a81) {
  Mat3 f, p;
  std::memcpy(f.a, f9, sizeof f.a);
  Mat9 a;
  const Law l = to_law(law);
  const bool ok = a81 ? law_eval_tangent(l, f, p, a) : law_eval(l, f, p);
  std::memcpy(p9, p.a, sizeof p.a);
  if (a81) std::memcpy(a81, a.a, sizeof a.a);
  return ok ? 0 : 1;
}

int oracle_spectrum_bounds(const oracle_law* law, const double* f9, double* lohi) {
  Mat3 f;
  std::memcpy(f.a, f9, sizeof f.a);
  law_spectrum_bounds(to_law(law), f, lohi[0], lohi[1]);
  return 0;
}

// finite_strain_solve (laminate.cpp:158-272). out: p9, fp9, fm9, a81, a3;
// istate: converged, iterations, back_projections, first_inadmissible_iter;
// dstate: residual, residual_rel.
int oracle_laminate_solve(const double* fbox9, const oracle_law* plus, const oracle_law* minus,
                          const double* normal3, double c_plus, const double* a0,
                          const oracle_lam_opts* opts, int want_tangent, double* p9, double* fp9,
                          double* fm9, double* a81, double* a3, int* istate, double* dstate) {
  try {
    Mat3 f;
    std::memcpy(f.a, fbox9, sizeof f.a);
    Vec3 n, a;
    for (int d = 0; d < 3; ++d) {
      n[d] = normal3[d];
      a[d] = a0[d];
    }
    const ComboMeta meta = ComboMeta::make(n, c_plus);
    const LaminateSolution s =
        finite_strain_solve(f, to_law(plus), to_law(minus), meta, a, to_opts(opts), want_tangent != 0);
    std::memcpy(p9, s.result.p_box.a, 72);
    std::memcpy(fp9, s.result.f_plus.a, 72);
    std::memcpy(fm9, s.result.f_minus.a, 72);
    if (a81) std::memcpy(a81, s.result.a_box.a, 648);
    for (int d = 0; d < 3; ++d) a3[d] = s.state.a[d];
    istate[0] = s.state.converged;
    istate[1] = s.state.iterations;
    istate[2] = s.state.back_projections;
    istate[3] = s.state.first_inadmissible_iter;
    dstate[0] = s.state.residual;
    dstate[1] = s.state.residual_rel;
    return 0;
  } catch (const InadmissibleMacroState& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CellMaterials handle built from a coarse grid (kind/c_plus/normal arrays).
void* oracle_cm_create(const std::int64_t* dims, const double* lengths, const std::uint8_t* kind,
                       const double* c_plus, const double* normal3, const oracle_law* matrix,
                       const oracle_law* inclusion, int combo, const oracle_lam_opts* opts) {
  try {
    ComboGrid g;
    g.dims = {dims[0], dims[1], dims[2]};
    g.lengths = {lengths[0], lengths[1], lengths[2]};
    const std::size_t n = std::size_t(g.boxel_count());
    g.kind.assign(kind, kind + n);
    g.c_plus.assign(c_plus, c_plus + n);
    g.normal.resize(n);
    for (std::size_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) g.normal[i][d] = normal3[3 * i + std::size_t(d)];
    return new CmHandle{CellMaterials(g, to_law(matrix), to_law(inclusion), combo != 0, to_opts(opts)),
                        DfmgState()};
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void oracle_cm_destroy(void* h) { delete static_cast<CmHandle*>(h); }

long long oracle_cm_composites(void* h) { return static_cast<CmHandle*>(h)->cm.composite_cells(); }

double oracle_cm_represented_c_plus(void* h) { return static_cast<CmHandle*>(h)->cm.represented_c_plus(); }

double oracle_cm_stress_floor(void* h) {
  return static_cast<CmHandle*>(h)->cm.laminate_options().stress_floor;
}

int oracle_cm_warm(void* h, double* warm3, int set) {
  auto& w = static_cast<CmHandle*>(h)->cm.warm_all();
  for (std::size_t i = 0; i < w.size(); ++i)
    for (int d = 0; d < 3; ++d) {
      if (set)
        w[i][d] = warm3[3 * i + std::size_t(d)];
      else
        warm3[3 * i + std::size_t(d)] = w[i][d];
    }
  return 0;
}

// recover_phase_fields + phase_averages (postprocess.cpp:13-106).
// out: pbar 9, pbar_plus 9, pbar_minus 9, c_plus, has_plus, has_minus,
// max_resolve_iterations (31 doubles)
int oracle_phase_averages(void* h, const double* F, double* out) {
  try {
    auto* H = static_cast<CmHandle*>(h);
    CellMaterials& cm = H->cm;
    Field9 f(cm.grid());
    std::memcpy(f.data.data(), F, f.data.size() * sizeof(double));
    // recover_phase_fields (postprocess.cpp:13-38): warm starts read only
    const std::int64_t nid = cm.composite_cells();
    std::vector<Mat3> pplus(static_cast<std::size_t>(nid)), pminus(static_cast<std::size_t>(nid));
    std::vector<std::int64_t> cell_of(static_cast<std::size_t>(nid), -1);
    for (std::int64_t i = 0; i < cm.cells(); ++i)
      if (cm.cell_phase(std::size_t(i)) == 2) cell_of[std::size_t(cm.combo_id(std::size_t(i)))] = i;
    int iter_max = 0;
    for (std::int64_t id = 0; id < nid; ++id) {
      const Mat3 fc = f.cell(std::size_t(cell_of[std::size_t(id)]));
      const LaminateSolution sol =
          finite_strain_solve(fc, cm.inclusion(), cm.matrix(), cm.meta(std::int32_t(id)),
                              cm.warm_all()[std::size_t(id)], cm.laminate_options(), false);
      pplus[std::size_t(id)] = sol.result.p_plus;
      pminus[std::size_t(id)] = sol.result.p_minus;
      iter_max = std::max(iter_max, sol.state.iterations);
    }
    // phase_averages (postprocess.cpp:49-106): chunk-4096 partials, fixed order
    const std::int64_t n = cm.cells(), chunk = 4096, nch = (n + chunk - 1) / chunk;
    Mat3 tps, tms;
    double tpw = 0.0, tmw = 0.0;
    for (std::int64_t c = 0; c < nch; ++c) {
      Mat3 aps, ams;
      double apw = 0.0, amw = 0.0;
      for (std::int64_t i = c * chunk; i < std::min(n, (c + 1) * chunk); ++i) {
        const std::uint8_t ph = cm.cell_phase(std::size_t(i));
        if (ph == 2) {
          const std::int32_t id = cm.combo_id(std::size_t(i));
          const ComboMeta& m = cm.meta(id);
          for (int q = 0; q < 9; ++q) {
            aps.a[q] += m.c_plus * pplus[std::size_t(id)].a[q];
            ams.a[q] += m.c_minus * pminus[std::size_t(id)].a[q];
          }
          apw += m.c_plus;
          amw += m.c_minus;
        } else {
          Mat3 p;
          law_eval(ph == 1 ? cm.inclusion() : cm.matrix(), f.cell(std::size_t(i)), p);
          Mat3& acc = ph == 1 ? aps : ams;
          for (int q = 0; q < 9; ++q) acc.a[q] += p.a[q];
          (ph == 1 ? apw : amw) += 1.0;
        }
      }
      for (int q = 0; q < 9; ++q) {
        tps.a[q] += aps.a[q];
        tms.a[q] += ams.a[q];
      }
      tpw += apw;
      tmw += amw;
    }
    for (int q = 0; q < 9; ++q) {
      const int i = q / 3, j = q % 3;
      out[q] = (tps(i, j) + tms(i, j)) / double(n);
      out[9 + q] = tpw > 0.0 ? tps(i, j) / tpw : 0.0;
      out[18 + q] = tmw > 0.0 ? tms(i, j) / tmw : 0.0;
    }
    out[27] = tpw / double(n);
    out[28] = tpw > 0.0;
    out[29] = tmw > 0.0;
    out[30] = iter_max;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// stress_sweep (cell_material.cpp:104-168); t45 nullable; stats4:
// inadmissible, failures, back_projections, iter_max
int oracle_stress_sweep(void* h, const double* F, double* P, double* t45, std::int64_t* stats4) {
  auto* H = static_cast<CmHandle*>(h);
  Field9 f(H->cm.grid()), p(H->cm.grid());
  std::memcpy(f.data.data(), F, f.data.size() * sizeof(double));
  std::vector<double> tv;
  const SweepStats st = stress_sweep(H->cm, f, p, t45 ? &tv : nullptr);
  std::memcpy(P, p.data.data(), p.data.size() * sizeof(double));
  if (t45) std::memcpy(t45, tv.data(), tv.size() * sizeof(double));
  stats4[0] = st.inadmissible_cells;
  stats4[1] = st.laminate_failures;
  stats4[2] = st.back_projections;
  stats4[3] = st.laminate_iter_max;
  return 0;
}

int oracle_tangent_matvec(const double* t45, const std::int64_t* dims, const double* x, double* y) {
  SimGrid g;
  g.dims = {dims[0], dims[1], dims[2]};
  Field9 X(g), Y(g);
  std::memcpy(X.data.data(), x, X.data.size() * sizeof(double));
  const std::vector<double> t(t45, t45 + 45 * g.cells());
  tangent_matvec(t, X, Y);
  std::memcpy(y, Y.data.data(), Y.data.size() * sizeof(double));
  return 0;
}

int oracle_dfmg_stress(void* h, const double* F, double* P, std::int64_t* stats4) {
  auto* H = static_cast<CmHandle*>(h);
  Field9 f(H->cm.grid()), p(H->cm.grid());
  std::memcpy(f.data.data(), F, f.data.size() * sizeof(double));
  const SweepStats st = dfmg_stress(H->cm, H->dfmg, f, p);
  std::memcpy(P, p.data.data(), p.data.size() * sizeof(double));
  stats4[0] = st.inadmissible_cells;
  stats4[1] = st.laminate_failures;
  stats4[2] = st.back_projections;
  stats4[3] = st.laminate_iter_max;
  return 0;
}

// exact linearization check: t45 per doubly-fine cell (8 per cell)
int oracle_dfmg_tangent(void* h, const double* F, const double* x, double* y) {
  auto* H = static_cast<CmHandle*>(h);
  Field9 f(H->cm.grid()), X(H->cm.grid()), Y(H->cm.grid());
  std::memcpy(f.data.data(), F, f.data.size() * sizeof(double));
  std::memcpy(X.data.data(), x, X.data.size() * sizeof(double));
  std::vector<double> t;
  dfmg_tangent_pass(H->cm, H->dfmg, f, t);
  dfmg_tangent_matvec(t, X, Y);
  std::memcpy(y, Y.data.data(), Y.data.size() * sizeof(double));
  return 0;
}

int oracle_dfmg_warm(void* h, double* warm3, int set) {
  auto* H = static_cast<CmHandle*>(h);
  const std::size_t n = std::size_t(8 * H->cm.cells());
  if (H->dfmg.warm_a.size() != n) H->dfmg.resize(H->cm.cells());
  for (std::size_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) {
      if (set)
        H->dfmg.warm_a[i][d] = warm3[3 * i + std::size_t(d)];
      else
        warm3[3 * i + std::size_t(d)] = H->dfmg.warm_a[i][d];
    }
  return 0;
}

// GreenOperator::project (green.cpp:133-151)
int oracle_project(const std::int64_t* dims, const double* lengths, int kind, const double* in,
                   double* out) {
  SimGrid g;
  g.dims = {dims[0], dims[1], dims[2]};
  g.lengths = {lengths[0], lengths[1], lengths[2]};
  Field9 a(g), b(g);
  std::memcpy(a.data.data(), in, a.data.size() * sizeof(double));
  GreenOperator green(kind, g);
  Fft3 fft(g.dims, 9);
  green.project(a, b, fft);
  std::memcpy(out, b.data.data(), b.data.size() * sizeof(double));
  return 0;
}

// raw r2c of ncomp components (fft.cpp:52): out is complex interleaved
int oracle_fft_forward(const std::int64_t* dims, int ncomp, const double* in, double* out) {
  Fft3 fft({dims[0], dims[1], dims[2]}, ncomp);
  for (int c = 0; c < ncomp; ++c) std::memcpy(fft.real(c), in + c * fft.n_real(), fft.n_real() * 8);
  fft.forward();
  for (int c = 0; c < ncomp; ++c) std::memcpy(out + 2 * c * fft.n_complex(), fft.cplx(c), fft.n_complex() * 16);
  return 0;
}

// solve (solver.cpp:286-346). Returns a malloc'd JSON report (free with
// oracle_free); F_out / P_out nullable.
char* oracle_solve(void* h, const double* fbar9, const oracle_solver_cfg* c, double* F_out,
                   double* P_out, double* pbar9) {
  auto* H = static_cast<CmHandle*>(h);
  SolverConfig cfg;
  cfg.scheme = c->scheme;
  cfg.green = c->green;
  cfg.eval = c->eval;
  cfg.tol_equilibrium = c->tol_equilibrium;
  cfg.max_outer = c->max_outer;
  cfg.cg_tol = c->cg_tol;
  cfg.cg_max = c->cg_max;
  cfg.load_steps = c->load_steps;
  cfg.max_bisections = c->max_bisections;
  cfg.threads = c->threads;
  cfg.verbose = c->verbose != 0;
  cfg.max_ls_iterations = c->max_ls_iterations;
  Mat3 fbar;
  std::memcpy(fbar.a, fbar9, 72);
  std::ostringstream js;
  try {
    const SolveResult r = solve(H->cm, fbar, cfg);
    if (F_out) std::memcpy(F_out, r.f.data.data(), r.f.data.size() * 8);
    if (P_out && !r.p.data.empty()) std::memcpy(P_out, r.p.data.data(), r.p.data.size() * 8);
    std::memcpy(pbar9, r.pbar.a, 72);
    const auto& rep = r.report;
    js << "{\"success\":" << (rep.success ? "true" : "false") << ",\"error\":\"" << rep.error
       << "\",\"bisections\":" << rep.bisections << ",\"alpha\":" << fmt(rep.alpha)
       << ",\"seconds_total\":" << fmt(rep.seconds_total) << ",\"ls_total\":" << rep.ls_total
       << ",\"ls_clock\":[";
    for (std::size_t i = 0; i < rep.ls_clock.size(); ++i) js << (i ? "," : "") << fmt(rep.ls_clock[i]);
    js << "],\"steps\":[";
    for (std::size_t s = 0; s < rep.steps.size(); ++s) {
      const auto& st = rep.steps[s];
      if (s) js << ",";
      js << "{\"t_start\":" << fmt(st.t_start) << ",\"t_end\":" << fmt(st.t_end)
         << ",\"converged\":" << (st.converged ? "true" : "false")
         << ",\"outer_iters\":" << st.outer_iters << ",\"cg_breakdowns\":" << st.cg_breakdowns
         << ",\"line_search_cuts\":" << st.line_search_cuts << ",\"seconds\":" << fmt(st.seconds)
         << ",\"ls_basic\":" << st.ls_basic << ",\"ls_residual\":" << st.ls_residual
         << ",\"ls_cg\":" << st.ls_cg << ",\"ls_trial\":" << st.ls_trial << ",\"fbar\":[";
      for (int i = 0; i < 9; ++i) js << (i ? "," : "") << fmt(st.fbar.a[i]);
      js << "],\"residuals\":[";
      for (std::size_t i = 0; i < st.residuals.size(); ++i) js << (i ? "," : "") << fmt(st.residuals[i]);
      js << "],\"cg_iters\":[";
      for (std::size_t i = 0; i < st.cg_iters.size(); ++i) js << (i ? "," : "") << st.cg_iters[i];
      js << "],\"pbar_history\":[";
      for (std::size_t i = 0; i < st.pbar_history.size(); ++i) {
        js << (i ? "," : "") << "[";
        for (int q = 0; q < 9; ++q) js << (q ? "," : "") << fmt(st.pbar_history[i].a[q]);
        js << "]";
      }
      js << "],\"sweep\":{\"inadmissible\":" << st.sweep.inadmissible_cells
         << ",\"failures\":" << st.sweep.laminate_failures
         << ",\"back_projections\":" << st.sweep.back_projections
         << ",\"iter_max\":" << st.sweep.laminate_iter_max << "}}";
    }
    js << "]}";
  } catch (const std::exception& e) {
    js.str("");
    js << "{\"success\":false,\"exception\":\"" << e.what() << "\"}";
  }
  const std::string s = js.str();
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

void oracle_free(void* p) { std::free(p); }

}  // extern "C"
