// TEST INFRASTRUCTURE ONLY (see oracle.hpp): fields, FFT, Green operator,
// cell binding, stress sweeps, DFMG and the LS solver, restated from
// /root/reference/proj/src/{field,fft,green,cell_material,dfmg,solver}.cpp.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <limits>
#include <map>
#include <memory>
#include <mutex>

#include "oracle.hpp"

namespace oracle {

// ------------------------------------------------------------------ fields
Mat3 Field9::cell(std::size_t idx) const {
  Mat3 m;
  const std::size_t n = std::size_t(cells());
  for (int c = 0; c < 9; ++c) m.a[c] = data[std::size_t(c) * n + idx];
  return m;
}
void Field9::set_cell(std::size_t idx, const Mat3& m) {
  const std::size_t n = std::size_t(cells());
  for (int c = 0; c < 9; ++c) data[std::size_t(c) * n + idx] = m.a[c];
}
// field.cpp:8-16
void Field9::fill(const Mat3& m) {
  const std::int64_t n = cells();
  for (int c = 0; c < 9; ++c) {
    double* p = comp(c);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < n; ++i) p[i] = m.a[c];
  }
}
// field.cpp:18-26
Mat3 Field9::mean() const {
  Mat3 m;
  const std::int64_t n = cells();
  for (int c = 0; c < 9; ++c) m.a[c] = deterministic_sum(comp(c), std::size_t(n)) / double(n);
  return m;
}
// field.cpp:28-38
void Field9::pin_mean(const Mat3& target) {
  const Mat3 cur = mean();
  const std::int64_t n = cells();
  for (int c = 0; c < 9; ++c) {
    const double shift = target.a[c] - cur.a[c];
    if (shift == 0.0) continue;
    double* p = comp(c);
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < n; ++i) p[i] += shift;
  }
}

// parallel.hpp:40-104: fixed chunk-4096 partials combined in chunk order
double deterministic_sum(const double* x, std::size_t n) {
  constexpr std::size_t chunk = 4096;
  const std::size_t nchunks = (n + chunk - 1) / chunk;
  std::vector<double> partial(nchunks, 0.0);
#pragma omp parallel for schedule(static)
  for (std::ptrdiff_t c = 0; c < std::ptrdiff_t(nchunks); ++c) {
    const std::size_t lo = std::size_t(c) * chunk, hi = std::min(lo + chunk, n);
    double s = 0.0;
    for (std::size_t i = lo; i < hi; ++i) s += x[i];
    partial[std::size_t(c)] = s;
  }
  double total = 0.0;
  for (double p : partial) total += p;
  return total;
}
double deterministic_dot(const double* x, const double* y, std::size_t n) {
  constexpr std::size_t chunk = 4096;
  const std::size_t nchunks = (n + chunk - 1) / chunk;
  std::vector<double> partial(nchunks, 0.0);
#pragma omp parallel for schedule(static)
  for (std::ptrdiff_t c = 0; c < std::ptrdiff_t(nchunks); ++c) {
    const std::size_t lo = std::size_t(c) * chunk, hi = std::min(lo + chunk, n);
    double s = 0.0;
    for (std::size_t i = lo; i < hi; ++i) s += x[i] * y[i];
    partial[std::size_t(c)] = s;
  }
  double total = 0.0;
  for (double p : partial) total += p;
  return total;
}
double deterministic_sumsq(const double* x, std::size_t n) { return deterministic_dot(x, x, n); }

// --------------------------------------------------------------------- FFT
namespace {
constexpr long double kPiL = 3.141592653589793238462643383279502884L;

/// Line FFT plan: mixed-radix Stockham autosort, twiddles rounded from long
/// double. Stands in for FFTW's many-plans (fft.cpp:35-40).
struct LinePlan {
  int n = 1;
  std::vector<int> radices;
  std::vector<std::complex<double>> tw;  // exp(-2 pi i k / n)
  explicit LinePlan(int n_) : n(n_) {
    int m = n;
    while (m % 4 == 0) { radices.push_back(4); m /= 4; }
    while (m % 2 == 0) { radices.push_back(2); m /= 2; }
    for (int p = 3; m > 1; p += 2)
      while (m % p == 0) { radices.push_back(p); m /= p; }
    tw.resize(std::size_t(n));
    for (int k = 0; k < n; ++k) {
      const long double ph = -2.0L * kPiL * (long double)k / (long double)n;
      tw[std::size_t(k)] = {double(cosl(ph)), double(sinl(ph))};
    }
  }
  // in-place transform of x (length n) using work (length n); sign -1 fwd
  void exec(std::complex<double>* x, std::complex<double>* work, bool inverse) const {
    if (n == 1) return;
    std::complex<double>* src = x;
    std::complex<double>* dst = work;
    int p = 1;
    std::complex<double> v[64], out[64];
    std::vector<std::complex<double>> vbig, obig;
    for (int R : radices) {
      std::complex<double>* vv = v;
      std::complex<double>* oo = out;
      if (R > 64) {
        vbig.resize(std::size_t(R));
        obig.resize(std::size_t(R));
        vv = vbig.data();
        oo = obig.data();
      }
      const int m = n / R;
      const int tstride = n / (p * R);
      for (int t = 0; t < m; ++t) {
        const int k = t % p;
        for (int r = 0; r < R; ++r) {
          std::complex<double> w = tw[std::size_t((std::int64_t(r) * k * tstride) % n)];
          if (inverse) w = std::conj(w);
          vv[r] = src[t + r * m] * w;
        }
        if (R == 2) {
          oo[0] = vv[0] + vv[1];
          oo[1] = vv[0] - vv[1];
        } else if (R == 4) {
          const std::complex<double> a0 = vv[0] + vv[2], a1 = vv[0] - vv[2];
          const std::complex<double> b0 = vv[1] + vv[3], b1 = vv[1] - vv[3];
          // multiply b1 by -i (forward) or +i (inverse)
          const std::complex<double> jb1 =
              inverse ? std::complex<double>(-b1.imag(), b1.real())
                      : std::complex<double>(b1.imag(), -b1.real());
          oo[0] = a0 + b0;
          oo[1] = a1 + jb1;
          oo[2] = a0 - b0;
          oo[3] = a1 - jb1;
        } else {
          const int step = n / R;
          for (int s = 0; s < R; ++s) {
            std::complex<double> acc = 0.0;
            for (int r = 0; r < R; ++r) {
              std::complex<double> w = tw[std::size_t(((r * s) % R) * step)];
              if (inverse) w = std::conj(w);
              acc += vv[r] * w;
            }
            oo[s] = acc;
          }
        }
        const int j = (t - k) * R + k;
        for (int r = 0; r < R; ++r) dst[j + r * p] = oo[r];
      }
      std::swap(src, dst);
      p *= R;
    }
    if (src != x) std::copy(src, src + n, x);
  }
};

std::shared_ptr<const LinePlan> get_plan(int n) {
  static std::mutex mu;
  static std::map<int, std::shared_ptr<const LinePlan>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  auto p = std::make_shared<const LinePlan>(n);
  cache[n] = p;
  return p;
}
}  // namespace

Fft3::Fft3(const std::array<std::int64_t, 3>& dims, int ncomp) : dims_(dims), ncomp_(ncomp) {
  n_ = dims[0] * dims[1] * dims[2];
  nc_ = dims[0] * dims[1] * (dims[2] / 2 + 1);
  real_.assign(std::size_t(ncomp_ * n_), 0.0);
  cplx_.assign(std::size_t(ncomp_ * nc_), 0.0);
}

void Fft3::forward() {
  const std::int64_t n1 = dims_[0], n2 = dims_[1], n3 = dims_[2], n3c = n3 / 2 + 1;
  const auto p1 = get_plan(int(n1)), p2 = get_plan(int(n2)), p3 = get_plan(int(n3));
  for (int c = 0; c < ncomp_; ++c) {
    const double* re = real(c);
    std::complex<double>* cx = cplx(c);
#pragma omp parallel
    {
      std::vector<std::complex<double>> buf(std::size_t(std::max({n1, n2, n3}))), work(buf.size());
#pragma omp for schedule(static)
      for (std::int64_t line = 0; line < n1 * n2; ++line) {
        for (std::int64_t k = 0; k < n3; ++k) buf[std::size_t(k)] = re[line * n3 + k];
        p3->exec(buf.data(), work.data(), false);
        for (std::int64_t k = 0; k < n3c; ++k) cx[line * n3c + k] = buf[std::size_t(k)];
      }
#pragma omp for schedule(static)
      for (std::int64_t q = 0; q < n1 * n3c; ++q) {
        const std::int64_t i = q / n3c, k = q % n3c;
        for (std::int64_t j = 0; j < n2; ++j) buf[std::size_t(j)] = cx[(i * n2 + j) * n3c + k];
        p2->exec(buf.data(), work.data(), false);
        for (std::int64_t j = 0; j < n2; ++j) cx[(i * n2 + j) * n3c + k] = buf[std::size_t(j)];
      }
#pragma omp for schedule(static)
      for (std::int64_t q = 0; q < n2 * n3c; ++q) {
        const std::int64_t j = q / n3c, k = q % n3c;
        for (std::int64_t i = 0; i < n1; ++i) buf[std::size_t(i)] = cx[(i * n2 + j) * n3c + k];
        p1->exec(buf.data(), work.data(), false);
        for (std::int64_t i = 0; i < n1; ++i) cx[(i * n2 + j) * n3c + k] = buf[std::size_t(i)];
      }
    }
  }
}

// fft.cpp:54-60: unnormalized c2r (imaginary parts of the DC / Nyquist
// coefficients of the last axis are ignored, as a halfcomplex c2r does),
// followed by the 1/n scaling.
void Fft3::inverse() {
  const std::int64_t n1 = dims_[0], n2 = dims_[1], n3 = dims_[2], n3c = n3 / 2 + 1;
  const auto p1 = get_plan(int(n1)), p2 = get_plan(int(n2)), p3 = get_plan(int(n3));
  const double scale = 1.0 / double(n_);
  for (int c = 0; c < ncomp_; ++c) {
    double* re = real(c);
    std::complex<double>* cx = cplx(c);
#pragma omp parallel
    {
      std::vector<std::complex<double>> buf(std::size_t(std::max({n1, n2, n3}))), work(buf.size());
#pragma omp for schedule(static)
      for (std::int64_t q = 0; q < n2 * n3c; ++q) {
        const std::int64_t j = q / n3c, k = q % n3c;
        for (std::int64_t i = 0; i < n1; ++i) buf[std::size_t(i)] = cx[(i * n2 + j) * n3c + k];
        p1->exec(buf.data(), work.data(), true);
        for (std::int64_t i = 0; i < n1; ++i) cx[(i * n2 + j) * n3c + k] = buf[std::size_t(i)];
      }
#pragma omp for schedule(static)
      for (std::int64_t q = 0; q < n1 * n3c; ++q) {
        const std::int64_t i = q / n3c, k = q % n3c;
        for (std::int64_t j = 0; j < n2; ++j) buf[std::size_t(j)] = cx[(i * n2 + j) * n3c + k];
        p2->exec(buf.data(), work.data(), true);
        for (std::int64_t j = 0; j < n2; ++j) cx[(i * n2 + j) * n3c + k] = buf[std::size_t(j)];
      }
#pragma omp for schedule(static)
      for (std::int64_t line = 0; line < n1 * n2; ++line) {
        for (std::int64_t k = 0; k < n3c; ++k) buf[std::size_t(k)] = cx[line * n3c + k];
        for (std::int64_t k = n3c; k < n3; ++k) buf[std::size_t(k)] = std::conj(cx[line * n3c + (n3 - k)]);
        buf[0] = {buf[0].real(), 0.0};
        if (n3 % 2 == 0 && n3 > 1) buf[std::size_t(n3 / 2)] = {buf[std::size_t(n3 / 2)].real(), 0.0};
        p3->exec(buf.data(), work.data(), true);
        for (std::int64_t k = 0; k < n3; ++k) re[line * n3 + k] = buf[std::size_t(k)].real();
      }
    }
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < n_; ++i) re[i] *= scale;
  }
}

// ------------------------------------------------------------------- green
namespace {
constexpr double kPi = 3.141592653589793238462643383279502884;
}

// green.cpp:16-57
GreenOperator::GreenOperator(int kind, const SimGrid& grid) : kind_(kind), grid_(grid) {
  for (int a = 0; a < 3; ++a) {
    const std::int64_t n = grid.dims[a];
    const double h = grid.spacing(a);
    const double l = grid.lengths[a];
    fwd_[a].resize(std::size_t(n));
    avg_[a].resize(std::size_t(n));
    xi_[a].resize(std::size_t(n));
    for (std::int64_t k = 0; k < n; ++k) {
      const auto sk = std::size_t(k);
      if (k == 0) {
        fwd_[a][sk] = 0.0;
        avg_[a][sk] = 1.0;
        xi_[a][sk] = 0.0;
        continue;
      }
      if (2 * k == n) {
        fwd_[a][sk] = -2.0 / h;
        avg_[a][sk] = 0.0;
        xi_[a][sk] = 2.0 * kPi * double(k) / l;
        continue;
      }
      const double phi = 2.0 * kPi * double(k) / double(n);
      const std::complex<double> e(std::cos(phi), std::sin(phi));
      fwd_[a][sk] = (e - 1.0) / h;
      avg_[a][sk] = 0.5 * (e + 1.0);
      const std::int64_t ks = 2 * k < n ? k : k - n;
      xi_[a][sk] = 2.0 * kPi * double(ks) / l;
    }
  }
}

// green.cpp:59-131
void GreenOperator::apply_fourier(Fft3& fft) const {
  const auto& d = grid_.dims;
  const std::int64_t n3c = d[2] / 2 + 1;
  std::array<std::complex<double>*, 9> buf;
  for (int c = 0; c < 9; ++c) buf[std::size_t(c)] = fft.cplx(c);
  const bool staggered = kind_ == kStaggered;
#pragma omp parallel for collapse(2) schedule(static)
  for (std::int64_t k1 = 0; k1 < d[0]; ++k1) {
    for (std::int64_t k2 = 0; k2 < d[1]; ++k2) {
      for (std::int64_t k3 = 0; k3 < n3c; ++k3) {
        const std::size_t idx = std::size_t((k1 * d[1] + k2) * n3c + k3);
        const auto s1 = std::size_t(k1), s2 = std::size_t(k2), s3 = std::size_t(k3);
        std::complex<double> g[3];
        if (kind_ == kContinuous) {
          const bool nyquist = 2 * k1 == d[0] || 2 * k2 == d[1] || 2 * k3 == d[2];
          if (nyquist) {
            for (int c = 0; c < 9; ++c) buf[std::size_t(c)][idx] = 0.0;
            continue;
          }
          g[0] = {0.0, xi_[0][s1]};
          g[1] = {0.0, xi_[1][s2]};
          g[2] = {0.0, xi_[2][s3]};
        } else if (kind_ == kRotated) {
          const auto a1 = avg_[0][s1], a2 = avg_[1][s2], a3 = avg_[2][s3];
          g[0] = fwd_[0][s1] * a2 * a3;
          g[1] = fwd_[1][s2] * a1 * a3;
          g[2] = fwd_[2][s3] * a1 * a2;
        } else {
          g[0] = fwd_[0][s1];
          g[1] = fwd_[1][s2];
          g[2] = fwd_[2][s3];
        }
        const double den = std::norm(g[0]) + std::norm(g[1]) + std::norm(g[2]);
        if (den == 0.0) {
          for (int c = 0; c < 9; ++c) buf[std::size_t(c)][idx] = 0.0;
          continue;
        }
        for (int i = 0; i < 3; ++i) {
          std::complex<double> gr[3];
          for (int J = 0; J < 3; ++J) gr[J] = (staggered && J != i) ? -std::conj(g[J]) : g[J];
          std::complex<double> s = 0.0;
          for (int L = 0; L < 3; ++L) s += std::conj(gr[L]) * buf[std::size_t(3 * i + L)][idx];
          s /= den;
          for (int J = 0; J < 3; ++J) buf[std::size_t(3 * i + J)][idx] = gr[J] * s;
        }
      }
    }
  }
}

// green.cpp:133-151
void GreenOperator::project(const Field9& in, Field9& out, Fft3& fft) const {
  const std::int64_t n = in.cells();
  for (int c = 0; c < 9; ++c) std::copy(in.comp(c), in.comp(c) + n, fft.real(c));
  fft.forward();
  apply_fourier(fft);
  fft.inverse();
  if (out.cells() != n) out = Field9(in.grid);
  for (int c = 0; c < 9; ++c) std::copy(fft.real(c), fft.real(c) + n, out.comp(c));
}

// ------------------------------------------------------------ cell binding
// cell_material.cpp:12-55
CellMaterials::CellMaterials(const ComboGrid& grid, const Law& matrix, const Law& inclusion,
                             bool combo, LaminateOptions lam)
    : matrix_(matrix), inclusion_(inclusion), lam_(lam), combo_(combo) {
  grid_.dims = grid.dims;
  grid_.lengths = grid.lengths;
  const std::int64_t n = grid_.cells();
  phase_.assign(std::size_t(n), 0);
  combo_id_.assign(std::size_t(n), -1);
  for (std::int64_t i = 0; i < n; ++i) {
    const auto si = std::size_t(i);
    switch (grid.kind[si]) {
      case kPureMatrix: phase_[si] = 0; break;
      case kPureInclusion: phase_[si] = 1; break;
      default:
        if (combo_ && grid.c_plus[si] >= lam_.c_min && 1.0 - grid.c_plus[si] >= lam_.c_min) {
          phase_[si] = 2;
          combo_id_[si] = std::int32_t(metas_.size());
          metas_.push_back(ComboMeta::make(grid.normal[si], grid.c_plus[si]));
          c_plus_.push_back(grid.c_plus[si]);
        } else {
          phase_[si] = grid.c_plus[si] >= 0.5 ? 1 : 0;
        }
    }
  }
  warm_a_.assign(metas_.size(), Vec3());
  if (lam_.stress_floor == 0.0) {
    double lo, hi;
    spectrum_bounds(Mat3::identity(), lo, hi);
    lam_.stress_floor = 1e-12 * std::max(hi, 1e-12);
  }
}

double CellMaterials::represented_c_plus() const {
  long double acc = 0.0L;
  for (std::size_t i = 0; i < phase_.size(); ++i) {
    if (phase_[i] == 1) acc += 1.0L;
    if (phase_[i] == 2) acc += c_plus_[std::size_t(combo_id_[i])];
  }
  return double(acc / (long double)phase_.size());
}

// cell_material.cpp:77-84
void CellMaterials::spectrum_bounds(const Mat3& fbar, double& lo, double& hi) const {
  double l0, h0, l1, h1;
  law_spectrum_bounds(matrix_, fbar, l0, h0);
  law_spectrum_bounds(inclusion_, fbar, l1, h1);
  lo = std::min(l0, l1);
  hi = std::max(h0, h1);
}

// cell_material.cpp:86-102
void pack45(const Mat9& a, double* dst) {
  int t = 0;
  for (int r = 0; r < 9; ++r)
    for (int c = r; c < 9; ++c) dst[t++] = 0.5 * (a(r, c) + a(c, r));
}
Mat9 unpack45(const double* src) {
  Mat9 a;
  int t = 0;
  for (int r = 0; r < 9; ++r)
    for (int c = r; c < 9; ++c) {
      a(r, c) = src[t];
      a(c, r) = src[t];
      ++t;
    }
  return a;
}

// cell_material.cpp:104-168. lean: t45 holds the composite cells' tangents
// only (by combo id); pure cells' tangents are recomputed from F by
// tangent_matvec_lean (same arithmetic, 360 B/cell less: the 512^3 fixture
// and CPU baseline fit the B200 box's host RAM).
SweepStats stress_sweep(CellMaterials& cm, const Field9& f, Field9& p, std::vector<double>* t45, bool lean) {
  const std::int64_t n = cm.cells();
  if (p.cells() != n) p = Field9(f.grid);
  if (t45) t45->resize(std::size_t(45 * (lean ? std::max<std::int64_t>(cm.composite_cells(), 1) : n)));
  std::atomic<std::int64_t> inadmissible{0}, failures{0}, backproj{0};
  std::atomic<int> iter_max{0};
  const bool want_tan = t45 != nullptr;
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < n; ++i) {
    const auto si = std::size_t(i);
    const Mat3 fc = f.cell(si);
    Mat3 pc;
    Mat9 ac;
    const std::uint8_t ph = cm.cell_phase(si);
    if (ph == 2) {
      const std::int32_t id = cm.combo_id(si);
      LaminateSolution sol;
      try {
        sol = finite_strain_solve(fc, cm.inclusion(), cm.matrix(), cm.meta(id),
                                  cm.warm_all()[std::size_t(id)], cm.laminate_options(), want_tan);
      } catch (const InadmissibleMacroState&) {
        inadmissible.fetch_add(1, std::memory_order_relaxed);
        p.set_cell(si, Mat3());
        if (want_tan) pack45(Mat9::identity(), t45->data() + 45 * (lean ? std::int64_t(id) : i));
        continue;
      }
      if (!sol.state.converged) failures.fetch_add(1, std::memory_order_relaxed);
      backproj.fetch_add(sol.state.back_projections, std::memory_order_relaxed);
      int prev = iter_max.load(std::memory_order_relaxed);
      while (prev < sol.state.iterations &&
             !iter_max.compare_exchange_weak(prev, sol.state.iterations)) {
      }
      cm.warm_all()[std::size_t(id)] = sol.state.a;
      pc = sol.result.p_box;
      if (want_tan) ac = sol.result.a_box;
      if (want_tan && lean) {
        pack45(ac, t45->data() + 45 * std::int64_t(id));
        p.set_cell(si, pc);
        continue;
      }
    } else {
      const Law& law = ph == 1 ? cm.inclusion() : cm.matrix();
      const bool ok = want_tan ? law_eval_tangent(law, fc, pc, ac) : law_eval(law, fc, pc);
      if (!ok) {
        inadmissible.fetch_add(1, std::memory_order_relaxed);
        pc = Mat3();
        if (want_tan) ac = Mat9::identity();
      }
    }
    p.set_cell(si, pc);
    if (want_tan && !lean) pack45(ac, t45->data() + 45 * i);
  }
  SweepStats st;
  st.inadmissible_cells = inadmissible.load();
  st.laminate_failures = failures.load();
  st.back_projections = backproj.load();
  st.laminate_iter_max = iter_max.load();
  return st;
}

// cell_material.cpp:170-194
void tangent_matvec(const std::vector<double>& t45, const Field9& x, Field9& y) {
  const std::int64_t n = x.cells();
  if (y.cells() != n) y = Field9(x.grid);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < n; ++i) {
    const double* a = t45.data() + 45 * i;
    double xv[9], yv[9];
    for (int c = 0; c < 9; ++c) xv[c] = x.data[std::size_t(c) * std::size_t(n) + std::size_t(i)];
    for (int c = 0; c < 9; ++c) yv[c] = 0.0;
    int t = 0;
    for (int r = 0; r < 9; ++r) {
      yv[r] += a[t] * xv[r];
      ++t;
      for (int c = r + 1; c < 9; ++c, ++t) {
        yv[r] += a[t] * xv[c];
        yv[c] += a[t] * xv[r];
      }
    }
    for (int c = 0; c < 9; ++c) y.data[std::size_t(c) * std::size_t(n) + std::size_t(i)] = yv[c];
  }
}

// tangent_matvec with the lean tangent storage of stress_sweep: composite
// tangents by combo id, pure cells' tangents re-evaluated at F (identical
// to the stored ones: same law, same F, same pack45 symmetrization)
void tangent_matvec_lean(const CellMaterials& cm, const std::vector<double>& t45c, const Field9& f,
                         const Field9& x, Field9& y) {
  const std::int64_t n = x.cells();
  if (y.cells() != n) y = Field9(x.grid);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < n; ++i) {
    const auto si = std::size_t(i);
    double own[45];
    const double* a = own;
    const std::uint8_t ph = cm.cell_phase(si);
    if (ph == 2) {
      a = t45c.data() + 45 * std::int64_t(cm.combo_id(si));
    } else {
      const Law& law = ph == 1 ? cm.inclusion() : cm.matrix();
      Mat3 pc;
      Mat9 ac;
      if (!law_eval_tangent(law, f.cell(si), pc, ac)) ac = Mat9::identity();
      pack45(ac, own);
    }
    double xv[9], yv[9];
    for (int c = 0; c < 9; ++c) xv[c] = x.data[std::size_t(c) * std::size_t(n) + si];
    for (int c = 0; c < 9; ++c) yv[c] = 0.0;
    int t = 0;
    for (int r = 0; r < 9; ++r) {
      yv[r] += a[t] * xv[r];
      ++t;
      for (int c = r + 1; c < 9; ++c, ++t) {
        yv[r] += a[t] * xv[c];
        yv[c] += a[t] * xv[r];
      }
    }
    for (int c = 0; c < 9; ++c) y.data[std::size_t(c) * std::size_t(n) + si] = yv[c];
  }
}

// -------------------------------------------------------------------- DFMG
namespace {
struct GridIdx {  // dfmg.cpp:11-22
  std::int64_t n1, n2, n3;
  static std::int64_t wrap(std::int64_t a, std::int64_t n) {
    a %= n;
    return a < 0 ? a + n : a;
  }
  std::size_t at(std::int64_t i, std::int64_t j, std::int64_t k) const {
    return std::size_t((wrap(i, n1) * n2 + wrap(j, n2)) * n3 + wrap(k, n3));
  }
};

// dfmg.cpp:27-47
Mat3 gather_dfc(const Field9& f, const GridIdx& g, std::int64_t n, std::int64_t ci,
                std::int64_t cj, std::int64_t ck, int s1, int s2, int s3) {
  const std::size_t c0 = g.at(ci, cj, ck);
  const std::size_t c12 = g.at(ci + s1, cj + s2, ck);
  const std::size_t c13 = g.at(ci + s1, cj, ck + s3);
  const std::size_t c23 = g.at(ci, cj + s2, ck + s3);
  const double* d = f.data.data();
  const auto sn = std::size_t(n);
  Mat3 m;
  m(0, 0) = d[0 * sn + c0];
  m(1, 1) = d[4 * sn + c0];
  m(2, 2) = d[8 * sn + c0];
  m(0, 1) = d[1 * sn + c12];
  m(1, 0) = d[3 * sn + c12];
  m(0, 2) = d[2 * sn + c13];
  m(2, 0) = d[6 * sn + c13];
  m(1, 2) = d[5 * sn + c23];
  m(2, 1) = d[7 * sn + c23];
  return m;
}

struct EvalCounters {
  std::atomic<std::int64_t> inadmissible{0}, failures{0}, backproj{0};
  std::atomic<int> iter_max{0};
  SweepStats stats() const {
    SweepStats st;
    st.inadmissible_cells = inadmissible.load();
    st.laminate_failures = failures.load();
    st.back_projections = backproj.load();
    st.laminate_iter_max = iter_max.load();
    return st;
  }
};

// dfmg.cpp:69-109
bool eval_dfc(CellMaterials& cm, const std::vector<Vec3>& snap, DfmgState& state,
              std::size_t host, std::size_t dfc, bool owner, const Mat3& fd, bool want_tan,
              Mat3& p, Mat9* a, EvalCounters& ctr) {
  const std::uint8_t ph = cm.cell_phase(host);
  if (ph == 2) {
    const std::int32_t id = cm.combo_id(host);
    LaminateSolution sol;
    try {
      sol = finite_strain_solve(fd, cm.inclusion(), cm.matrix(), cm.meta(id), snap[dfc],
                                cm.laminate_options(), want_tan);
    } catch (const InadmissibleMacroState&) {
      ctr.inadmissible.fetch_add(1, std::memory_order_relaxed);
      return false;
    }
    if (!sol.state.converged) ctr.failures.fetch_add(1, std::memory_order_relaxed);
    if (owner) {
      ctr.backproj.fetch_add(sol.state.back_projections, std::memory_order_relaxed);
      int prev = ctr.iter_max.load(std::memory_order_relaxed);
      while (prev < sol.state.iterations &&
             !ctr.iter_max.compare_exchange_weak(prev, sol.state.iterations)) {
      }
      state.warm_a[dfc] = sol.state.a;
    }
    p = sol.result.p_box;
    if (a) *a = sol.result.a_box;
    return true;
  }
  const Law& law = ph == 1 ? cm.inclusion() : cm.matrix();
  const bool ok = want_tan && a ? law_eval_tangent(law, fd, p, *a) : law_eval(law, fd, p);
  if (!ok) {
    ctr.inadmissible.fetch_add(1, std::memory_order_relaxed);
    p = Mat3();
    if (a) *a = Mat9::identity();
  }
  return ok;
}

struct PositionClass {  // dfmg.cpp:113-124
  int axis_a, axis_b;
  std::array<int, 3> components;
  int ncomp;
};
constexpr PositionClass kClasses[4] = {
    {-1, -1, {0, 4, 8}, 3},
    {0, 1, {1, 3, -1}, 2},
    {0, 2, {2, 6, -1}, 2},
    {1, 2, {5, 7, -1}, 2},
};
}  // namespace

// dfmg.cpp:128-176
SweepStats dfmg_stress(CellMaterials& cm, DfmgState& state, const Field9& f, Field9& p) {
  const SimGrid& grid = f.grid;
  const std::int64_t n = grid.cells();
  if (state.warm_a.size() != std::size_t(8 * n)) state.resize(n);
  if (p.cells() != n) p = Field9(grid);
  const GridIdx g{grid.dims[0], grid.dims[1], grid.dims[2]};
  const std::vector<Vec3> snapshot = state.warm_a;
  EvalCounters ctr;
#pragma omp parallel for collapse(2) schedule(static)
  for (std::int64_t i = 0; i < grid.dims[0]; ++i) {
    for (std::int64_t j = 0; j < grid.dims[1]; ++j) {
      for (std::int64_t k = 0; k < grid.dims[2]; ++k) {
        const std::size_t cell = grid.index(i, j, k);
        double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (const auto& cls : kClasses) {
          for (int code = 0; code < 8; ++code) {
            const int l1 = code & 1, l2 = (code >> 1) & 1, l3 = (code >> 2) & 1;
            const int l[3] = {l1, l2, l3};
            std::int64_t hi = i, hj = j, hk = k;
            if (cls.axis_a >= 0) {
              const int la = l[cls.axis_a], lb = l[cls.axis_b];
              if (cls.axis_a == 0) hi -= la;
              if (cls.axis_a == 1) hj -= la;
              if (cls.axis_b == 1) hj -= lb;
              if (cls.axis_b == 2) hk -= lb;
            }
            const std::size_t host = g.at(hi, hj, hk);
            const Mat3 fd = gather_dfc(f, g, n, hi, hj, hk, l1, l2, l3);
            const std::size_t dfc = host * 8 + std::size_t(code);
            const bool owner = cls.axis_a < 0;
            Mat3 pd;
            eval_dfc(cm, snapshot, state, host, dfc, owner, fd, false, pd, nullptr, ctr);
            for (int c = 0; c < cls.ncomp; ++c) {
              const int comp = cls.components[std::size_t(c)];
              acc[comp] += pd.a[comp];
            }
          }
        }
        for (int c = 0; c < 9; ++c) p.data[std::size_t(c) * std::size_t(n) + cell] = acc[c] / 8.0;
      }
    }
  }
  return ctr.stats();
}

// dfmg.cpp:178-207
SweepStats dfmg_tangent_pass(CellMaterials& cm, DfmgState& state, const Field9& f,
                             std::vector<double>& t45) {
  const SimGrid& grid = f.grid;
  const std::int64_t n = grid.cells();
  if (state.warm_a.size() != std::size_t(8 * n)) state.resize(n);
  t45.resize(std::size_t(45 * 8 * n));
  const GridIdx g{grid.dims[0], grid.dims[1], grid.dims[2]};
  const std::vector<Vec3> snapshot = state.warm_a;
  EvalCounters ctr;
#pragma omp parallel for schedule(static)
  for (std::int64_t cell = 0; cell < n; ++cell) {
    const std::int64_t i = cell / (grid.dims[1] * grid.dims[2]);
    const std::int64_t j = (cell / grid.dims[2]) % grid.dims[1];
    const std::int64_t k = cell % grid.dims[2];
    for (int code = 0; code < 8; ++code) {
      const int l1 = code & 1, l2 = (code >> 1) & 1, l3 = (code >> 2) & 1;
      const Mat3 fd = gather_dfc(f, g, n, i, j, k, l1, l2, l3);
      const std::size_t dfc = std::size_t(cell) * 8 + std::size_t(code);
      Mat3 pd;
      Mat9 ad;
      eval_dfc(cm, snapshot, state, std::size_t(cell), dfc, true, fd, true, pd, &ad, ctr);
      pack45(ad, t45.data() + 45 * std::ptrdiff_t(dfc));
    }
  }
  return ctr.stats();
}

// dfmg.cpp:209-253
void dfmg_tangent_matvec(const std::vector<double>& t45, const Field9& x, Field9& y) {
  const SimGrid& grid = x.grid;
  const std::int64_t n = grid.cells();
  if (y.cells() != n) y = Field9(grid);
  const GridIdx g{grid.dims[0], grid.dims[1], grid.dims[2]};
#pragma omp parallel for collapse(2) schedule(static)
  for (std::int64_t i = 0; i < grid.dims[0]; ++i) {
    for (std::int64_t j = 0; j < grid.dims[1]; ++j) {
      for (std::int64_t k = 0; k < grid.dims[2]; ++k) {
        const std::size_t cell = grid.index(i, j, k);
        double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (const auto& cls : kClasses) {
          for (int code = 0; code < 8; ++code) {
            const int l1 = code & 1, l2 = (code >> 1) & 1, l3 = (code >> 2) & 1;
            const int l[3] = {l1, l2, l3};
            std::int64_t hi = i, hj = j, hk = k;
            if (cls.axis_a >= 0) {
              const int la = l[cls.axis_a], lb = l[cls.axis_b];
              if (cls.axis_a == 0) hi -= la;
              if (cls.axis_a == 1) hj -= la;
              if (cls.axis_b == 1) hj -= lb;
              if (cls.axis_b == 2) hk -= lb;
            }
            const std::size_t host = g.at(hi, hj, hk);
            const Mat3 xd = gather_dfc(x, g, n, hi, hj, hk, l1, l2, l3);
            const std::size_t dfc = host * 8 + std::size_t(code);
            const Mat9 ad = unpack45(t45.data() + 45 * std::ptrdiff_t(dfc));
            double yd[9];
            for (int r = 0; r < 9; ++r) {
              double v = 0.0;
              for (int c = 0; c < 9; ++c) v += ad(r, c) * xd.a[c];
              yd[r] = v;
            }
            for (int c = 0; c < cls.ncomp; ++c) {
              const int comp = cls.components[std::size_t(c)];
              acc[comp] += yd[comp];
            }
          }
        }
        for (int c = 0; c < 9; ++c) y.data[std::size_t(c) * std::size_t(n) + cell] = acc[c] / 8.0;
      }
    }
  }
}

// ------------------------------------------------------------------ solver
namespace {
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// solver.cpp:22-37
double rms9(const Field9& f) {
  const auto n = std::size_t(f.cells());
  double ss = 0.0;
  for (int c = 0; c < 9; ++c) ss += deterministic_sumsq(f.comp(c), n);
  return std::sqrt(ss / double(n));
}
double dot9(const Field9& a, const Field9& b) {
  return deterministic_dot(a.data.data(), b.data.data(), a.data.size());
}
void axpy(Field9& y, double a, const Field9& x) {
  const std::int64_t n = std::int64_t(y.data.size());
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < n; ++i) y.data[std::size_t(i)] += a * x.data[std::size_t(i)];
}

struct LsBudgetExhausted {};

// solver.cpp:41-122
class CellSolver {
 public:
  CellSolver(CellMaterials& cm, const SolverConfig& cfg)
      : t0_(Clock::now()), cm_(cm), cfg_(cfg), grid_(cm.grid()), green_(cfg.green, cm.grid()),
        fft_(cm.grid().dims, 9), p_(cm.grid()), proj_(cm.grid()) {
    double lo, hi;
    cm_.spectrum_bounds(Mat3::identity(), lo, hi);
    stress_floor_ = 1e-12 * std::max(hi, 1e-12);
    if (cfg_.eval == kDfmg) dfmg_state_.resize(grid_.cells());
    const char* lean = std::getenv("ORACLE_LEAN_TANGENTS");
    lean_ = lean && std::atoi(lean) != 0 && cfg_.eval != kDfmg;
  }
  StepReport run_step(Field9& f, const Mat3& fbar, double t0, double t1);
  const Field9& stress() const { return p_; }
  Mat3 pbar() const { return pbar_; }
  double alpha() const { return alpha_; }
  DfmgState& dfmg_state() { return dfmg_state_; }
  std::int64_t ls_total = 0;
  std::vector<double> ls_clock;  // end of every LS iteration (CPU-baseline timing)
  StepReport partial;  // the step cut short by the LS budget

 private:
  void project(const Field9& in, Field9& out) {
    if (cfg_.max_ls_iterations > 0 && ls_total >= cfg_.max_ls_iterations) throw LsBudgetExhausted{};
    ++ls_total;
    green_.project(in, out, fft_);
    ls_clock.push_back(seconds_since(t0_));
  }
  SweepStats eval_stress(const Field9& f) {
    if (cfg_.eval == kDfmg) return dfmg_stress(cm_, dfmg_state_, f, p_);
    return stress_sweep(cm_, f, p_, nullptr);
  }
  SweepStats eval_tangent(const Field9& f) {
    if (cfg_.eval == kDfmg) {
      const SweepStats s1 = dfmg_stress(cm_, dfmg_state_, f, p_);
      SweepStats s2 = dfmg_tangent_pass(cm_, dfmg_state_, f, tangents_);
      s2.inadmissible_cells += s1.inadmissible_cells;
      s2.laminate_failures = s1.laminate_failures;
      s2.back_projections = s1.back_projections;
      return s2;
    }
    tan_f_ = &f;
    return stress_sweep(cm_, f, p_, &tangents_, lean_);
  }
  void apply_tangent(const Field9& x, Field9& y) {
    if (cfg_.eval == kDfmg)
      dfmg_tangent_matvec(tangents_, x, y);
    else if (lean_)
      tangent_matvec_lean(cm_, tangents_, *tan_f_, x, y);
    else
      tangent_matvec(tangents_, x, y);
  }
  double residual_from_stress(Field9& out) {
    project(p_, out);
    pbar_ = p_.mean();
    return rms9(out) / std::max(norm(pbar_), stress_floor_);
  }
  void pick_alpha(const Mat3& fbar) {
    double lo, hi;
    cm_.spectrum_bounds(fbar, lo, hi);
    alpha_ = 0.5 * (std::max(lo, 0.0) + hi);
    if (!(alpha_ > 0.0)) alpha_ = std::max(hi, 1.0);
  }
  bool run_basic(Field9& f, const Mat3& fbar, StepReport& rep);
  bool run_newton(Field9& f, const Mat3& fbar, StepReport& rep);
  int cg_solve(Field9& x, const Field9& b, double tol_rel, bool& breakdown, StepReport& rep);

  Clock::time_point t0_;
  CellMaterials& cm_;
  SolverConfig cfg_;
  SimGrid grid_;
  GreenOperator green_;
  Fft3 fft_;
  Field9 p_, proj_;
  std::vector<double> tangents_;
  bool lean_ = false;             // ORACLE_LEAN_TANGENTS=1 (see stress_sweep)
  const Field9* tan_f_ = nullptr;  // F of the tangents (lean matvec)
  DfmgState dfmg_state_;
  Mat3 pbar_;
  double alpha_ = 1.0;
  double stress_floor_ = 1e-300;
};

// solver.cpp:124-164
bool CellSolver::run_basic(Field9& f, const Mat3& fbar, StepReport& rep) {
  pick_alpha(fbar);
  Field9 tau(grid_);
  for (int it = 1; it <= cfg_.max_outer; ++it) {
    rep.sweep = eval_stress(f);
    if (rep.sweep.inadmissible_cells > 0) return false;
    pbar_ = p_.mean();
    rep.pbar_history.push_back(pbar_);
    tau.data = p_.data;
    axpy(tau, -alpha_, f);
    project(tau, proj_);
    ++rep.ls_basic;
    const std::int64_t cells = f.cells();
    Field9 fnew(grid_);
    for (int c = 0; c < 9; ++c) {
      const double fb = fbar.a[c];
      const double* g = proj_.comp(c);
      double* out = fnew.comp(c);
#pragma omp parallel for schedule(static)
      for (std::int64_t i = 0; i < cells; ++i) out[i] = fb - g[i] / alpha_;
    }
    Field9 diff = fnew;
    axpy(diff, -1.0, f);
    const double resid = alpha_ * rms9(diff) / std::max(norm(pbar_), stress_floor_);
    rep.residuals.push_back(resid);
    rep.cg_iters.push_back(0);
    rep.outer_iters = it;
    if (cfg_.verbose) std::printf("  basic it %3d resid %.3e\n", it, resid);
    f.data.swap(fnew.data);
    f.pin_mean(fbar);
    if (rep.sweep.laminate_failures > 0 && resid <= cfg_.tol_equilibrium) return false;
    if (resid <= cfg_.tol_equilibrium) {
      rep.converged = true;
      return true;
    }
  }
  return false;
}

// solver.cpp:166-200
int CellSolver::cg_solve(Field9& x, const Field9& b, double tol_rel, bool& breakdown,
                         StepReport& rep) {
  breakdown = false;
  x = Field9(grid_);
  Field9 r = b;
  Field9 q(grid_), ap(grid_);
  double rr = dot9(r, r);
  const double bnorm = std::sqrt(rr);
  if (bnorm == 0.0) return 0;
  Field9 pdir = r;
  int it = 0;
  while (it < cfg_.cg_max) {
    apply_tangent(pdir, q);
    project(q, ap);
    ++rep.ls_cg;
    const double pap = dot9(pdir, ap);
    if (!(pap > 0.0)) {
      breakdown = true;
      return it;
    }
    const double step = rr / pap;
    axpy(x, step, pdir);
    axpy(r, -step, ap);
    ++it;
    const double rr_new = dot9(r, r);
    if (std::sqrt(rr_new) <= tol_rel * bnorm) return it;
    const double beta = rr_new / rr;
    rr = rr_new;
    const std::int64_t nn = std::int64_t(pdir.data.size());
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < nn; ++i)
      pdir.data[std::size_t(i)] = r.data[std::size_t(i)] + beta * pdir.data[std::size_t(i)];
  }
  return it;
}

// solver.cpp:202-259
bool CellSolver::run_newton(Field9& f, const Mat3& fbar, StepReport& rep) {
  Field9 b(grid_), x(grid_), ftrial(grid_);
  for (int it = 1; it <= cfg_.max_outer; ++it) {
    rep.sweep = eval_tangent(f);
    if (rep.sweep.inadmissible_cells > 0) return false;
    project(p_, b);
    ++rep.ls_residual;
    pbar_ = p_.mean();
    rep.pbar_history.push_back(pbar_);
    const double den = std::max(norm(pbar_), stress_floor_);
    const double resid = rms9(b) / den;
    rep.residuals.push_back(resid);
    rep.outer_iters = it;
    if (cfg_.verbose) std::printf("  newton it %3d resid %.3e\n", it, resid);
    if (resid <= cfg_.tol_equilibrium) {
      rep.cg_iters.push_back(0);
      rep.converged = rep.sweep.laminate_failures == 0;
      return rep.converged;
    }
    const std::int64_t nb = std::int64_t(b.data.size());
#pragma omp parallel for schedule(static)
    for (std::int64_t i = 0; i < nb; ++i) b.data[std::size_t(i)] = -b.data[std::size_t(i)];
    const double eta = std::max(std::min(cfg_.cg_tol, std::sqrt(resid)), 1e-8);
    bool breakdown = false;
    const int cg_its = cg_solve(x, b, eta, breakdown, rep);
    rep.cg_iters.push_back(cg_its);
    if (breakdown) {
      ++rep.cg_breakdowns;
      if (cg_its == 0) return false;
    }
    double s = 1.0;
    bool accepted = false;
    for (int ls = 0; ls < 10; ++ls) {
      ftrial.data = f.data;
      axpy(ftrial, s, x);
      ftrial.pin_mean(fbar);
      const SweepStats st = eval_stress(ftrial);
      if (st.inadmissible_cells == 0) {
        const double rtrial = residual_from_stress(proj_);
        ++rep.ls_trial;
        if (rtrial <= resid * (1.0 + 1e-12)) {
          accepted = true;
          break;
        }
      }
      s *= 0.5;
      ++rep.line_search_cuts;
    }
    if (!accepted) return false;
    f.data.swap(ftrial.data);
  }
  return false;
}

StepReport CellSolver::run_step(Field9& f, const Mat3& fbar, double t0, double t1) {
  const auto tic = Clock::now();
  StepReport rep;
  rep.t_start = t0;
  rep.t_end = t1;
  rep.fbar = fbar;
  bool ok = false;
  try {
    ok = cfg_.scheme == kBasic ? run_basic(f, fbar, rep) : run_newton(f, fbar, rep);
  } catch (const LsBudgetExhausted&) {
    // the partial step is reported (parity of budgeted runs, not reference
    // behaviour: the reference has no LS budget)
    rep.seconds = seconds_since(tic);
    partial = std::move(rep);
    throw;
  }
  rep.converged = ok;
  rep.seconds = seconds_since(tic);
  return rep;
}
}  // namespace

// solver.cpp:277-346
SolveResult solve(CellMaterials& cm, const Mat3& fbar_target, const SolverConfig& cfg) {
  if (cfg.eval == kDfmg && cfg.green != kStaggered)
    throw ConfigInvalid("solver: dfmg material evaluation requires the staggered Green operator");
  if (cfg.load_steps < 1) throw ConfigInvalid("solver: load_steps must be >= 1");
  if (!(cfg.tol_equilibrium > 0.0)) throw ConfigInvalid("solver: tol_equilibrium must be positive");
  if (!(det3(fbar_target) > 0.0)) throw InadmissibleMacroState("solve: det(fbar) <= 0");

  const auto tic = Clock::now();
  CellSolver solver(cm, cfg);
  SolveResult out;
  out.f = Field9(cm.grid());
  Mat3 h = sub(fbar_target, Mat3::identity());
  double t = 0.0;
  double dt = 1.0 / cfg.load_steps;
  Mat3 fbar_prev = Mat3::identity();
  out.f.fill(Mat3::identity());
  ConvergenceReport& report = out.report;
  report.success = true;
  try {
    while (t < 1.0 - 1e-12) {
      const double dt_try = std::min(dt, 1.0 - t);
      const Mat3 fbar = add(Mat3::identity(), scale(t + dt_try, h));
      Field9 backup_f = out.f;
      const std::vector<Vec3> backup_warm = cm.warm_all();
      const std::vector<Vec3> backup_dfmg = solver.dfmg_state().warm_a;
      out.f.pin_mean(fbar);
      StepReport rep = solver.run_step(out.f, fbar, t, t + dt_try);
      if (rep.converged) {
        report.steps.push_back(std::move(rep));
        t += dt_try;
        fbar_prev = fbar;
        continue;
      }
      out.f = std::move(backup_f);
      out.f.pin_mean(fbar_prev);
      cm.warm_all() = backup_warm;
      solver.dfmg_state().warm_a = backup_dfmg;
      ++report.bisections;
      if (report.bisections > cfg.max_bisections) {
        report.steps.push_back(std::move(rep));
        report.success = false;
        report.error = "LoadPathFailed: bisection budget exhausted";
        break;
      }
      dt = 0.5 * dt_try;
    }
  } catch (const LsBudgetExhausted&) {
    report.steps.push_back(std::move(solver.partial));
    report.success = false;
    report.error = "LsBudgetExhausted";
  }
  report.alpha = solver.alpha();
  report.ls_total = solver.ls_total;
  report.ls_clock = solver.ls_clock;
  report.seconds_total = seconds_since(tic);
  out.p = solver.stress();
  out.pbar = solver.pbar();
  return out;
}

}  // namespace oracle
