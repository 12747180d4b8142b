// TEST INFRASTRUCTURE ONLY (see oracle.hpp): tensor algebra, Neo-Hookean /
// linear laws and the finite-strain laminate kernel, restated from
// /root/reference/proj/src/{tensor,materials,laminate}.cpp.
#include <algorithm>
#include <limits>

#include "oracle.hpp"

namespace oracle {

Mat3 add(const Mat3& x, const Mat3& y) {
  Mat3 r;
  for (int i = 0; i < 9; ++i) r.a[i] = x.a[i] + y.a[i];
  return r;
}
Mat3 sub(const Mat3& x, const Mat3& y) {
  Mat3 r;
  for (int i = 0; i < 9; ++i) r.a[i] = x.a[i] - y.a[i];
  return r;
}
Mat3 scale(double s, const Mat3& x) {
  Mat3 r;
  for (int i = 0; i < 9; ++i) r.a[i] = s * x.a[i];
  return r;
}
Mat3 matmul(const Mat3& x, const Mat3& y) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r(i, j) = x(i, 0) * y(0, j) + x(i, 1) * y(1, j) + x(i, 2) * y(2, j);
  return r;
}
Mat3 transpose(const Mat3& x) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r(i, j) = x(j, i);
  return r;
}
Vec3 matvec(const Mat3& x, const Vec3& v) {
  Vec3 r;
  for (int i = 0; i < 3; ++i) r[i] = x(i, 0) * v[0] + x(i, 1) * v[1] + x(i, 2) * v[2];
  return r;
}
double norm(const Mat3& x) {
  double s = 0.0;
  for (int i = 0; i < 9; ++i) s += x.a[i] * x.a[i];
  return std::sqrt(s);
}
double norm(const Vec3& v) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }
double dot(const Vec3& x, const Vec3& y) { return x[0] * y[0] + x[1] * y[1] + x[2] * y[2]; }
double norm9(const Mat9& a) {
  double s = 0.0;
  for (int i = 0; i < 81; ++i) s += a.a[i] * a.a[i];
  return std::sqrt(s);
}
Vec3 mat3_col(const Mat3& m, int c) {
  Vec3 v;
  for (int i = 0; i < 3; ++i) v[i] = m(i, c);
  return v;
}

// Eigen's 3x3 determinant: cofactor expansion along the first column
// (Eigen/src/LU/Determinant.h bruteforce_det3_helper), used by
// Matrix3d::determinant() at materials.cpp:43 / laminate.cpp:127.
double det3(const Mat3& m) {
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) -
         m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2)) +
         m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2));
}

// tensor.cpp:49-63
Mat3 inv3(const Mat3& t) {
  const double d = det3(t);
  if (std::abs(d) <= 1e-300) throw SingularMatrix("inv3: |det| <= 1e-300");
  Mat3 adj;
  adj(0, 0) = t(1, 1) * t(2, 2) - t(1, 2) * t(2, 1);
  adj(0, 1) = t(0, 2) * t(2, 1) - t(0, 1) * t(2, 2);
  adj(0, 2) = t(0, 1) * t(1, 2) - t(0, 2) * t(1, 1);
  adj(1, 0) = t(1, 2) * t(2, 0) - t(1, 0) * t(2, 2);
  adj(1, 1) = t(0, 0) * t(2, 2) - t(0, 2) * t(2, 0);
  adj(1, 2) = t(0, 2) * t(1, 0) - t(0, 0) * t(1, 2);
  adj(2, 0) = t(1, 0) * t(2, 1) - t(1, 1) * t(2, 0);
  adj(2, 1) = t(0, 1) * t(2, 0) - t(0, 0) * t(2, 1);
  adj(2, 2) = t(0, 0) * t(1, 1) - t(0, 1) * t(1, 0);
  for (int i = 0; i < 9; ++i) adj.a[i] = adj.a[i] / d;
  return adj;
}

namespace {
constexpr int kPair[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
inline double mweight(int a) { return a < 3 ? 1.0 : kSqrt2; }
inline std::size_t idx81(int i, int j, int k, int l) {
  return std::size_t(((i * 3 + j) * 3 + k) * 3 + l);
}
}  // namespace

// tensor.cpp:101-116
std::array<double, 81> mandel_to_full(const Mat6& c) {
  std::array<double, 81> f{};
  for (int a = 0; a < 6; ++a) {
    const int i = kPair[a][0], j = kPair[a][1];
    for (int b = 0; b < 6; ++b) {
      const int k = kPair[b][0], l = kPair[b][1];
      const double v = c(a, b) / (mweight(a) * mweight(b));
      f[idx81(i, j, k, l)] = v;
      f[idx81(j, i, k, l)] = v;
      f[idx81(i, j, l, k)] = v;
      f[idx81(j, i, l, k)] = v;
    }
  }
  return f;
}

// tensor.cpp:118-125
Mat6 full_to_mandel(const std::array<double, 81>& f) {
  Mat6 c;
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b)
      c(a, b) = mweight(a) * mweight(b) *
                f[idx81(kPair[a][0], kPair[a][1], kPair[b][0], kPair[b][1])];
  return c;
}

// tensor.cpp:127-136
Mat9 mandel_to_mat9(const Mat6& c) {
  const auto f = mandel_to_full(c);
  Mat9 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) m(3 * i + j, 3 * k + l) = f[idx81(i, j, k, l)];
  return m;
}

// ------------------------------------------------------------ eigen-solvers
namespace {
// One Jacobi rotation zeroing a[p][q] of a symmetric n x n matrix (row-major)
// and accumulating it into the eigenvector matrix v (columns).
void jacobi_rotate(int n, double* a, double* v, int p, int q) {
  const double apq = a[p * n + q];
  const double app = a[p * n + p], aqq = a[q * n + q];
  const double g = 100.0 * std::fabs(apq);
  if (std::fabs(app) + g == std::fabs(app) && std::fabs(aqq) + g == std::fabs(aqq)) {
    a[p * n + q] = 0.0;
    a[q * n + p] = 0.0;
    return;
  }
  const double h = aqq - app;
  double t;
  if (std::fabs(h) + g == std::fabs(h)) {
    t = apq / h;
  } else {
    const double theta = 0.5 * h / apq;
    t = 1.0 / (std::fabs(theta) + std::sqrt(1.0 + theta * theta));
    if (theta < 0.0) t = -t;
  }
  const double c = 1.0 / std::sqrt(1.0 + t * t);
  const double s = t * c;
  const double tau = s / (1.0 + c);
  a[p * n + p] = app - t * apq;
  a[q * n + q] = aqq + t * apq;
  a[p * n + q] = 0.0;
  a[q * n + p] = 0.0;
  for (int r = 0; r < n; ++r) {
    if (r == p || r == q) continue;
    const double gr = a[r * n + p], hr = a[r * n + q];
    const double np = gr - s * (hr + gr * tau);
    const double nq = hr + s * (gr - hr * tau);
    a[r * n + p] = np;
    a[p * n + r] = np;
    a[r * n + q] = nq;
    a[q * n + r] = nq;
  }
  for (int r = 0; r < n; ++r) {
    const double gr = v[r * n + p], hr = v[r * n + q];
    v[r * n + p] = gr - s * (hr + gr * tau);
    v[r * n + q] = hr + s * (gr - hr * tau);
  }
}

void jacobi(int n, double* a, double* v) {
  for (int i = 0; i < n * n; ++i) v[i] = 0.0;
  for (int i = 0; i < n; ++i) v[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool any = false;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q)
        if (a[p * n + q] != 0.0) any = true;
    if (!any) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q)
        if (a[p * n + q] != 0.0) jacobi_rotate(n, a, v, p, q);
  }
}

void sort_ascending(int n, double* lam, double* vec) {
  for (int i = 0; i < n; ++i) {
    int m = i;
    for (int j = i + 1; j < n; ++j)
      if (lam[j] < lam[m]) m = j;
    if (m != i) {
      std::swap(lam[i], lam[m]);
      for (int r = 0; r < n; ++r) std::swap(vec[r * n + i], vec[r * n + m]);
    }
  }
}
}  // namespace

void sym_eig(int n, const double* m, double* lam, double* vec) {
  std::vector<double> a(m, m + n * n);
  jacobi(n, a.data(), vec);
  for (int i = 0; i < n; ++i) lam[i] = a[i * n + i];
  sort_ascending(n, lam, vec);
}

void sym_eig3_jacobi(const double m[9], double lam[3], double vec[9]) {
  double a[9];
  for (int i = 0; i < 9; ++i) a[i] = m[i];
  jacobi(3, a, vec);
  for (int i = 0; i < 3; ++i) lam[i] = a[4 * i];
  sort_ascending(3, lam, vec);
}

// -------------------------------------------------------------- materials
Law Law::neo_hookean(double lambda, double mu) {
  Law l;
  l.kind = kNeoHookean;
  l.lambda = lambda;
  l.mu = mu;
  return l;
}

// materials.cpp:11-20
Law Law::neo_hookean_enu(double e, double nu) {
  if (!(e > 0.0) || !(nu > -1.0) || !(nu < 0.5))
    throw std::runtime_error("neo_hookean: require E > 0 and -1 < nu < 0.5");
  return neo_hookean(e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), e / (2.0 * (1.0 + nu)));
}

// materials.cpp:22-30
Mat6 Law::iso_mandel(double lambda, double mu) {
  Mat6 c;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) c(i, j) = lambda;
    c(i, i) += 2.0 * mu;
    c(i + 3, i + 3) = 2.0 * mu;
  }
  return c;
}

Law Law::linear(const Mat6& c6) {
  Law l;
  l.kind = kLinear;
  l.c6 = c6;
  l.a9 = mandel_to_mat9(c6);
  return l;
}

namespace {
struct HyperelasticEval {
  Mat3 pk2;
  Mat6 stiffness;
};

// materials.cpp:41-66 (energy omitted: not on the solver path)
bool neo_hookean(const Mat3& f, double lambda, double mu, HyperelasticEval& out) {
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  const Mat3 c = matmul(transpose(f), f);
  const Mat3 ci = inv3(c);
  const double lnj = std::log(j);
  const double ll = lambda * lnj;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      out.pk2(i, k) = ll * ci(i, k) + mu * ((i == k ? 1.0 : 0.0) - ci(i, k));
  const double g = mu - lambda * lnj;
  std::array<double, 81> full{};
  for (int i = 0; i < 3; ++i)
    for (int jj = 0; jj < 3; ++jj)
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l)
          full[idx81(i, jj, k, l)] = lambda * ci(i, jj) * ci(k, l) +
                                     g * (ci(i, k) * ci(jj, l) + ci(i, l) * ci(jj, k));
  out.stiffness = full_to_mandel(full);
  return true;
}

// materials.cpp:68-95
Mat9 tangent_pk1(const Mat3& f, const Mat3& s, const Mat6& c) {
  const auto cf = mandel_to_full(c);
  std::array<double, 81> t1{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int l = 0; l < 3; ++l)
        for (int q = 0; q < 3; ++q) {
          double v = 0.0;
          for (int m = 0; m < 3; ++m) v += f(i, m) * cf[idx81(m, j, l, q)];
          t1[idx81(i, j, l, q)] = v;
        }
  Mat9 a;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) {
          double v = (i == k) ? s(j, l) : 0.0;
          for (int q = 0; q < 3; ++q) v += t1[idx81(i, j, l, q)] * f(k, q);
          a(3 * i + j, 3 * k + l) = v;
        }
  return a;
}

// materials.cpp:132-137: P = C : sym(F - I) through the Mandel maps
Mat3 linear_eval(const Law& law, const Mat3& f) {
  Mat3 eps;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      eps(i, j) = 0.5 * (f(i, j) + f(j, i)) - (i == j ? 1.0 : 0.0);
  double v[6] = {eps(0, 0), eps(1, 1), eps(2, 2), kSqrt2 * eps(0, 1),
                 kSqrt2 * eps(0, 2), kSqrt2 * eps(1, 2)};
  double s[6];
  for (int a = 0; a < 6; ++a) {
    double acc = 0.0;
    for (int b = 0; b < 6; ++b) acc += law.c6(a, b) * v[b];
    s[a] = acc;
  }
  Mat3 p;
  p(0, 0) = s[0];
  p(1, 1) = s[1];
  p(2, 2) = s[2];
  p(0, 1) = p(1, 0) = s[3] / kSqrt2;
  p(0, 2) = p(2, 0) = s[4] / kSqrt2;
  p(1, 2) = p(2, 1) = s[5] / kSqrt2;
  return p;
}
}  // namespace

// materials.cpp:97-110, 132-142
bool law_eval(const Law& law, const Mat3& f, Mat3& p) {
  if (law.kind == kLinear) {
    p = linear_eval(law, f);
    return true;
  }
  HyperelasticEval r;
  if (!neo_hookean(f, law.lambda, law.mu, r)) return false;
  p = matmul(f, r.pk2);
  return true;
}

bool law_eval_tangent(const Law& law, const Mat3& f, Mat3& p, Mat9& a) {
  if (law.kind == kLinear) {
    p = linear_eval(law, f);
    a = law.a9;
    return true;
  }
  HyperelasticEval r;
  if (!neo_hookean(f, law.lambda, law.mu, r)) return false;
  p = matmul(f, r.pk2);
  a = tangent_pk1(f, r.pk2, r.stiffness);
  return true;
}

// materials.cpp:112-125, 144-150
void law_spectrum_bounds(const Law& law, const Mat3& f, double& lo, double& hi) {
  if (law.kind == kLinear) {
    double lam[6], vec[36];
    sym_eig(6, law.c6.a, lam, vec);
    lo = std::min(0.0, lam[0]);
    hi = lam[5];
    return;
  }
  Mat3 p;
  Mat9 a;
  if (law_eval_tangent(law, f, p, a)) {
    Mat9 sym;
    for (int i = 0; i < 9; ++i)
      for (int j = 0; j < 9; ++j) sym(i, j) = 0.5 * (a(i, j) + a(j, i));
    double lam[9], vec[81];
    sym_eig(9, sym.a, lam, vec);
    lo = lam[0];
    hi = lam[8];
  } else {
    lo = law.mu;
    hi = law.lambda + 2.0 * law.mu;
  }
}

// --------------------------------------------------------------- laminate
// laminate.cpp:28-34
ComboMeta ComboMeta::make(const Vec3& n, double cp) {
  if (!(cp > 0.0) || !(cp < 1.0))
    throw std::runtime_error("ComboMeta: volume fraction must lie in (0,1)");
  const double len = norm(n);
  if (!(len > 0.0)) throw std::runtime_error("ComboMeta: zero normal");
  ComboMeta m;
  for (int i = 0; i < 3; ++i) m.normal[i] = n[i] / len;
  m.c_plus = cp;
  m.c_minus = 1.0 - cp;
  return m;
}

// laminate.cpp:125-136
AdmissibleBounds admissibility_bounds(const Mat3& f_box, const ComboMeta& meta) {
  if (!(det3(f_box) > 0.0))
    throw InadmissibleMacroState("admissibility_bounds: det(F_box) <= 0");
  const Vec3 w = matvec(transpose(inv3(f_box)), meta.normal);
  const double len = norm(w);
  AdmissibleBounds b;
  for (int i = 0; i < 3; ++i) b.m_beta[i] = w[i] / len;
  b.beta_plus = -meta.c_plus / len;
  b.beta_minus = meta.c_minus / len;
  return b;
}

// laminate.cpp:138-144
Vec3 back_project(const Vec3& a1, const Vec3& a0, const AdmissibleBounds& b) {
  const double beta1 = dot(a1, b.m_beta);
  const double beta0 = dot(a0, b.m_beta);
  const double beta_c = (beta1 <= b.beta_plus) ? b.beta_plus : b.beta_minus;
  const double beta_star = 0.5 * (beta0 + beta_c);
  Vec3 r;
  for (int i = 0; i < 3; ++i) r[i] = a1[i] + (beta_star - beta1) * b.m_beta[i];
  return r;
}

namespace {
// Delta = D^T M D for the 9x3 jump matrix D[(i,J),k] = delta_ik N_J
// (tensor.cpp:138-142), evaluated as the dense (D^T M) D product.
void dtmd(const Mat9& m, const Vec3& n, double out[9]) {
  double d[9][3];
  for (int r = 0; r < 9; ++r)
    for (int k = 0; k < 3; ++k) d[r][k] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) d[3 * i + j][i] = n[j];
  double t[3][9];
  for (int k = 0; k < 3; ++k)
    for (int c = 0; c < 9; ++c) {
      double v = 0.0;
      for (int r = 0; r < 9; ++r) v += d[r][k] * m(r, c);
      t[k][c] = v;
    }
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) {
      double v = 0.0;
      for (int c = 0; c < 9; ++c) v += t[k][c] * d[c][l];
      out[3 * k + l] = v;
    }
}

// Eigen::FullPivLU<Matrix3d> (laminate.cpp:20-24, 215-217): complete pivoting,
// rank test against eps * size * max pivot, solve P^-1 L U Q^-1.
struct FullPivLU3 {
  double lu[9];
  int rowt[3], colt[3];
  int nonzero = 3;
  double maxpivot = 0.0;
  explicit FullPivLU3(const double m[9]) {
    for (int i = 0; i < 9; ++i) lu[i] = m[i];
    for (int k = 0; k < 3; ++k) {
      // maxCoeff visitor over the bottom-right corner, column-major order
      double biggest = -1.0;
      int br = k, bc = k;
      for (int c = k; c < 3; ++c)
        for (int r = k; r < 3; ++r) {
          const double v = std::fabs(lu[3 * r + c]);
          if (v > biggest) {
            biggest = v;
            br = r;
            bc = c;
          }
        }
      if (biggest == 0.0) {
        nonzero = k;
        for (int i = k; i < 3; ++i) rowt[i] = colt[i] = i;
        break;
      }
      if (biggest > maxpivot) maxpivot = biggest;
      rowt[k] = br;
      colt[k] = bc;
      if (br != k)
        for (int c = 0; c < 3; ++c) std::swap(lu[3 * k + c], lu[3 * br + c]);
      if (bc != k)
        for (int r = 0; r < 3; ++r) std::swap(lu[3 * r + k], lu[3 * r + bc]);
      for (int r = k + 1; r < 3; ++r) lu[3 * r + k] /= lu[3 * k + k];
      for (int r = k + 1; r < 3; ++r)
        for (int c = k + 1; c < 3; ++c) lu[3 * r + c] -= lu[3 * r + k] * lu[3 * k + c];
    }
  }
  bool invertible() const {
    const double thr = std::fabs(maxpivot) * (std::numeric_limits<double>::epsilon() * 3.0);
    int rank = 0;
    for (int i = 0; i < nonzero; ++i) rank += std::fabs(lu[4 * i]) > thr ? 1 : 0;
    return rank == 3;
  }
  Vec3 solve(const Vec3& b) const {
    double c[3] = {b[0], b[1], b[2]};
    for (int k = 0; k < 3; ++k) std::swap(c[k], c[rowt[k]]);
    for (int r = 1; r < 3; ++r)
      for (int k = 0; k < r; ++k) c[r] -= lu[3 * r + k] * c[k];
    for (int r = 2; r >= 0; --r) {
      for (int k = r + 1; k < 3; ++k) c[r] -= lu[3 * r + k] * c[k];
      c[r] /= lu[4 * r];
    }
    for (int k = 2; k >= 0; --k) std::swap(c[k], c[colt[k]]);
    Vec3 x;
    for (int i = 0; i < 3; ++i) x[i] = c[i];
    return x;
  }
  void inverse(double out[9]) const {
    for (int col = 0; col < 3; ++col) {
      Vec3 e;
      e[col] = 1.0;
      const Vec3 x = solve(e);
      for (int r = 0; r < 3; ++r) out[3 * r + col] = x[r];
    }
  }
};
}  // namespace

// laminate.cpp:146-156
Mat9 effective_tangent(const Mat9& ap, const Mat9& am, const ComboMeta& meta) {
  Mat9 m;
  for (int i = 0; i < 81; ++i) m.a[i] = ap.a[i] / meta.c_plus + am.a[i] / meta.c_minus;
  double delta[9];
  dtmd(m, meta.normal, delta);
  FullPivLU3 lu(delta);
  if (!lu.invertible()) throw SingularMatrix("effective_tangent: singular Hessian");
  double dinv[9];
  lu.inverse(dinv);
  // mm = (ap - am) D  (9x3)
  double mm[9][3];
  for (int r = 0; r < 9; ++r)
    for (int k = 0; k < 3; ++k) {
      double v = 0.0;
      for (int c = 0; c < 9; ++c) {
        const int i = c / 3, j = c % 3;
        const double dck = (i == k) ? meta.normal[j] : 0.0;
        v += (ap(r, c) - am(r, c)) * dck;
      }
      mm[r][k] = v;
    }
  // t = mm * dinv (9x3)
  double t[9][3];
  for (int r = 0; r < 9; ++r)
    for (int k = 0; k < 3; ++k) {
      double v = 0.0;
      for (int l = 0; l < 3; ++l) v += mm[r][l] * dinv[3 * l + k];
      t[r][k] = v;
    }
  Mat9 out;
  for (int r = 0; r < 9; ++r)
    for (int c = 0; c < 9; ++c) {
      double corr = 0.0;
      for (int k = 0; k < 3; ++k) corr += t[r][k] * mm[c][k];
      out(r, c) = (meta.c_plus * ap(r, c) + meta.c_minus * am(r, c)) - corr;
    }
  return out;
}

// laminate.cpp:158-272
LaminateSolution finite_strain_solve(const Mat3& f_box, const Law& mat_plus,
                                     const Law& mat_minus, const ComboMeta& meta,
                                     const Vec3& a0, const LaminateOptions& opt,
                                     bool want_tangent) {
  LaminateSolution sol;
  JumpVectorState& st = sol.state;
  const AdmissibleBounds bounds = admissibility_bounds(f_box, meta);
  const Vec3& n = meta.normal;

  Vec3 a = bounds.admissible(a0) ? a0 : Vec3();
  Mat3 fp, fm, pp, pm;
  Mat9 ap, am;
  auto update_phases = [&](const Vec3& jump) -> bool {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const double an = jump[i] * n[j];
        fp(i, j) = f_box(i, j) + an / meta.c_plus;
        fm(i, j) = f_box(i, j) - an / meta.c_minus;
      }
    return law_eval_tangent(mat_plus, fp, pp, ap) && law_eval_tangent(mat_minus, fm, pm, am);
  };
  auto traction_scale = [&]() {
    return std::max({norm(matvec(pp, n)), norm(matvec(pm, n)), opt.stress_floor});
  };
  auto noise_floor = [&]() {
    constexpr double eps = 2.220446049250313e-16;
    return 16.0 * eps * std::max(norm9(ap) * norm(fp), norm9(am) * norm(fm));
  };
  auto traction_jump = [&]() {
    const Vec3 tp = matvec(pp, n), tm = matvec(pm, n);
    Vec3 r;
    for (int i = 0; i < 3; ++i) r[i] = tp[i] - tm[i];
    return r;
  };

  if (!update_phases(a)) {
    st.converged = false;
    st.residual = std::numeric_limits<double>::infinity();
    return sol;
  }
  Vec3 f = traction_jump();
  double best_res = norm(f);
  Vec3 best_a = a;
  st.residual = best_res;
  st.residual_rel = best_res / std::max(traction_scale(), 1e-300);
  auto converged = [&]() {
    return norm(f) <= opt.tol_abs + noise_floor() +
                          opt.tol_rel * std::max(traction_scale(), 1e-300);
  };

  int k = 0;
  bool ok = converged();
  while (!ok && k < opt.max_iter) {
    Mat9 m;
    for (int i = 0; i < 81; ++i) m.a[i] = ap.a[i] / meta.c_plus + am.a[i] / meta.c_minus;
    double delta[9];
    dtmd(m, n, delta);
    FullPivLU3 lu(delta);
    if (!lu.invertible()) break;
    const Vec3 step = lu.solve(f);
    Vec3 a1;
    for (int i = 0; i < 3; ++i) a1[i] = a[i] - step[i];
    ++k;
    if (!bounds.admissible(a1)) {
      if (st.first_inadmissible_iter < 0) st.first_inadmissible_iter = k;
      if (!opt.back_projection) {
        st.iterations = k;
        st.converged = false;
        st.a = a;
        st.residual = norm(f);
        st.residual_rel = st.residual / std::max(traction_scale(), 1e-300);
        return sol;
      }
      a1 = back_project(a1, a, bounds);
      ++st.back_projections;
    }
    a = a1;
    if (!update_phases(a)) break;
    f = traction_jump();
    if (norm(f) < best_res) {
      best_res = norm(f);
      best_a = a;
    }
    ok = converged();
  }
  if (!ok) {
    if (best_a[0] != a[0] || best_a[1] != a[1] || best_a[2] != a[2]) {
      a = best_a;
      update_phases(a);
      f = traction_jump();
    }
  }
  st.a = a;
  st.converged = ok;
  st.iterations = k;
  st.residual = norm(f);
  st.residual_rel = st.residual / std::max(traction_scale(), 1e-300);

  LaminateResult& r = sol.result;
  r.f_plus = fp;
  r.f_minus = fm;
  r.p_plus = pp;
  r.p_minus = pm;
  for (int i = 0; i < 9; ++i) r.p_box.a[i] = meta.c_plus * pp.a[i] + meta.c_minus * pm.a[i];
  const Mat3 s = matmul(inv3(f_box), r.p_box);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.s_box(i, j) = 0.5 * (s(i, j) + s(j, i));
  const Vec3 tp = matvec(pp, n), tm = matvec(pm, n);
  for (int i = 0; i < 3; ++i) r.traction[i] = ok ? tp[i] : 0.5 * (tp[i] + tm[i]);
  if (want_tangent) {
    r.a_box = effective_tangent(ap, am, meta);
    r.tangent_valid = true;
  }
  return sol;
}

}  // namespace oracle
