// B200 material point: compressible Neo-Hookean phases in closed form and the
// finite-strain rank-1 laminate (ComBo boxel) solved per thread.
//
// Reference semantics followed (file:line in /root/reference/proj):
//   NeoHookeanLaw::eval / eval_tangent     src/materials.cpp:41-110
//   LinearElasticLaw                        src/materials.cpp:127-150
//   admissibility_bounds / back_project     src/laminate.cpp:125-144
//   finite_strain_solve (Newton + best it.) src/laminate.cpp:158-272
//   effective_tangent (as a matvec)         src/laminate.cpp:146-156
//
// The reference builds S, the Mandel stiffness and the 9x9 first elasticity
// tensor explicitly. Here everything is closed form in G = F^{-T}:
//   P      = mu F + (lambda lnJ - mu) G
//   A : X  = mu X + lambda (G:X) G + beta G X^T G,   beta = mu - lambda lnJ
//   |A|_F^2 = 9mu^2 + (lambda^2+beta^2)|G|^4 + 2mu(lambda+beta)|G|^2
//             + 2 lambda beta |G G^T|^2                (noise floor, :186-190)
//   D^T A D = mu |N|^2 I + (lambda + beta) (G N)(G N)^T  (Newton Hessian)
// which are the same tensors to rounding, at a fraction of the registers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace combo_dev {

struct LawP {
  int kind;  // 0 neo-hookean, 1 linear (tests; materials.hpp:88-107)
  double lambda, mu;
  const double* a9;  // linear law: mandel_to_mat9(C), device memory
};

struct LamP {
  double tol_abs, tol_rel, stress_floor;
  int max_iter;
  int back_projection;
};

struct MatParams {
  LawP law[2];  // [0] matrix ("-"), [1] inclusion ("+")
  LamP lam;
};

// ------------------------------------------------------------ 3x3 helpers
__host__ __device__ inline double det3(const double* m) {
  // Eigen 3x3 cofactor order (materials.cpp:43 via Matrix3d::determinant)
  return m[0] * (m[4] * m[8] - m[7] * m[5]) - m[3] * (m[1] * m[8] - m[7] * m[2]) +
         m[6] * (m[1] * m[5] - m[4] * m[2]);
}

// G = F^{-T} from the adjugate; returns det
__device__ inline double inv_transpose(const double* f, double* g) {
  const double d = det3(f);
  const double id = 1.0 / d;
  // adj(F)_ij = cof(F)_ji ; G_ij = (F^{-1})_ji = adj_ji / d = cof_ij / d
  g[0] = (f[4] * f[8] - f[5] * f[7]) * id;
  g[1] = (f[5] * f[6] - f[3] * f[8]) * id;
  g[2] = (f[3] * f[7] - f[4] * f[6]) * id;
  g[3] = (f[2] * f[7] - f[1] * f[8]) * id;
  g[4] = (f[0] * f[8] - f[2] * f[6]) * id;
  g[5] = (f[1] * f[6] - f[0] * f[7]) * id;
  g[6] = (f[1] * f[5] - f[2] * f[4]) * id;
  g[7] = (f[2] * f[3] - f[0] * f[5]) * id;
  g[8] = (f[0] * f[4] - f[1] * f[3]) * id;
  return d;
}

__device__ inline double sq9(const double* a) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) s += a[i] * a[i];
  return s;
}

// ------------------------------------------------------------- phase laws
// Phase state of one Neo-Hookean evaluation, enough for P, A:X, |A|.
struct NhState {
  double g[9];  // F^{-T}
  double lnj;
};

// NeoHookeanLaw::eval (materials.cpp:97-102); false when det F <= 0.
__device__ inline bool nh_eval(const LawP& L, const double* f, double* p, NhState& s) {
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  inv_transpose(f, s.g);
  s.lnj = log(j);
  const double c = L.lambda * s.lnj - L.mu;
#pragma unroll
  for (int i = 0; i < 9; ++i) p[i] = L.mu * f[i] + c * s.g[i];
  return true;
}

// y = A : x for a Neo-Hookean phase at state s
__device__ inline void nh_apply(const LawP& L, const NhState& s, const double* x, double* y) {
  const double beta = L.mu - L.lambda * s.lnj;
  double gx = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) gx += s.g[i] * x[i];
  // t = G x^T  (t_iK = sum_L G_iL x_KL)
  double t[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      t[3 * i + k] = s.g[3 * i] * x[3 * k] + s.g[3 * i + 1] * x[3 * k + 1] + s.g[3 * i + 2] * x[3 * k + 2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double tg = t[3 * i] * s.g[j] + t[3 * i + 1] * s.g[3 + j] + t[3 * i + 2] * s.g[6 + j];
      y[3 * i + j] = L.mu * x[3 * i + j] + L.lambda * gx * s.g[3 * i + j] + beta * tg;
    }
}

__device__ inline double nh_tangent_norm(const LawP& L, const NhState& s) {
  const double beta = L.mu - L.lambda * s.lnj;
  const double g2 = sq9(s.g);
  double ggt2 = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double v = s.g[3 * i] * s.g[3 * k] + s.g[3 * i + 1] * s.g[3 * k + 1] + s.g[3 * i + 2] * s.g[3 * k + 2];
      ggt2 += v * v;
    }
  const double v = 9.0 * L.mu * L.mu + (L.lambda * L.lambda + beta * beta) * g2 * g2 +
                   2.0 * L.mu * (L.lambda + beta) * g2 + 2.0 * L.lambda * beta * ggt2;
  return sqrt(fmax(v, 0.0));
}

// D^T A D (3x3, row major) for normal n
__device__ inline void nh_dtad(const LawP& L, const NhState& s, const double* n, double* q) {
  const double beta = L.mu - L.lambda * s.lnj;
  double m[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) m[i] = s.g[3 * i] * n[0] + s.g[3 * i + 1] * n[1] + s.g[3 * i + 2] * n[2];
  const double nn = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
  const double lb = L.lambda + beta;
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int l = 0; l < 3; ++l) q[3 * k + l] = (k == l ? L.mu * nn : 0.0) + lb * m[k] * m[l];
}

// Generic law wrappers (linear elasticity only for the reference's tests:
// P = C : sym(F - I), materials.cpp:132-142)
__device__ inline bool law_eval(const LawP& L, const double* f, double* p, NhState& s) {
  if (L.kind == 0) return nh_eval(L, f, p, s);
  double e[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) e[3 * i + j] = 0.5 * (f[3 * i + j] + f[3 * j + i]) - (i == j ? 1.0 : 0.0);
  for (int r = 0; r < 9; ++r) {
    double v = 0.0;
    for (int c = 0; c < 9; ++c) v += L.a9[9 * r + c] * e[c];
    p[r] = v;
  }
  return true;
}
// The tangent state only (G, ln J) of law_eval: bitwise the same state
// without forming P (the CG matvec needs A, not P).
__device__ inline bool law_state(const LawP& L, const double* f, NhState& s) {
  if (L.kind != 0) return true;
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  inv_transpose(f, s.g);
  s.lnj = log(j);
  return true;
}
__device__ inline void law_apply(const LawP& L, const NhState& s, const double* x, double* y) {
  if (L.kind == 0) {
    nh_apply(L, s, x, y);
    return;
  }
  for (int r = 0; r < 9; ++r) {
    double v = 0.0;
    for (int c = 0; c < 9; ++c) v += L.a9[9 * r + c] * x[c];
    y[r] = v;
  }
}
__device__ inline double law_tangent_norm(const LawP& L, const NhState& s) {
  if (L.kind == 0) return nh_tangent_norm(L, s);
  return sqrt(sq9(L.a9) + sq9(L.a9 + 9) + sq9(L.a9 + 18) + sq9(L.a9 + 27) + sq9(L.a9 + 36) +
              sq9(L.a9 + 45) + sq9(L.a9 + 54) + sq9(L.a9 + 63) + sq9(L.a9 + 72));
}
__device__ inline void law_dtad(const LawP& L, const NhState& s, const double* n, double* q) {
  if (L.kind == 0) {
    nh_dtad(L, s, n, q);
    return;
  }
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) {
      double v = 0.0;
      for (int J = 0; J < 3; ++J)
        for (int Lc = 0; Lc < 3; ++Lc) v += n[J] * L.a9[9 * (3 * k + J) + 3 * l + Lc] * n[Lc];
      q[3 * k + l] = v;
    }
}

// ---------------------------------------------------------- 3x3 full-pivot LU
// Eigen::FullPivLU<Matrix3d> semantics (laminate.cpp:215-217): complete
// pivoting, rank test against eps * 3 * max pivot.
struct Lu3 {
  double lu[9];
  int rt[3], ct[3];
  bool ok;
  __device__ inline void factor(const double* m) {
#pragma unroll
    for (int i = 0; i < 9; ++i) lu[i] = m[i];
    double maxpivot = 0.0;
    int nonzero = 3;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double big = -1.0;
      int br = k, bc = k;
      for (int c = k; c < 3; ++c)
        for (int r = k; r < 3; ++r) {
          const double v = fabs(lu[3 * r + c]);
          if (v > big) {
            big = v;
            br = r;
            bc = c;
          }
        }
      if (big == 0.0) {
        if (nonzero == 3) nonzero = k;
        for (int i = k; i < 3; ++i) rt[i] = ct[i] = i;
        break;
      }
      maxpivot = fmax(maxpivot, big);
      rt[k] = br;
      ct[k] = bc;
      if (br != k)
        for (int c = 0; c < 3; ++c) {
          const double t = lu[3 * k + c];
          lu[3 * k + c] = lu[3 * br + c];
          lu[3 * br + c] = t;
        }
      if (bc != k)
        for (int r = 0; r < 3; ++r) {
          const double t = lu[3 * r + k];
          lu[3 * r + k] = lu[3 * r + bc];
          lu[3 * r + bc] = t;
        }
      for (int r = k + 1; r < 3; ++r) lu[3 * r + k] /= lu[3 * k + k];
      for (int r = k + 1; r < 3; ++r)
        for (int c = k + 1; c < 3; ++c) lu[3 * r + c] -= lu[3 * r + k] * lu[3 * k + c];
    }
    const double thr = maxpivot * (2.220446049250313e-16 * 3.0);
    int rank = 0;
    for (int i = 0; i < 3; ++i) rank += (i < nonzero && fabs(lu[4 * i]) > thr) ? 1 : 0;
    ok = rank == 3;
  }
  __device__ inline void solve(const double* b, double* x) const {
    double c[3] = {b[0], b[1], b[2]};
    for (int k = 0; k < 3; ++k) {
      const double t = c[k];
      c[k] = c[rt[k]];
      c[rt[k]] = t;
    }
    c[1] -= lu[3] * c[0];
    c[2] -= lu[6] * c[0] + lu[7] * c[1];
    c[2] /= lu[8];
    c[1] = (c[1] - lu[5] * c[2]) / lu[4];
    c[0] = (c[0] - lu[1] * c[1] - lu[2] * c[2]) / lu[0];
    for (int k = 2; k >= 0; --k) {
      const double t = c[k];
      c[k] = c[ct[k]];
      c[ct[k]] = t;
    }
    x[0] = c[0];
    x[1] = c[1];
    x[2] = c[2];
  }
};

// ----------------------------------------------------------------- laminate
struct LamResult {
  double p[9];
  double a[3];
  int iterations;
  int back_projections;
  bool converged;
  bool inadmissible;  // det F_box <= 0 (InadmissibleMacroState)
};

__device__ inline void form_phases(const double* fbox, const double* n, double cp, double cm,
                                   const double* a, double* fp, double* fm) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double an = a[i] * n[j];
      fp[3 * i + j] = fbox[3 * i + j] + an / cp;
      fm[3 * i + j] = fbox[3 * i + j] - an / cm;
    }
}

__device__ inline void mat_n(const double* p, const double* n, double* t) {
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = p[3 * i] * n[0] + p[3 * i + 1] * n[1] + p[3 * i + 2] * n[2];
}
__device__ inline double norm3(const double* v) { return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

// finite_strain_solve (laminate.cpp:158-272) for phases (+ = inclusion,
// - = matrix); warm start a0 used only if admissible (:169).
__device__ inline void laminate_solve(const MatParams& M, const double* fbox, const double* n,
                                      double cp, double cm, const double* a0, LamResult& R) {
  const LawP& Lp = M.law[1];
  const LawP& Lm = M.law[0];
  R.iterations = 0;
  R.back_projections = 0;
  R.converged = false;
  R.inadmissible = false;
  // admissibility_bounds (:125-136)
  const double jb = det3(fbox);
  if (!(jb > 0.0)) {
    R.inadmissible = true;
#pragma unroll
    for (int i = 0; i < 9; ++i) R.p[i] = 0.0;
    R.a[0] = a0[0];
    R.a[1] = a0[1];
    R.a[2] = a0[2];
    return;
  }
  double mb[3];
  {
    double g[9];
    inv_transpose(fbox, g);
    mat_n(g, n, mb);  // F^{-T} N
  }
  const double len = norm3(mb);
  mb[0] /= len;
  mb[1] /= len;
  mb[2] /= len;
  const double beta_plus = -cp / len, beta_minus = cm / len;
  auto admissible = [&](const double* x) {
    const double b = x[0] * mb[0] + x[1] * mb[1] + x[2] * mb[2];
    return beta_plus < b && b < beta_minus;
  };

  double a[3] = {0.0, 0.0, 0.0};
  if (admissible(a0)) {
    a[0] = a0[0];
    a[1] = a0[1];
    a[2] = a0[2];
  }
  double fp[9], fm[9], pp[9], pm[9];
  NhState sp, sm;
  auto update = [&]() -> bool {
    form_phases(fbox, n, cp, cm, a, fp, fm);
    return law_eval(Lp, fp, pp, sp) && law_eval(Lm, fm, pm, sm);
  };
  double f[3];
  auto jump = [&]() {
    double tp[3], tm[3];
    mat_n(pp, n, tp);
    mat_n(pm, n, tm);
    f[0] = tp[0] - tm[0];
    f[1] = tp[1] - tm[1];
    f[2] = tp[2] - tm[2];
  };
  auto scale = [&]() {
    double tp[3], tm[3];
    mat_n(pp, n, tp);
    mat_n(pm, n, tm);
    return fmax(fmax(norm3(tp), norm3(tm)), M.lam.stress_floor);
  };
  auto converged = [&]() {
    const double floor_ = 16.0 * 2.220446049250313e-16 *
                          fmax(law_tangent_norm(Lp, sp) * sqrt(sq9(fp)), law_tangent_norm(Lm, sm) * sqrt(sq9(fm)));
    return norm3(f) <= M.lam.tol_abs + floor_ + M.lam.tol_rel * fmax(scale(), 1e-300);
  };

  if (!update()) {
    // cannot happen inside the admissible band; :192-196 returns the default
    // result (P = 0) and state (a = 0)
#pragma unroll
    for (int i = 0; i < 9; ++i) R.p[i] = 0.0;
    R.a[0] = R.a[1] = R.a[2] = 0.0;
    return;
  }
  jump();
  double best = norm3(f);
  double best_a[3] = {a[0], a[1], a[2]};
  int k = 0;
  bool ok = converged();
  while (!ok && k < M.lam.max_iter) {
    double q1[9], q2[9], h[9];
    law_dtad(Lp, sp, n, q1);
    law_dtad(Lm, sm, n, q2);
#pragma unroll
    for (int i = 0; i < 9; ++i) h[i] = q1[i] / cp + q2[i] / cm;
    Lu3 lu;
    lu.factor(h);
    if (!lu.ok) break;
    double step[3];
    lu.solve(f, step);
    double a1[3] = {a[0] - step[0], a[1] - step[1], a[2] - step[2]};
    ++k;
    if (!admissible(a1)) {
      if (!M.lam.back_projection) {
        // :221-229 returns the default result (P = 0) with the last state
        R.iterations = k;
        R.converged = false;
#pragma unroll
        for (int i = 0; i < 9; ++i) R.p[i] = 0.0;
        R.a[0] = a[0];
        R.a[1] = a[1];
        R.a[2] = a[2];
        return;
      }
      // back_project (:138-144)
      const double b1 = a1[0] * mb[0] + a1[1] * mb[1] + a1[2] * mb[2];
      const double b0 = a[0] * mb[0] + a[1] * mb[1] + a[2] * mb[2];
      const double bc = (b1 <= beta_plus) ? beta_plus : beta_minus;
      const double bs = 0.5 * (b0 + bc);
      a1[0] += (bs - b1) * mb[0];
      a1[1] += (bs - b1) * mb[1];
      a1[2] += (bs - b1) * mb[2];
      ++R.back_projections;
    }
    a[0] = a1[0];
    a[1] = a1[1];
    a[2] = a1[2];
    if (!update()) break;
    jump();
    const double r = norm3(f);
    if (r < best) {
      best = r;
      best_a[0] = a[0];
      best_a[1] = a[1];
      best_a[2] = a[2];
    }
    ok = converged();
  }
  if (!ok && (best_a[0] != a[0] || best_a[1] != a[1] || best_a[2] != a[2])) {
    a[0] = best_a[0];
    a[1] = best_a[1];
    a[2] = best_a[2];
    update();
  }
  R.converged = ok;
  R.iterations = k;
#pragma unroll
  for (int i = 0; i < 9; ++i) R.p[i] = cp * pp[i] + cm * pm[i];
  R.a[0] = a[0];
  R.a[1] = a[1];
  R.a[2] = a[2];
}

// Phase states + factored Newton Hessian of a converged laminate: everything
// the effective tangent needs (laminate.cpp:146-156).
struct LamTangent {
  NhState sp, sm;
  Lu3 lu;
  double n[3], cp, cm;
  bool ok;
};

__device__ inline void laminate_prepare(const MatParams& M, const double* fbox, const double* n, double cp,
                                        double cm, const double* a, LamTangent& S) {
  double fp[9], fm[9], pp[9], pm[9];
  form_phases(fbox, n, cp, cm, a, fp, fm);
  S.n[0] = n[0];
  S.n[1] = n[1];
  S.n[2] = n[2];
  S.cp = cp;
  S.cm = cm;
  S.ok = law_eval(M.law[1], fp, pp, S.sp) && law_eval(M.law[0], fm, pm, S.sm);
  if (!S.ok) return;
  double q1[9], q2[9], h[9];
  law_dtad(M.law[1], S.sp, n, q1);
  law_dtad(M.law[0], S.sm, n, q2);
#pragma unroll
  for (int i = 0; i < 9; ++i) h[i] = q1[i] / cp + q2[i] / cm;
  S.lu.factor(h);
}

// y = A_box x (matrix-free effective_tangent): y = c+ A+x + c- A-x
// - dA (z (x) N), z = (D^T (A+/c+ + A-/c-) D)^{-1} D^T dA x.
__device__ inline void laminate_apply_prepared(const MatParams& M, const LamTangent& S, const double* x,
                                               double* y) {
  if (!S.ok) {
#pragma unroll
    for (int i = 0; i < 9; ++i) y[i] = x[i];  // identity tangent (cell_material.cpp:134)
    return;
  }
  double u[9], v[9];
  law_apply(M.law[1], S.sp, x, u);
  law_apply(M.law[0], S.sm, x, v);
  double w[3];
  {
    double d[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) d[i] = u[i] - v[i];
    mat_n(d, S.n, w);
  }
  double z[3];
  S.lu.solve(w, z);
  double zn[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) zn[3 * i + j] = z[i] * S.n[j];
  double cu[9], cv[9];
  law_apply(M.law[1], S.sp, zn, cu);
  law_apply(M.law[0], S.sm, zn, cv);
#pragma unroll
  for (int i = 0; i < 9; ++i) y[i] = (S.cp * u[i] + S.cm * v[i]) - (cu[i] - cv[i]);
}

__device__ inline void laminate_apply(const MatParams& M, const double* fbox, const double* n, double cp,
                                      double cm, const double* a, const double* x, double* y) {
  LamTangent S;
  laminate_prepare(M, fbox, n, cp, cm, a, S);
  laminate_apply_prepared(M, S, x, y);
}

// Symmetrized packed upper triangle of A_box (pack45, cell_material.cpp:86-92)
// from nine matrix-free column applications; t45[t * stride] for t < 45.
__device__ inline void laminate_tangent45(const MatParams& M, const LamTangent& S, double* t45, int64_t stride) {
  double v[45];
#pragma unroll
  for (int t = 0; t < 45; ++t) v[t] = 0.0;
#pragma unroll
  for (int c = 0; c < 9; ++c) {
    double x[9], y[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) x[i] = i == c ? 1.0 : 0.0;
    laminate_apply_prepared(M, S, x, y);
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      if (r == c) {
        v[r * 9 - r * (r - 1) / 2] += y[r];
      } else if (r < c) {
        v[r * 9 - r * (r - 1) / 2 + (c - r)] += 0.5 * y[r];
      } else {
        v[c * 9 - c * (c - 1) / 2 + (r - c)] += 0.5 * y[r];
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 45; ++t) t45[t * stride] = v[t];
}

// y = A x with the packed symmetric tangent (tangent_matvec,
// cell_material.cpp:170-194), t45[t * stride]
__device__ __forceinline__ void packed45_apply(const double* __restrict__ t45, int64_t stride, const double* x,
                                               double* y) {
#pragma unroll
  for (int c = 0; c < 9; ++c) y[c] = 0.0;
  int t = 0;
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    const double d = __ldg(t45 + (t++) * stride);
    y[r] += d * x[r];
#pragma unroll
    for (int c = r + 1; c < 9; ++c) {
      const double a = __ldg(t45 + (t++) * stride);
      y[r] += a * x[c];
      y[c] += a * x[r];
    }
  }
}

}  // namespace combo_dev
