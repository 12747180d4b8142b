// TEST INFRASTRUCTURE ONLY (see oracle.hpp): image generators, coarsening,
// Laplace weights and interface normals, restated from
// /root/reference/proj/src/{image,combo_grid,normals}.cpp. Built with
// -ffp-contract=off: these paths are compared bit for bit with the GPU.
#include <algorithm>
#include <atomic>

#include "oracle.hpp"

namespace oracle {

namespace {
inline double wrapd(double d, double l) { return d - l * std::round(d / l); }  // image.cpp:34
inline std::int64_t wrapi(std::int64_t a, std::int64_t n) {
  a %= n;
  return a < 0 ? a + n : a;
}
}  // namespace

// image.cpp:36-55
std::int64_t PhaseImage::inclusion_count() const {
  std::int64_t total = 0;
  for (auto v : data) total += v;
  return total;
}

// image.cpp:57-86
PhaseImage generate_from_predicate(const std::array<std::int64_t, 3>& dims,
                                   const std::array<double, 3>& lengths,
                                   const std::function<bool(const Vec3&)>& inside) {
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 1) throw BadShapeSpec("generate: dims must be >= 1");
    if (!(lengths[a] > 0.0)) throw BadShapeSpec("generate: lengths must be positive");
  }
  PhaseImage img;
  img.dims = dims;
  img.lengths = lengths;
  img.data.assign(std::size_t(img.size()), 0);
  const double h1 = img.spacing(0), h2 = img.spacing(1), h3 = img.spacing(2);
#pragma omp parallel for schedule(static)
  for (std::int64_t i = 0; i < dims[0]; ++i) {
    const double x = (double(i) + 0.5) * h1;
    for (std::int64_t j = 0; j < dims[1]; ++j) {
      const double y = (double(j) + 0.5) * h2;
      const std::size_t base = img.index(i, j, 0);
      for (std::int64_t k = 0; k < dims[2]; ++k) {
        Vec3 p;
        p[0] = x;
        p[1] = y;
        p[2] = (double(k) + 0.5) * h3;
        img.data[base + std::size_t(k)] = inside(p) ? 1 : 0;
      }
    }
  }
  return img;
}

// image.cpp:88-103
PhaseImage generate_sphere(const std::array<std::int64_t, 3>& dims,
                           const std::array<double, 3>& lengths, double radius) {
  if (radius < 0.0) throw BadShapeSpec("sphere: radius must be >= 0");
  const double c0 = 0.5 * lengths[0], c1 = 0.5 * lengths[1], c2 = 0.5 * lengths[2];
  const double r2 = radius * radius;
  return generate_from_predicate(dims, lengths, [&](const Vec3& x) {
    const double dx = wrapd(x[0] - c0, lengths[0]);
    const double dy = wrapd(x[1] - c1, lengths[1]);
    const double dz = wrapd(x[2] - c2, lengths[2]);
    return dx * dx + dy * dy + dz * dz < r2;
  });
}

// image.cpp:105-119
PhaseImage generate_octahedron(const std::array<std::int64_t, 3>& dims,
                               const std::array<double, 3>& lengths, double radius) {
  if (radius < 0.0) throw BadShapeSpec("octahedron: radius must be >= 0");
  const double c0 = 0.5 * lengths[0], c1 = 0.5 * lengths[1], c2 = 0.5 * lengths[2];
  return generate_from_predicate(dims, lengths, [&](const Vec3& x) {
    return std::abs(wrapd(x[0] - c0, lengths[0])) + std::abs(wrapd(x[1] - c1, lengths[1])) +
               std::abs(wrapd(x[2] - c2, lengths[2])) <
           radius;
  });
}

namespace {
// image.cpp:123-129
double capsule_dist(const Vec3& p, const Vec3& dir, double hl) {
  const double t = std::clamp(dot(p, dir), -hl, hl);
  Vec3 q;
  for (int i = 0; i < 3; ++i) q[i] = p[i] - t * dir[i];
  return norm(q);
}
}  // namespace

// image.cpp:133-155
PhaseImage generate_fiber(const std::array<std::int64_t, 3>& dims,
                          const std::array<double, 3>& lengths, int axis, double radius,
                          double length) {
  if (axis < 0 || axis > 2) throw BadShapeSpec("fiber: axis must be 0, 1, 2");
  if (radius < 0.0) throw BadShapeSpec("fiber: radius must be >= 0");
  const double c[3] = {0.5 * lengths[0], 0.5 * lengths[1], 0.5 * lengths[2]};
  const bool full = length >= lengths[std::size_t(axis)];
  Vec3 dir;
  dir[axis] = 1.0;
  const double hl = 0.5 * length;
  return generate_from_predicate(dims, lengths, [&](const Vec3& x) {
    Vec3 d;
    for (int a = 0; a < 3; ++a) d[a] = wrapd(x[a] - c[a], lengths[a]);
    if (full) {
      d[axis] = 0.0;
      return norm(d) < radius;
    }
    return capsule_dist(d, dir, hl) < radius;
  });
}

// image.cpp:157-177
PhaseImage generate_cross_ply(const std::array<std::int64_t, 3>& dims,
                              const std::array<double, 3>& lengths, double radius,
                              double pitch, int layers) {
  if (layers < 1) throw BadShapeSpec("cross_ply: need at least one layer");
  if (!(pitch > 0.0) || radius < 0.0) throw BadShapeSpec("cross_ply: pitch/radius");
  const double lt = lengths[0] / layers;
  return generate_from_predicate(dims, lengths, [&](const Vec3& x) {
    const int ply = std::min<int>(layers - 1, int(x[0] / lt));
    const double xc = (ply + 0.5) * lt;
    const double dx = x[0] - xc;
    const double t = (ply % 2 == 0) ? x[2] : x[1];
    const double dt = wrapd(t - 0.5 * pitch, pitch);
    return dx * dx + dt * dt < radius * radius;
  });
}

// image.cpp:179-212
PhaseImage generate_fiber_pack(const std::array<std::int64_t, 3>& dims,
                               const std::array<double, 3>& lengths, std::uint64_t seed,
                               int count, double radius, double length, double spread) {
  if (count < 0) throw BadShapeSpec("fiber_pack: count must be >= 0");
  if (radius < 0.0 || length < 0.0) throw BadShapeSpec("fiber_pack: radius/length");
  Splitmix64 rng(seed);
  std::vector<Vec3> centers(static_cast<std::size_t>(count));
  std::vector<Vec3> dirs(static_cast<std::size_t>(count));
  for (int f = 0; f < count; ++f) {
    Vec3& c = centers[std::size_t(f)];
    c[0] = rng.unit() * lengths[0];
    c[1] = rng.unit() * lengths[1];
    c[2] = rng.unit() * lengths[2];
    Vec3 d;
    d[0] = 1.0;
    d[1] = spread * rng.symmetric();
    d[2] = spread * rng.symmetric();
    const double len = norm(d);
    for (int a = 0; a < 3; ++a) d[a] = d[a] / len;
    dirs[std::size_t(f)] = d;
  }
  const double hl = 0.5 * length;
  return generate_from_predicate(dims, lengths, [&](const Vec3& x) {
    for (int f = 0; f < count; ++f) {
      const auto fi = std::size_t(f);
      Vec3 d;
      for (int a = 0; a < 3; ++a) d[a] = wrapd(x[a] - centers[fi][a], lengths[a]);
      if (capsule_dist(d, dirs[fi], hl) < radius) return true;
    }
    return false;
  });
}

// image.cpp:214-227
PhaseImage generate_slab(const std::array<std::int64_t, 3>& dims,
                         const std::array<double, 3>& lengths, int axis, double fraction) {
  if (axis < 0 || axis > 2) throw BadShapeSpec("slab: axis must be 0, 1, 2");
  if (!(fraction >= 0.0 && fraction <= 1.0)) throw BadShapeSpec("slab: fraction");
  const double l = lengths[std::size_t(axis)];
  const double half = 0.5 * fraction * l;
  const double c = 0.5 * l;
  return generate_from_predicate(dims, lengths,
                                 [&](const Vec3& x) { return std::abs(wrapd(x[axis] - c, l)) < half; });
}

// image.cpp:229-244
PhaseImage mirrored(const PhaseImage& img, int axis) {
  PhaseImage out;
  out.dims = img.dims;
  out.lengths = img.lengths;
  out.data.resize(img.data.size());
  const auto n1 = img.dims[0], n2 = img.dims[1], n3 = img.dims[2];
  for (std::int64_t i = 0; i < n1; ++i)
    for (std::int64_t j = 0; j < n2; ++j)
      for (std::int64_t k = 0; k < n3; ++k) {
        const std::int64_t mi = axis == 0 ? n1 - 1 - i : i;
        const std::int64_t mj = axis == 1 ? n2 - 1 - j : j;
        const std::int64_t mk = axis == 2 ? n3 - 1 - k : k;
        out.data[out.index(mi, mj, mk)] = img.at(i, j, k);
      }
  return out;
}

// ------------------------------------------------ seeded config generators
// The BASELINE configs' microstructures do not exist in the reference
// (SURVEY.md §8d). This restates the product's generators (random sequential
// addition of periodic spheres / z-disks, Boolean ellipsoids; splitmix64 as
// image.cpp:18-32) on the CPU with the same draw order and the same voxel
// predicates, so both arms see bit-identical images.
namespace {
struct Obj {
  double c[3], a[3], R[9], r;
  int type;  // 0 sphere, 1 z-cylinder, 2 ellipsoid
};

std::vector<Obj> rsa_objects(const std::array<double, 3>& L, double h, std::uint64_t seed, double rmin,
                             double rmax, double phi, bool dim2) {
  const double r_lo = rmin * h, r_hi = rmax * h;
  const double target = dim2 ? phi * L[0] * L[1] : phi * L[0] * L[1] * L[2];
  const double kPi = 3.141592653589793238462643383279502884;
  Splitmix64 rng(seed);
  const double cs = 2.0 * r_hi;
  int nc[3];
  for (int a = 0; a < 3; ++a) nc[a] = std::max(1, int(L[a] / cs));
  if (dim2) nc[2] = 1;
  std::vector<std::vector<int>> cells(std::size_t(nc[0]) * nc[1] * nc[2]);
  std::vector<Obj> out;
  double acc = 0.0;
  for (std::int64_t att = 0; acc < target; ++att) {
    if (att >= 200000000LL) throw BadShapeSpec("rsa: volume fraction not reachable");
    Obj o{};
    o.c[0] = rng.unit() * L[0];
    o.c[1] = rng.unit() * L[1];
    o.c[2] = dim2 ? 0.5 * L[2] : rng.unit() * L[2];
    const double r = r_lo + (r_hi - r_lo) * rng.unit();
    int ci[3];
    for (int a = 0; a < 3; ++a) ci[a] = std::min(nc[a] - 1, int(o.c[a] / L[a] * nc[a]));
    auto clash = [&](const Obj& q) {
      const double ex = wrapd(o.c[0] - q.c[0], L[0]), ey = wrapd(o.c[1] - q.c[1], L[1]);
      const double ez = dim2 ? 0.0 : wrapd(o.c[2] - q.c[2], L[2]);
      const double rr = r + q.a[0];
      return ex * ex + ey * ey + ez * ez < rr * rr;
    };
    bool ok = true;
    if (nc[0] < 3 || nc[1] < 3 || (!dim2 && nc[2] < 3)) {
      for (const Obj& q : out)
        if (clash(q)) {
          ok = false;
          break;
        }
    } else {
      for (int dx = -1; dx <= 1 && ok; ++dx)
        for (int dy = -1; dy <= 1 && ok; ++dy)
          for (int dz = (dim2 ? 0 : -1); dz <= (dim2 ? 0 : 1) && ok; ++dz) {
            const int a = ((ci[0] + dx) % nc[0] + nc[0]) % nc[0];
            const int b = ((ci[1] + dy) % nc[1] + nc[1]) % nc[1];
            const int c = ((ci[2] + dz) % nc[2] + nc[2]) % nc[2];
            for (int idx : cells[(std::size_t(a) * nc[1] + b) * nc[2] + c])
              if (clash(out[std::size_t(idx)])) {
                ok = false;
                break;
              }
          }
    }
    if (!ok) continue;
    o.type = dim2 ? 1 : 0;
    o.a[0] = o.a[1] = o.a[2] = r;
    o.r = r;
    cells[(std::size_t(ci[0]) * nc[1] + ci[1]) * nc[2] + ci[2]].push_back(int(out.size()));
    out.push_back(o);
    acc += dim2 ? kPi * r * r : 4.0 / 3.0 * kPi * r * r * r;
  }
  return out;
}

std::vector<Obj> boolean_ellipsoid_objects(const std::array<double, 3>& L, double h, std::uint64_t seed,
                                           double amin, double amax, double phi) {
  const double kPi = 3.141592653589793238462643383279502884;
  const double target = -std::log(1.0 - phi) * (L[0] * L[1] * L[2]);
  Splitmix64 rng(seed);
  std::vector<Obj> out;
  double acc = 0.0;
  while (acc < target) {
    Obj o{};
    for (int a = 0; a < 3; ++a) o.c[a] = rng.unit() * L[a];
    for (int a = 0; a < 3; ++a) o.a[a] = h * (amin + (amax - amin) * rng.unit());
    const double u1 = rng.unit(), u2 = rng.unit(), u3 = rng.unit();
    const double s1 = std::sqrt(1.0 - u1), s2 = std::sqrt(u1);
    const double qx = s1 * std::sin(2 * kPi * u2), qy = s1 * std::cos(2 * kPi * u2);
    const double qz = s2 * std::sin(2 * kPi * u3), qw = s2 * std::cos(2 * kPi * u3);
    const double R[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw),     2 * (qx * qz + qy * qw),
                         2 * (qx * qy + qz * qw),     1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw),
                         2 * (qx * qz - qy * qw),     2 * (qy * qz + qx * qw),     1 - 2 * (qx * qx + qy * qy)};
    for (int i = 0; i < 9; ++i) o.R[i] = R[i];
    o.r = std::max(o.a[0], std::max(o.a[1], o.a[2]));
    o.type = 2;
    out.push_back(o);
    acc += 4.0 / 3.0 * kPi * o.a[0] * o.a[1] * o.a[2];
  }
  return out;
}
}  // namespace

PhaseImage generate_config(int shape, const std::array<std::int64_t, 3>& dims, const std::array<double, 3>& L,
                           const double* p) {
  PhaseImage img;
  img.dims = dims;
  img.lengths = L;
  img.data.assign(std::size_t(img.size()), 0);
  const double h[3] = {L[0] / double(dims[0]), L[1] / double(dims[1]), L[2] / double(dims[2])};
  std::vector<Obj> objs;
  if (shape == 10) objs = rsa_objects(L, h[0], std::uint64_t(p[0]), p[1], p[2], p[3], false);
  else if (shape == 11) objs = rsa_objects(L, h[0], std::uint64_t(p[0]), p[1], p[1], p[2], true);
  else if (shape == 12) objs = boolean_ellipsoid_objects(L, h[0], std::uint64_t(p[0]), p[1], p[2], p[3]);
  else throw BadShapeSpec("generate_config: unknown shape");
  const auto n1 = dims[0], n2 = dims[1], n3 = dims[2];
#pragma omp parallel for schedule(dynamic, 64)
  for (std::int64_t o = 0; o < std::int64_t(objs.size()); ++o) {
    const Obj& ob = objs[std::size_t(o)];
    const std::int64_t i0 = std::int64_t(std::floor((ob.c[0] - ob.r) / h[0])) - 1;
    const std::int64_t i1 = std::int64_t(std::floor((ob.c[0] + ob.r) / h[0])) + 1;
    const std::int64_t j0 = std::int64_t(std::floor((ob.c[1] - ob.r) / h[1])) - 1;
    const std::int64_t j1 = std::int64_t(std::floor((ob.c[1] + ob.r) / h[1])) + 1;
    std::int64_t k0 = std::int64_t(std::floor((ob.c[2] - ob.r) / h[2])) - 1;
    std::int64_t k1 = std::int64_t(std::floor((ob.c[2] + ob.r) / h[2])) + 1;
    if (ob.type == 1) {
      k0 = 0;
      k1 = n3 - 1;
    }
    const std::int64_t ni = std::min(i1 - i0 + 1, n1), nj = std::min(j1 - j0 + 1, n2), nk = std::min(k1 - k0 + 1, n3);
    for (std::int64_t ii = 0; ii < ni; ++ii)
      for (std::int64_t jj = 0; jj < nj; ++jj)
        for (std::int64_t kk = 0; kk < nk; ++kk) {
          const std::int64_t i = wrapi(i0 + ii, n1), j = wrapi(j0 + jj, n2), k = wrapi(k0 + kk, n3);
          const double x = (double(i) + 0.5) * h[0], y = (double(j) + 0.5) * h[1], z = (double(k) + 0.5) * h[2];
          const double dx = wrapd(x - ob.c[0], L[0]), dy = wrapd(y - ob.c[1], L[1]), dz = wrapd(z - ob.c[2], L[2]);
          bool in;
          if (ob.type == 0) {
            in = dx * dx + dy * dy + dz * dz < ob.a[0] * ob.a[0];
          } else if (ob.type == 1) {
            in = dx * dx + dy * dy < ob.a[0] * ob.a[0];
          } else {
            const double b0 = ob.R[0] * dx + ob.R[3] * dy + ob.R[6] * dz;
            const double b1 = ob.R[1] * dx + ob.R[4] * dy + ob.R[7] * dz;
            const double b2 = ob.R[2] * dx + ob.R[5] * dy + ob.R[8] * dz;
            const double q = (b0 / ob.a[0]) * (b0 / ob.a[0]) + (b1 / ob.a[1]) * (b1 / ob.a[1]) +
                             (b2 / ob.a[2]) * (b2 / ob.a[2]);
            in = q < 1.0;
          }
          if (in) {
            // idempotent byte store; objects may overlap (Boolean model)
            std::uint8_t* px = &img.data[std::size_t((i * n2 + j) * n3 + k)];
#pragma omp atomic write
            *px = 1;
          }
        }
  }
  return img;
}

// ---------------------------------------------------------------- coarsen
std::int64_t ComboGrid::composite_count() const {
  std::int64_t n = 0;
  for (auto k : kind) n += k == kComposite ? 1 : 0;
  return n;
}
std::int64_t ComboGrid::global_count_plus() const {
  std::int64_t n = 0;
  for (auto c : count_plus) n += c;
  return n;
}
double ComboGrid::global_c_plus() const {
  return double(global_count_plus()) / double(boxel_count() * fine_per_boxel());
}

// combo_grid.cpp:28-71
ComboGrid coarsen(const PhaseImage& img, const std::array<std::int64_t, 3>& factors) {
  ComboGrid g;
  g.factors = factors;
  g.lengths = img.lengths;
  for (int a = 0; a < 3; ++a) {
    const auto f = factors[a];
    const auto n = img.dims[a];
    if (f < 1 || n % f != 0) throw NonDividingFactor("coarsen: factor does not divide image dims");
    g.dims[a] = n / f;
  }
  const std::int64_t nb = g.boxel_count();
  const std::int64_t vol = g.fine_per_boxel();
  g.kind.assign(std::size_t(nb), kPureMatrix);
  g.c_plus.assign(std::size_t(nb), 0.0);
  g.count_plus.assign(std::size_t(nb), 0);
  g.normal.assign(std::size_t(nb), Vec3());
  g.normal_flag.assign(std::size_t(nb), kNormalNone);
  const auto f1 = factors[0], f2 = factors[1], f3 = factors[2];
#pragma omp parallel for collapse(2) schedule(static)
  for (std::int64_t bi = 0; bi < g.dims[0]; ++bi) {
    for (std::int64_t bj = 0; bj < g.dims[1]; ++bj) {
      for (std::int64_t bk = 0; bk < g.dims[2]; ++bk) {
        std::int64_t cnt = 0;
        for (std::int64_t a = 0; a < f1; ++a)
          for (std::int64_t b = 0; b < f2; ++b) {
            const std::size_t base = img.index(bi * f1 + a, bj * f2 + b, bk * f3);
            for (std::int64_t c = 0; c < f3; ++c) cnt += img.data[base + std::size_t(c)];
          }
        const std::size_t ib = g.index(bi, bj, bk);
        g.count_plus[ib] = cnt;
        g.c_plus[ib] = double(cnt) / double(vol);
        g.kind[ib] = cnt == 0 ? kPureMatrix : cnt == vol ? kPureInclusion : kComposite;
      }
    }
  }
  return g;
}

// ---------------------------------------------------------------- normals
// normals.cpp:25-52 (direct 7-point stencil, periodic)
std::vector<double> laplace_weights(const PhaseImage& img) {
  const std::int64_t n = img.size();
  std::vector<double> w(std::size_t(n), 0.0);
  const double h1 = img.spacing(0), h2 = img.spacing(1), h3 = img.spacing(2);
  const double r1 = h2 * h3 / h1, r2 = h1 * h3 / h2, r3 = h1 * h2 / h3;
  const auto n1 = img.dims[0], n2 = img.dims[1], n3 = img.dims[2];
#pragma omp parallel for collapse(2) schedule(static)
  for (std::int64_t i = 0; i < n1; ++i) {
    for (std::int64_t j = 0; j < n2; ++j) {
      const std::int64_t im = wrapi(i - 1, n1), ip = wrapi(i + 1, n1);
      const std::int64_t jm = wrapi(j - 1, n2), jp = wrapi(j + 1, n2);
      for (std::int64_t k = 0; k < n3; ++k) {
        const std::int64_t km = wrapi(k - 1, n3), kp = wrapi(k + 1, n3);
        const double c = img.at(i, j, k);
        const double s = r1 * (img.at(im, j, k) - 2.0 * c + img.at(ip, j, k)) +
                         r2 * (img.at(i, jm, k) - 2.0 * c + img.at(i, jp, k)) +
                         r3 * (img.at(i, j, km) - 2.0 * c + img.at(i, j, kp));
        w[img.index(i, j, k)] = std::abs(s);
      }
    }
  }
  return w;
}

namespace {
struct BarycenterNormal {
  Vec3 n;
  bool degenerate = false;
};

// normals.cpp:87-137
BarycenterNormal boxel_barycenter_normal(const PhaseImage& img, const ComboGrid& grid,
                                         std::int64_t bi, std::int64_t bj, std::int64_t bk) {
  const auto f1 = grid.factors[0], f2 = grid.factors[1], f3 = grid.factors[2];
  double sp[3] = {0, 0, 0}, sm[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  std::int64_t np = 0, nm = 0;
  for (std::int64_t a = 0; a < f1; ++a)
    for (std::int64_t b = 0; b < f2; ++b)
      for (std::int64_t c = 0; c < f3; ++c) {
        const std::int64_t i = bi * f1 + a, j = bj * f2 + b, k = bk * f3 + c;
        const Vec3 x = img.voxel_center(i, j, k);
        if (img.at(i, j, k)) {
          for (int d = 0; d < 3; ++d) sp[d] += x[d];
          if (np == 0) {
            for (int d = 0; d < 3; ++d) lo[d] = hi[d] = x[d];
          } else {
            for (int d = 0; d < 3; ++d) {
              lo[d] = std::min(lo[d], x[d]);
              hi[d] = std::max(hi[d], x[d]);
            }
          }
          ++np;
        } else {
          for (int d = 0; d < 3; ++d) sm[d] += x[d];
          ++nm;
        }
      }
  BarycenterNormal out;
  if (np == 0 || nm == 0) {
    out.degenerate = true;
    out.n[0] = 1.0;
    return out;
  }
  Vec3 d;
  for (int q = 0; q < 3; ++q) d[q] = sm[q] / double(nm) - sp[q] / double(np);
  Vec3 bl;
  for (int q = 0; q < 3; ++q) bl[q] = grid.boxel_length(q);
  const double diag = norm(bl);
  const double dn = norm(d);
  if (dn < 1e-12 * diag) {
    out.degenerate = true;
    double ext[3];
    for (int q = 0; q < 3; ++q) ext[q] = hi[q] - lo[q];
    int axis = 0;
    if (ext[1] > ext[axis]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    out.n[axis] = 1.0;
    return out;
  }
  for (int q = 0; q < 3; ++q) out.n[q] = d[q] / dn;
  return out;
}

struct SecondMomentResult {
  Vec3 n;
  bool too_few = false;
};

// normals.cpp:146-207; sym_eig3 (tensor.cpp:70-91) replaced by the
// sqrt-only Jacobi solver so the GPU can reproduce the bits.
SecondMomentResult boxel_second_moment_normal(const PhaseImage& img, const ComboGrid& grid,
                                              const std::vector<double>& w, std::int64_t bi,
                                              std::int64_t bj, std::int64_t bk, int centering,
                                              int min_support) {
  const auto f1 = grid.factors[0], f2 = grid.factors[1], f3 = grid.factors[2];
  SecondMomentResult out;
  double wx[3] = {0, 0, 0};
  double wsum = 0.0;
  std::int64_t support = 0;
  for (std::int64_t a = 0; a < f1; ++a)
    for (std::int64_t b = 0; b < f2; ++b)
      for (std::int64_t c = 0; c < f3; ++c) {
        const std::int64_t i = bi * f1 + a, j = bj * f2 + b, k = bk * f3 + c;
        const double wt = w[img.index(i, j, k)];
        if (wt <= 0.0) continue;
        ++support;
        wsum += wt;
        const Vec3 x = img.voxel_center(i, j, k);
        for (int d = 0; d < 3; ++d) wx[d] += wt * x[d];
      }
  if (support < min_support) {
    out.too_few = true;
    return out;
  }
  double center[3];
  if (centering == kWeightedCentroid) {
    for (int d = 0; d < 3; ++d) center[d] = wx[d] / wsum;
  } else {
    center[0] = (double(bi) + 0.5) * grid.boxel_length(0);
    center[1] = (double(bj) + 0.5) * grid.boxel_length(1);
    center[2] = (double(bk) + 0.5) * grid.boxel_length(2);
  }
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (std::int64_t a = 0; a < f1; ++a)
    for (std::int64_t b = 0; b < f2; ++b)
      for (std::int64_t c = 0; c < f3; ++c) {
        const std::int64_t i = bi * f1 + a, j = bj * f2 + b, k = bk * f3 + c;
        const double wt = w[img.index(i, j, k)];
        if (wt <= 0.0) continue;
        const Vec3 xc = img.voxel_center(i, j, k);
        double x[3];
        for (int d = 0; d < 3; ++d) x[d] = xc[d] - center[d];
        for (int r = 0; r < 3; ++r)
          for (int q = 0; q < 3; ++q) m[3 * r + q] += wt * (x[r] * x[q]);
      }
  const double big = (m[0] + m[4] + m[8]) + 1.0;
  for (int ax = 0; ax < 3; ++ax) {
    if (grid.factors[std::size_t(ax)] == 1) {
      for (int o = 0; o < 3; ++o) {
        m[3 * ax + o] = 0.0;
        m[3 * o + ax] = 0.0;
      }
      m[4 * ax] = big;
    }
  }
  double lam[3], vec[9];
  sym_eig3_jacobi(m, lam, vec);
  for (int d = 0; d < 3; ++d) out.n[d] = vec[3 * d + 0];
  return out;
}
}  // namespace

// normals.cpp:211-256
NormalStats compute_normals(const PhaseImage& img, ComboGrid& grid, int method, int centering,
                            int min_support) {
  NormalStats stats;
  std::vector<double> weights;
  if (method == kSecondMoment) weights = laplace_weights(img);
  std::atomic<std::int64_t> composite{0}, degenerate{0}, too_few{0};
#pragma omp parallel for collapse(2) schedule(static)
  for (std::int64_t bi = 0; bi < grid.dims[0]; ++bi) {
    for (std::int64_t bj = 0; bj < grid.dims[1]; ++bj) {
      for (std::int64_t bk = 0; bk < grid.dims[2]; ++bk) {
        const std::size_t ib = grid.index(bi, bj, bk);
        if (grid.kind[ib] != kComposite) continue;
        composite.fetch_add(1, std::memory_order_relaxed);
        const BarycenterNormal bary = boxel_barycenter_normal(img, grid, bi, bj, bk);
        Vec3 n = bary.n;
        std::uint8_t flag = bary.degenerate ? kNormalDegenerate : kNormalBarycenterOk;
        if (bary.degenerate) degenerate.fetch_add(1, std::memory_order_relaxed);
        if (method == kSecondMoment) {
          const SecondMomentResult sm =
              boxel_second_moment_normal(img, grid, weights, bi, bj, bk, centering, min_support);
          if (sm.too_few) {
            too_few.fetch_add(1, std::memory_order_relaxed);
            flag = kNormalTooFew;
          } else {
            if (dot(sm.n, bary.n) >= 0.0) {
              n = sm.n;
            } else {
              for (int d = 0; d < 3; ++d) n[d] = -sm.n[d];
            }
            flag = kNormalSecondMomentOk;
          }
        }
        grid.normal[ib] = n;
        grid.normal_flag[ib] = flag;
      }
    }
  }
  stats.composite = composite.load();
  stats.degenerate_fallbacks = degenerate.load();
  stats.too_few_fallbacks = too_few.load();
  return stats;
}

}  // namespace oracle
