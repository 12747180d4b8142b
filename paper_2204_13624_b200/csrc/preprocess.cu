// Volume-fraction and interface-normal preprocessing on the GPU, plus the
// image generators (reference shapes and the seeded config microstructures).
//
// Compiled with --fmad=false (and -ffp-contract=off on the host side): every
// floating-point operation below is an IEEE-exact +,-,*,/,sqrt or round in the
// reference's order, so kinds, counts, fractions and normals are bit-identical
// to the CPU oracle restating
//   coarsen                 /root/reference/proj/src/combo_grid.cpp:28-71
//   laplace_weights(direct) /root/reference/proj/src/normals.cpp:25-52
//   barycenter normal       /root/reference/proj/src/normals.cpp:87-137
//   second-moment normal    /root/reference/proj/src/normals.cpp:146-207
//   compute_normals         /root/reference/proj/src/normals.cpp:211-256
//   generate_*              /root/reference/proj/src/image.cpp:57-227
// sym_eig3 (tensor.cpp:70-91, Eigen closed form) is replaced by a sqrt-only
// cyclic Jacobi solver shared in algorithm with the oracle.
#include <cmath>
#include <cstdio>
#include <vector>

#include "context.hpp"

using namespace combo_host;

namespace {

// --------------------------------------------------------------- kernels
__device__ __forceinline__ double wrapd(double d, double l) { return d - l * round(d / l); }
__device__ __forceinline__ int64_t wrapi(int64_t a, int64_t n) {
  a %= n;
  return a < 0 ? a + n : a;
}

// A window of fine planes [i0, i0 + planes) (mod n1) of the n1 x n2 x n3
// image: at() takes global (wrapped) plane indices. The whole image is the
// window i0 = 0; a slab rank's window adds one halo plane on each side
// (the Laplace stencil of the second-moment normals, normals.cpp:39-46).
struct ImgView {
  const uint8_t* p;
  int64_t n1, n2, n3;
  double h1, h2, h3;
  int64_t i0 = 0;
  __device__ __forceinline__ uint8_t at(int64_t i, int64_t j, int64_t k) const {
    int64_t li = i - i0;
    if (li < 0) li += n1;
    return p[(li * n2 + j) * n3 + k];
  }
};

__global__ void k_coarsen(ImgView im, int64_t f1, int64_t f2, int64_t f3, int64_t b1, int64_t b2, int64_t b3,
                          uint8_t* kind, double* cplus, int64_t* count) {
  const int64_t nb = b1 * b2 * b3;
  const int64_t vol = f1 * f2 * f3;
  for (int64_t ib = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; ib < nb; ib += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bk = ib % b3, bj = (ib / b3) % b2, bi = ib / (b2 * b3);
    int64_t cnt = 0;
    for (int64_t a = 0; a < f1; ++a)
      for (int64_t b = 0; b < f2; ++b) {
        const uint8_t* row = im.p + ((bi * f1 + a) * im.n2 + bj * f2 + b) * im.n3 + bk * f3;
        for (int64_t c = 0; c < f3; ++c) cnt += row[c];
      }
    count[ib] = cnt;
    cplus[ib] = double(cnt) / double(vol);
    kind[ib] = cnt == 0 ? 0 : (cnt == vol ? 1 : 2);
  }
}

// laplace weight of one voxel (normals.cpp:36-50)
__device__ __forceinline__ double lap_weight(const ImgView& im, double r1, double r2, double r3, int64_t i, int64_t j,
                                             int64_t k) {
  const int64_t im1 = wrapi(i - 1, im.n1), ip1 = wrapi(i + 1, im.n1);
  const int64_t jm1 = wrapi(j - 1, im.n2), jp1 = wrapi(j + 1, im.n2);
  const int64_t km1 = wrapi(k - 1, im.n3), kp1 = wrapi(k + 1, im.n3);
  const double c = double(im.at(i, j, k));
  const double s = r1 * ((double(im.at(im1, j, k)) - 2.0 * c) + double(im.at(ip1, j, k))) +
                   r2 * ((double(im.at(i, jm1, k)) - 2.0 * c) + double(im.at(i, jp1, k))) +
                   r3 * ((double(im.at(i, j, km1)) - 2.0 * c) + double(im.at(i, j, kp1)));
  return fabs(s);
}

__global__ void k_laplace(ImgView im, double r1, double r2, double r3, double* w) {
  const int64_t n = im.n1 * im.n2 * im.n3;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = v % im.n3, j = (v / im.n3) % im.n2, i = v / (im.n2 * im.n3);
    w[v] = lap_weight(im, r1, r2, r3, i, j, k);
  }
}

// --- cyclic Jacobi for symmetric 3x3 (same operation order as the oracle)
__device__ void jac_rotate(double* a, double* v, int p, int q) {
  const double apq = a[p * 3 + q];
  const double app = a[p * 3 + p], aqq = a[q * 3 + q];
  const double g = 100.0 * fabs(apq);
  if (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) {
    a[p * 3 + q] = 0.0;
    a[q * 3 + p] = 0.0;
    return;
  }
  const double h = aqq - app;
  double t;
  if (fabs(h) + g == fabs(h)) {
    t = apq / h;
  } else {
    const double theta = 0.5 * h / apq;
    t = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
    if (theta < 0.0) t = -t;
  }
  const double c = 1.0 / sqrt(1.0 + t * t);
  const double s = t * c;
  const double tau = s / (1.0 + c);
  a[p * 3 + p] = app - t * apq;
  a[q * 3 + q] = aqq + t * apq;
  a[p * 3 + q] = 0.0;
  a[q * 3 + p] = 0.0;
  for (int r = 0; r < 3; ++r) {
    if (r == p || r == q) continue;
    const double gr = a[r * 3 + p], hr = a[r * 3 + q];
    const double np = gr - s * (hr + gr * tau);
    const double nq = hr + s * (gr - hr * tau);
    a[r * 3 + p] = np;
    a[p * 3 + r] = np;
    a[r * 3 + q] = nq;
    a[q * 3 + r] = nq;
  }
  for (int r = 0; r < 3; ++r) {
    const double gr = v[r * 3 + p], hr = v[r * 3 + q];
    v[r * 3 + p] = gr - s * (hr + gr * tau);
    v[r * 3 + q] = hr + s * (gr - hr * tau);
  }
}

// smallest-eigenvalue eigenvector (column 0 after the ascending sort)
__device__ void smallest_eigvec(const double* m, double* out) {
  double a[9], v[9];
  for (int i = 0; i < 9; ++i) {
    a[i] = m[i];
    v[i] = 0.0;
  }
  v[0] = v[4] = v[8] = 1.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    if (!(a[1] != 0.0 || a[2] != 0.0 || a[5] != 0.0)) break;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q)
        if (a[p * 3 + q] != 0.0) jac_rotate(a, v, p, q);
  }
  double lam[3] = {a[0], a[4], a[8]};
  int col[3] = {0, 1, 2};
  // selection sort ascending with strict <, swapping columns (oracle order)
  for (int i = 0; i < 3; ++i) {
    int mi = i;
    for (int j = i + 1; j < 3; ++j)
      if (lam[j] < lam[mi]) mi = j;
    if (mi != i) {
      const double tl = lam[i];
      lam[i] = lam[mi];
      lam[mi] = tl;
      const int tc = col[i];
      col[i] = col[mi];
      col[mi] = tc;
    }
  }
  for (int r = 0; r < 3; ++r) out[r] = v[r * 3 + col[0]];
}

struct NormalArgs {
  ImgView im;
  int64_t f1, f2, f3, b1, b2, b3;
  int64_t bp0, nbp;  // boxel planes [bp0, bp0 + nbp) of the grid (kind / outputs: local)
  double bl0, bl1, bl2;  // boxel lengths
  double r1, r2, r3;
  int method, centering, min_support;
};

__global__ void k_normals(NormalArgs A, const uint8_t* kind, double* normal3, uint8_t* flags,
                          unsigned long long* stats) {
  const int64_t nb = A.nbp * A.b2 * A.b3;
  const ImgView& im = A.im;
  for (int64_t ib = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; ib < nb; ib += int64_t(gridDim.x) * blockDim.x) {
    if (kind[ib] != 2) continue;
    atomicAdd(stats, 1ull);
    const int64_t bk = ib % A.b3, bj = (ib / A.b3) % A.b2, bi = A.bp0 + ib / (A.b2 * A.b3);
    // barycenter normal (normals.cpp:87-137)
    double sp[3] = {0, 0, 0}, smn[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    int64_t np = 0, nm = 0;
    for (int64_t a = 0; a < A.f1; ++a)
      for (int64_t b = 0; b < A.f2; ++b)
        for (int64_t c = 0; c < A.f3; ++c) {
          const int64_t i = bi * A.f1 + a, j = bj * A.f2 + b, k = bk * A.f3 + c;
          const double x[3] = {(double(i) + 0.5) * im.h1, (double(j) + 0.5) * im.h2, (double(k) + 0.5) * im.h3};
          if (im.at(i, j, k)) {
            for (int d = 0; d < 3; ++d) sp[d] += x[d];
            if (np == 0) {
              for (int d = 0; d < 3; ++d) lo[d] = hi[d] = x[d];
            } else {
              for (int d = 0; d < 3; ++d) {
                lo[d] = x[d] < lo[d] ? x[d] : lo[d];
                hi[d] = hi[d] < x[d] ? x[d] : hi[d];
              }
            }
            ++np;
          } else {
            for (int d = 0; d < 3; ++d) smn[d] += x[d];
            ++nm;
          }
        }
    double n[3] = {1.0, 0.0, 0.0};
    bool degenerate = false;
    if (np == 0 || nm == 0) {
      degenerate = true;
    } else {
      double dv[3];
      for (int q = 0; q < 3; ++q) dv[q] = smn[q] / double(nm) - sp[q] / double(np);
      const double diag = sqrt(A.bl0 * A.bl0 + A.bl1 * A.bl1 + A.bl2 * A.bl2);
      const double dn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
      if (dn < 1e-12 * diag) {
        degenerate = true;
        const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
        int axis = 0;
        if (ext[1] > ext[axis]) axis = 1;
        if (ext[2] > ext[axis]) axis = 2;
        n[0] = n[1] = n[2] = 0.0;
        n[axis] = 1.0;
      } else {
        for (int q = 0; q < 3; ++q) n[q] = dv[q] / dn;
      }
    }
    uint8_t flag = degenerate ? 3 : 1;
    if (degenerate) atomicAdd(stats + 1, 1ull);
    if (A.method == 1) {
      // second moment (normals.cpp:146-207), weights recomputed on the fly
      double wx[3] = {0, 0, 0};
      double wsum = 0.0;
      int64_t support = 0;
      for (int64_t a = 0; a < A.f1; ++a)
        for (int64_t b = 0; b < A.f2; ++b)
          for (int64_t c = 0; c < A.f3; ++c) {
            const int64_t i = bi * A.f1 + a, j = bj * A.f2 + b, k = bk * A.f3 + c;
            const double wt = lap_weight(im, A.r1, A.r2, A.r3, i, j, k);
            if (wt <= 0.0) continue;
            ++support;
            wsum += wt;
            const double x[3] = {(double(i) + 0.5) * im.h1, (double(j) + 0.5) * im.h2, (double(k) + 0.5) * im.h3};
            for (int d = 0; d < 3; ++d) wx[d] += wt * x[d];
          }
      if (support < A.min_support) {
        atomicAdd(stats + 2, 1ull);
        flag = 4;
      } else {
        double center[3];
        if (A.centering == 0) {
          for (int d = 0; d < 3; ++d) center[d] = wx[d] / wsum;
        } else {
          center[0] = (double(bi) + 0.5) * A.bl0;
          center[1] = (double(bj) + 0.5) * A.bl1;
          center[2] = (double(bk) + 0.5) * A.bl2;
        }
        double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t a = 0; a < A.f1; ++a)
          for (int64_t b = 0; b < A.f2; ++b)
            for (int64_t c = 0; c < A.f3; ++c) {
              const int64_t i = bi * A.f1 + a, j = bj * A.f2 + b, k = bk * A.f3 + c;
              const double wt = lap_weight(im, A.r1, A.r2, A.r3, i, j, k);
              if (wt <= 0.0) continue;
              const double x[3] = {(double(i) + 0.5) * im.h1 - center[0], (double(j) + 0.5) * im.h2 - center[1],
                                   (double(k) + 0.5) * im.h3 - center[2]};
              for (int r = 0; r < 3; ++r)
                for (int q = 0; q < 3; ++q) m[3 * r + q] += wt * (x[r] * x[q]);
            }
        const double big = (m[0] + m[4] + m[8]) + 1.0;
        const int64_t fac[3] = {A.f1, A.f2, A.f3};
        for (int ax = 0; ax < 3; ++ax)
          if (fac[ax] == 1) {
            for (int o = 0; o < 3; ++o) {
              m[3 * ax + o] = 0.0;
              m[3 * o + ax] = 0.0;
            }
            m[4 * ax] = big;
          }
        double ev[3];
        smallest_eigvec(m, ev);
        const double dp = ev[0] * n[0] + ev[1] * n[1] + ev[2] * n[2];
        if (dp >= 0.0) {
          n[0] = ev[0];
          n[1] = ev[1];
          n[2] = ev[2];
        } else {
          n[0] = -ev[0];
          n[1] = -ev[1];
          n[2] = -ev[2];
        }
        flag = 2;
      }
    }
    normal3[3 * ib] = n[0];
    normal3[3 * ib + 1] = n[1];
    normal3[3 * ib + 2] = n[2];
    flags[ib] = flag;
  }
}

// ------------------------------------------------------------ generators
struct GenArgs {
  int64_t n1, n2, n3;
  double L[3], h[3];
  int shape;
  double p[8];
  int64_t plane0 = 0, nplanes = 0;  // output window: global planes [plane0, plane0 + nplanes) mod n1
};

// image.cpp:88-227 predicates (same arithmetic, --fmad=false)
__device__ bool predicate(const GenArgs& g, double x, double y, double z) {
  const double c0 = 0.5 * g.L[0], c1 = 0.5 * g.L[1], c2 = 0.5 * g.L[2];
  switch (g.shape) {
    case 0: {  // sphere (image.cpp:88-103)
      const double dx = wrapd(x - c0, g.L[0]), dy = wrapd(y - c1, g.L[1]), dz = wrapd(z - c2, g.L[2]);
      return dx * dx + dy * dy + dz * dz < g.p[0] * g.p[0];
    }
    case 1:  // octahedron (:105-119)
      return fabs(wrapd(x - c0, g.L[0])) + fabs(wrapd(y - c1, g.L[1])) + fabs(wrapd(z - c2, g.L[2])) < g.p[0];
    case 2: {  // fiber (image.cpp:123-155): p = axis, radius, length
      const int axis = int(g.p[0]);
      const double radius = g.p[1], hl = 0.5 * g.p[2];
      double d[3] = {wrapd(x - c0, g.L[0]), wrapd(y - c1, g.L[1]), wrapd(z - c2, g.L[2])};
      if (g.p[2] >= g.L[axis]) {
        d[axis] = 0.0;
      } else {
        // capsule_dist with dir = e_axis: t = clamp(d . dir), q = d - t dir
        const double t = fmin(fmax(d[axis], -hl), hl);
        d[axis] = d[axis] - t;
      }
      return sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) < radius;
    }
    case 3: {  // cross_ply (image.cpp:157-177): p = radius, pitch, layers
      const double radius = g.p[0], pitch = g.p[1];
      const int layers = int(g.p[2]);
      const double lt = g.L[0] / layers;
      const int ply = min(layers - 1, int(x / lt));
      const double xc = (ply + 0.5) * lt;
      const double dx = x - xc;
      const double t = (ply % 2 == 0) ? z : y;
      const double dt = wrapd(t - 0.5 * pitch, pitch);
      return dx * dx + dt * dt < radius * radius;
    }
    case 5: {  // slab (:214-227)
      const int axis = int(g.p[0]);
      const double l = g.L[axis];
      const double half = 0.5 * g.p[1] * l;
      const double c = 0.5 * l;
      const double xa = axis == 0 ? x : (axis == 1 ? y : z);
      return fabs(wrapd(xa - c, l)) < half;
    }
    default:
      return false;
  }
}

__global__ void k_generate(GenArgs g, uint8_t* out) {
  const int64_t n = g.nplanes * g.n2 * g.n3;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = v % g.n3, j = (v / g.n3) % g.n2, i = wrapi(g.plane0 + v / (g.n2 * g.n3), g.n1);
    const double x = (double(i) + 0.5) * g.h[0];
    const double y = (double(j) + 0.5) * g.h[1];
    const double z = (double(k) + 0.5) * g.h[2];
    out[v] = predicate(g, x, y, z) ? 1 : 0;
  }
}

// fiber_pack (image.cpp:179-212): every voxel centre against the capsule
// list (centre, unit axis; generated on the host from the seed)
__global__ void k_generate_pack(GenArgs g, const double* __restrict__ fib, int count, double hl, double radius,
                                uint8_t* out) {
  const int64_t n = g.nplanes * g.n2 * g.n3;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = v % g.n3, j = (v / g.n3) % g.n2, i = wrapi(g.plane0 + v / (g.n2 * g.n3), g.n1);
    const double x[3] = {(double(i) + 0.5) * g.h[0], (double(j) + 0.5) * g.h[1], (double(k) + 0.5) * g.h[2]};
    uint8_t in = 0;
    for (int f = 0; f < count && !in; ++f) {
      const double* c = fib + 6 * f;
      const double* u = c + 3;
      double d[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) d[a] = wrapd(x[a] - c[a], g.L[a]);
      const double t = fmin(fmax(d[0] * u[0] + d[1] * u[1] + d[2] * u[2], -hl), hl);
      double q[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) q[a] = d[a] - t * u[a];
      in = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]) < radius;
    }
    out[v] = in;
  }
}

// Object rasterization for the seeded config microstructures: one block per
// object, threads sweep the (periodically wrapped) bounding box.
struct Obj {
  double c[3];
  double r;       // bounding radius
  double a[3];    // semi-axes (ellipsoid) / radius
  double R[9];    // rotation (ellipsoid): body = R^T d
  int type;       // 0 sphere, 1 z-cylinder, 2 ellipsoid
};

// objects -> voxels of the plane window [plane0, plane0 + nplanes) (mod n1)
// of the image; one block per object, plane by plane (planes outside the
// window cost one test)
__global__ void k_raster(const Obj* objs, int64_t nobj, int64_t n1, int64_t n2, int64_t n3, double L0, double L1,
                         double L2, double h0, double h1, double h2, int64_t plane0, int64_t nplanes, uint8_t* out) {
  for (int64_t o = blockIdx.x; o < nobj; o += gridDim.x) {
    const Obj ob = objs[o];
    const int64_t i0 = int64_t(floor((ob.c[0] - ob.r) / h0)) - 1, i1 = int64_t(floor((ob.c[0] + ob.r) / h0)) + 1;
    const int64_t j0 = int64_t(floor((ob.c[1] - ob.r) / h1)) - 1, j1 = int64_t(floor((ob.c[1] + ob.r) / h1)) + 1;
    int64_t k0 = int64_t(floor((ob.c[2] - ob.r) / h2)) - 1, k1 = int64_t(floor((ob.c[2] + ob.r) / h2)) + 1;
    if (ob.type == 1) {
      k0 = 0;
      k1 = n3 - 1;
    }
    const int64_t ni = min(i1 - i0 + 1, n1), nj = min(j1 - j0 + 1, n2), nk = min(k1 - k0 + 1, n3);
    const int64_t tot = nj * nk;
    for (int64_t ii = 0; ii < ni; ++ii) {
      const int64_t i = wrapi(i0 + ii, n1);
      const int64_t li = wrapi(i - plane0, n1);
      if (li >= nplanes) continue;
      const double x = (double(i) + 0.5) * h0;
      const double dx = wrapd(x - ob.c[0], L0);
      for (int64_t t = threadIdx.x; t < tot; t += blockDim.x) {
        const int64_t kk = t % nk, jj = t / nk;
        const int64_t j = wrapi(j0 + jj, n2), k = wrapi(k0 + kk, n3);
        const double y = (double(j) + 0.5) * h1, z = (double(k) + 0.5) * h2;
        const double dy = wrapd(y - ob.c[1], L1), dz = wrapd(z - ob.c[2], L2);
        bool in;
        if (ob.type == 0) {
          in = dx * dx + dy * dy + dz * dz < ob.a[0] * ob.a[0];
        } else if (ob.type == 1) {
          in = dx * dx + dy * dy < ob.a[0] * ob.a[0];
        } else {
          const double b0 = ob.R[0] * dx + ob.R[3] * dy + ob.R[6] * dz;
          const double b1 = ob.R[1] * dx + ob.R[4] * dy + ob.R[7] * dz;
          const double b2 = ob.R[2] * dx + ob.R[5] * dy + ob.R[8] * dz;
          const double q =
              (b0 / ob.a[0]) * (b0 / ob.a[0]) + (b1 / ob.a[1]) * (b1 / ob.a[1]) + (b2 / ob.a[2]) * (b2 / ob.a[2]);
          in = q < 1.0;
        }
        if (in) out[(li * n2 + j) * n3 + k] = 1;
      }
    }
  }
}

// single laminate solve for tests
__global__ void k_laminate_one(combo_dev::MatParams M, const double* in, double* out, int* ist) {
  const double* f = in;
  const double* n = in + 9;
  const double cp = in[12];
  const double* a0 = in + 13;
  combo_dev::LamResult R;
  combo_dev::laminate_solve(M, f, n, cp, 1.0 - cp, a0, R);
  for (int i = 0; i < 9; ++i) out[i] = R.p[i];
  for (int i = 0; i < 3; ++i) out[9 + i] = R.a[i];
  ist[0] = R.converged;
  ist[1] = R.iterations;
  ist[2] = R.back_projections;
  ist[3] = R.inadmissible;
}

// ------------------------------------------------------------ host RSA
struct Sm64 {  // image.cpp:18-32
  uint64_t s;
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return double(next() >> 11) * 0x1.0p-53; }
};

inline double hwrap(double d, double l) { return d - l * std::round(d / l); }

// Random sequential addition with a periodic cell list. dim2 = true: disks
// in the (0,1) plane (z-fibres); false: spheres.
std::vector<Obj> rsa(const GenArgs& g, uint64_t seed, double rmin, double rmax, double phi, bool dim2) {
  const double h = g.h[0];
  const double r_lo = rmin * h, r_hi = rmax * h;
  const double target = dim2 ? phi * g.L[0] * g.L[1] : phi * g.L[0] * g.L[1] * g.L[2];
  const double kPi = 3.141592653589793238462643383279502884;
  Sm64 rng{seed};
  const double cs = 2.0 * r_hi;
  int nc[3];
  for (int a = 0; a < 3; ++a) nc[a] = std::max(1, int(g.L[a] / cs));
  if (dim2) nc[2] = 1;
  std::vector<std::vector<int>> cells(size_t(nc[0]) * nc[1] * nc[2]);
  std::vector<Obj> out;
  double acc = 0.0;
  const int64_t max_attempts = 200000000LL;
  for (int64_t att = 0; acc < target; ++att) {
    if (att >= max_attempts) throw ComboError(COMBO_ERR_BAD_SHAPE, "rsa: volume fraction not reachable");
    Obj o{};
    o.c[0] = rng.unit() * g.L[0];
    o.c[1] = rng.unit() * g.L[1];
    o.c[2] = dim2 ? 0.5 * g.L[2] : rng.unit() * g.L[2];
    const double r = r_lo + (r_hi - r_lo) * rng.unit();
    int ci[3];
    for (int a = 0; a < 3; ++a) ci[a] = std::min(nc[a] - 1, int(o.c[a] / g.L[a] * nc[a]));
    bool ok = true;
    for (int dx = -1; dx <= 1 && ok; ++dx)
      for (int dy = -1; dy <= 1 && ok; ++dy)
        for (int dz = (dim2 ? 0 : -1); dz <= (dim2 ? 0 : 1) && ok; ++dz) {
          const int a = ((ci[0] + dx) % nc[0] + nc[0]) % nc[0];
          const int b = ((ci[1] + dy) % nc[1] + nc[1]) % nc[1];
          const int c = ((ci[2] + dz) % nc[2] + nc[2]) % nc[2];
          for (int idx : cells[(size_t(a) * nc[1] + b) * nc[2] + c]) {
            const Obj& q = out[size_t(idx)];
            const double ex = hwrap(o.c[0] - q.c[0], g.L[0]), ey = hwrap(o.c[1] - q.c[1], g.L[1]);
            const double ez = dim2 ? 0.0 : hwrap(o.c[2] - q.c[2], g.L[2]);
            const double rr = r + q.a[0];
            if (ex * ex + ey * ey + ez * ez < rr * rr) {
              ok = false;
              break;
            }
          }
          if (nc[0] < 3 || nc[1] < 3 || (!dim2 && nc[2] < 3)) {
            // tiny boxes: the 3x3x3 stencil revisits cells; brute force
            for (const Obj& q : out) {
              const double ex = hwrap(o.c[0] - q.c[0], g.L[0]), ey = hwrap(o.c[1] - q.c[1], g.L[1]);
              const double ez = dim2 ? 0.0 : hwrap(o.c[2] - q.c[2], g.L[2]);
              const double rr = r + q.a[0];
              if (ex * ex + ey * ey + ez * ez < rr * rr) {
                ok = false;
                break;
              }
            }
          }
        }
    if (!ok) continue;
    o.type = dim2 ? 1 : 0;
    o.a[0] = o.a[1] = o.a[2] = r;
    o.r = r;
    cells[(size_t(ci[0]) * nc[1] + ci[1]) * nc[2] + ci[2]].push_back(int(out.size()));
    out.push_back(o);
    acc += dim2 ? kPi * r * r : 4.0 / 3.0 * kPi * r * r * r;
  }
  return out;
}

// Boolean model of uniformly rotated ellipsoids (Shoemake quaternions);
// objects are added until sum V_i >= -ln(1 - phi) V.
std::vector<Obj> boolean_ellipsoids(const GenArgs& g, uint64_t seed, double amin, double amax, double phi) {
  const double h = g.h[0];
  const double kPi = 3.141592653589793238462643383279502884;
  const double V = g.L[0] * g.L[1] * g.L[2];
  const double target = -std::log(1.0 - phi) * V;
  Sm64 rng{seed};
  std::vector<Obj> out;
  double acc = 0.0;
  while (acc < target) {
    Obj o{};
    for (int a = 0; a < 3; ++a) o.c[a] = rng.unit() * g.L[a];
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

template <class Fn>
int guarded(combo_ctx* c, Fn&& fn) {
  try {
    if (c) COMBO_CK(cudaSetDevice(c->device));
    fn();
    return COMBO_OK;
  } catch (const ComboError& e) {
    if (c) c->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return COMBO_ERR_BAD_ARGUMENT;
  }
}

template <class T>
T* dev_or_stage(combo_ctx* c, T* p, size_t n, int mem, DBuf<T>& tmp, bool copy_in) {
  if (mem == COMBO_MEM_DEVICE) return p;
  tmp.alloc(n);
  if (copy_in) COMBO_CK(cudaMemcpyAsync(tmp.p, p, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return tmp.p;
}
template <class T>
void copy_back(combo_ctx* c, T* host, const T* dev, size_t n, int mem) {
  if (mem == COMBO_MEM_DEVICE) return;
  COMBO_CK(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
}

int grid_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32))); }

}  // namespace

extern "C" {

// fine-image planes [plane0, plane0 + nplanes) (mod dims[0]) of the image
// generate_* / the seeded config generators would produce for the whole
// dims grid (same voxels bit for bit); seed: the generator seed of the
// seeded shapes (4, 10, 11, 12), which ignore params[0]
int combo_generate_planes(combo_ctx* c, int shape, const int64_t dims[3], const double lengths[3],
                          const double* params, int nparams, uint64_t seed, int64_t plane0, int64_t nplanes,
                          uint8_t* out, int mem) {
  return guarded(c, [&] {
    GenArgs g{};
    g.n1 = dims[0];
    g.n2 = dims[1];
    g.n3 = dims[2];
    for (int a = 0; a < 3; ++a) {
      if (dims[a] < 1) throw ComboError(COMBO_ERR_BAD_SHAPE, "generate: dims must be >= 1");
      if (!(lengths[a] > 0.0)) throw ComboError(COMBO_ERR_BAD_SHAPE, "generate: lengths must be positive");
      g.L[a] = lengths[a];
      g.h[a] = lengths[a] / double(dims[a]);
    }
    if (nplanes < 1 || nplanes > dims[0]) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "generate: bad plane window");
    g.plane0 = ((plane0 % dims[0]) + dims[0]) % dims[0];
    g.nplanes = nplanes;
    g.shape = shape;
    for (int i = 0; i < nparams && i < 8; ++i) g.p[i] = params[i];
    const int64_t n = nplanes * g.n2 * g.n3;
    DBuf<uint8_t> tmp;
    uint8_t* d = dev_or_stage(c, out, size_t(n), mem, tmp, false);
    if (shape == 0 || shape == 1 || shape == 2 || shape == 3 || shape == 5) {
      if ((shape == 0 || shape == 1) && g.p[0] < 0.0)
        throw ComboError(COMBO_ERR_BAD_SHAPE, "generate: radius must be >= 0");
      if (shape == 2 && (g.p[0] < 0 || g.p[0] > 2)) throw ComboError(COMBO_ERR_BAD_SHAPE, "fiber: axis must be 0, 1, 2");
      if (shape == 2 && g.p[1] < 0.0) throw ComboError(COMBO_ERR_BAD_SHAPE, "fiber: radius must be >= 0");
      if (shape == 3 && g.p[2] < 1.0) throw ComboError(COMBO_ERR_BAD_SHAPE, "cross_ply: need at least one layer");
      if (shape == 3 && (!(g.p[1] > 0.0) || g.p[0] < 0.0))
        throw ComboError(COMBO_ERR_BAD_SHAPE, "cross_ply: pitch must be > 0 and radius >= 0");
      if (shape == 5 && (g.p[0] < 0 || g.p[0] > 2 || !(g.p[1] >= 0.0 && g.p[1] <= 1.0)))
        throw ComboError(COMBO_ERR_BAD_SHAPE, "slab: bad axis / fraction");
      k_generate<<<grid_for(n), 256, 0, c->stream>>>(g, d);
      ++c->launches;
    } else if (shape == 4) {
      // p = (seed), count, radius, length, orientation_spread
      const int count = int(g.p[1]);
      const double radius = g.p[2], length = g.p[3], spread = g.p[4];
      if (count < 0) throw ComboError(COMBO_ERR_BAD_SHAPE, "fiber_pack: count must be >= 0");
      if (radius < 0.0 || length < 0.0) throw ComboError(COMBO_ERR_BAD_SHAPE, "fiber_pack: radius/length");
      Sm64 rng{seed};
      std::vector<double> fib(size_t(6) * size_t(std::max(count, 1)));
      for (int f = 0; f < count; ++f) {
        double* c = fib.data() + 6 * f;
        c[0] = rng.unit() * g.L[0];
        c[1] = rng.unit() * g.L[1];
        c[2] = rng.unit() * g.L[2];
        double d[3] = {1.0, 0.0, 0.0};
        d[1] = spread * (2.0 * rng.unit() - 1.0);
        d[2] = spread * (2.0 * rng.unit() - 1.0);
        const double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        for (int a = 0; a < 3; ++a) c[3 + a] = d[a] / len;
      }
      DBuf<double> dfib;
      dfib.alloc(fib.size());
      COMBO_CK(cudaMemcpyAsync(dfib.p, fib.data(), fib.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      k_generate_pack<<<grid_for(n), 256, 0, c->stream>>>(g, dfib.p, count, 0.5 * length, radius, d);
      ++c->launches;
      COMBO_CK(cudaGetLastError());
      COMBO_CK(cudaStreamSynchronize(c->stream));
    } else if (shape >= 10 && shape <= 12) {
      std::vector<Obj> all;
      if (shape == 10) all = rsa(g, seed, g.p[1], g.p[2], g.p[3], false);
      if (shape == 11) all = rsa(g, seed, g.p[1], g.p[1], g.p[2], true);
      if (shape == 12) all = boolean_ellipsoids(g, seed, g.p[1], g.p[2], g.p[3]);
      // objects whose plane range (k_raster's, widened by one plane for the
      // host rounding) meets the window
      std::vector<Obj> objs;
      if (nplanes == g.n1) {
        objs.swap(all);
      } else {
        for (const Obj& o : all) {
          const int64_t a = int64_t(std::floor((o.c[0] - o.r) / g.h[0])) - 2;
          const int64_t b = int64_t(std::floor((o.c[0] + o.r) / g.h[0])) + 2;
          bool hit = b - a + 1 >= g.n1;
          for (int64_t i = a; i <= b && !hit; ++i) {
            const int64_t li = (((i - g.plane0) % g.n1) + g.n1) % g.n1;
            hit = li < nplanes;
          }
          if (hit) objs.push_back(o);
        }
      }
      COMBO_CK(cudaMemsetAsync(d, 0, size_t(n), c->stream));
      DBuf<Obj> dobj;
      dobj.alloc(objs.size());
      COMBO_CK(cudaMemcpyAsync(dobj.p, objs.data(), objs.size() * sizeof(Obj), cudaMemcpyHostToDevice, c->stream));
      const int64_t blocks = std::min<int64_t>(int64_t(objs.size()), 148 * 64);
      if (blocks > 0) {
        k_raster<<<unsigned(blocks), 256, 0, c->stream>>>(dobj.p, int64_t(objs.size()), g.n1, g.n2, g.n3, g.L[0],
                                                          g.L[1], g.L[2], g.h[0], g.h[1], g.h[2], g.plane0,
                                                          g.nplanes, d);
        ++c->launches;
      }
      COMBO_CK(cudaStreamSynchronize(c->stream));
    } else {
      throw ComboError(COMBO_ERR_BAD_SHAPE, "generate: unsupported shape id");
    }
    COMBO_CK(cudaGetLastError());
    copy_back(c, out, d, size_t(n), mem);
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

// the whole image; seeded shapes take the seed from params[0]
int combo_generate(combo_ctx* c, int shape, const int64_t dims[3], const double lengths[3], const double* params,
                   int nparams, uint8_t* out, int mem) {
  const uint64_t seed = (nparams > 0 && params && params[0] >= 0.0) ? uint64_t(params[0]) : 0;
  return combo_generate_planes(c, shape, dims, lengths, params, nparams, seed, 0, dims ? dims[0] : 1, out, mem);
}

int combo_coarsen(combo_ctx* c, const uint8_t* img, const int64_t dims[3], const int64_t factors[3], uint8_t* kind,
                  double* c_plus, int64_t* count_plus, int mem) {
  return guarded(c, [&] {
    int64_t b[3];
    for (int a = 0; a < 3; ++a) {
      if (factors[a] < 1 || dims[a] % factors[a] != 0)
        throw ComboError(COMBO_ERR_NON_DIVIDING_FACTOR, "coarsen: factor does not divide image dims");
      b[a] = dims[a] / factors[a];
    }
    const int64_t n = dims[0] * dims[1] * dims[2], nb = b[0] * b[1] * b[2];
    DBuf<uint8_t> ti, tk;
    DBuf<double> tc;
    DBuf<int64_t> tn;
    const uint8_t* di = dev_or_stage(c, const_cast<uint8_t*>(img), size_t(n), mem, ti, true);
    uint8_t* dk = dev_or_stage(c, kind, size_t(nb), mem, tk, false);
    double* dc = dev_or_stage(c, c_plus, size_t(nb), mem, tc, false);
    int64_t* dn = dev_or_stage(c, count_plus, size_t(nb), mem, tn, false);
    ImgView im{di, dims[0], dims[1], dims[2], 0, 0, 0};
    k_coarsen<<<grid_for(nb), 256, 0, c->stream>>>(im, factors[0], factors[1], factors[2], b[0], b[1], b[2], dk, dc, dn);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    copy_back(c, kind, dk, size_t(nb), mem);
    copy_back(c, c_plus, dc, size_t(nb), mem);
    copy_back(c, count_plus, dn, size_t(nb), mem);
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

int combo_laplace_weights(combo_ctx* c, const uint8_t* img, const int64_t dims[3], const double lengths[3], double* w,
                          int mem) {
  return guarded(c, [&] {
    const int64_t n = dims[0] * dims[1] * dims[2];
    DBuf<uint8_t> ti;
    DBuf<double> tw;
    const uint8_t* di = dev_or_stage(c, const_cast<uint8_t*>(img), size_t(n), mem, ti, true);
    double* dw = dev_or_stage(c, w, size_t(n), mem, tw, false);
    const double h1 = lengths[0] / double(dims[0]), h2 = lengths[1] / double(dims[1]), h3 = lengths[2] / double(dims[2]);
    ImgView im{di, dims[0], dims[1], dims[2], h1, h2, h3};
    k_laplace<<<grid_for(n), 256, 0, c->stream>>>(im, h2 * h3 / h1, h1 * h3 / h2, h1 * h2 / h3, dw);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    copy_back(c, w, dw, size_t(n), mem);
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

// compute_normals (normals.cpp:211-256) for boxel planes [bp0, bp0 + nbp) of
// the grid of a dims image, from an image window of planes [img0, img0 +
// img_planes) (mod dims[0]) that covers the boxels' fine planes plus one
// halo plane on each side for the second-moment method (the whole image
// qualifies). kind / normal3 / flags: the nbp boxel planes.
int combo_normals_slab(combo_ctx* c, const uint8_t* img, int64_t img0, int64_t img_planes, const int64_t dims[3],
                       const double lengths[3], const int64_t factors[3], int64_t bp0, int64_t nbp,
                       const uint8_t* kind, int method, int centering, int min_support, double* normal3,
                       uint8_t* flags, combo_normal_stats* stats, int mem) {
  return guarded(c, [&] {
    int64_t b[3];
    for (int a = 0; a < 3; ++a) {
      if (factors[a] < 1 || dims[a] % factors[a] != 0)
        throw ComboError(COMBO_ERR_NON_DIVIDING_FACTOR, "normals: factor does not divide image dims");
      b[a] = dims[a] / factors[a];
    }
    if (nbp < 1 || bp0 < 0 || bp0 + nbp > b[0] || img_planes < 1 || img_planes > dims[0])
      throw ComboError(COMBO_ERR_BAD_ARGUMENT, "normals: bad plane window");
    const int64_t w0 = ((img0 % dims[0]) + dims[0]) % dims[0];
    if (img_planes < dims[0]) {
      // fine planes the kernel reads: the boxels' own, +-1 for the stencil
      const int64_t need0 = bp0 * factors[0] - (method == 1 ? 1 : 0);
      const int64_t need1 = (bp0 + nbp) * factors[0] + (method == 1 ? 1 : 0);
      for (int64_t i = need0; i < need1; ++i) {
        const int64_t li = (((i - w0) % dims[0]) + dims[0]) % dims[0];
        if (li >= img_planes) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "normals: image window misses a needed plane");
      }
    }
    const int64_t n = img_planes * dims[1] * dims[2], nb = nbp * b[1] * b[2];
    DBuf<uint8_t> ti, tk, tf;
    DBuf<double> tn;
    const uint8_t* di = dev_or_stage(c, const_cast<uint8_t*>(img), size_t(n), mem, ti, true);
    const uint8_t* dk = dev_or_stage(c, const_cast<uint8_t*>(kind), size_t(nb), mem, tk, true);
    double* dn = dev_or_stage(c, normal3, size_t(3 * nb), mem, tn, false);
    uint8_t* df = dev_or_stage(c, flags, size_t(nb), mem, tf, false);
    COMBO_CK(cudaMemsetAsync(dn, 0, size_t(3 * nb) * 8, c->stream));
    COMBO_CK(cudaMemsetAsync(df, 0, size_t(nb), c->stream));
    DBuf<unsigned long long> ds;
    ds.alloc(3);
    COMBO_CK(cudaMemsetAsync(ds.p, 0, 24, c->stream));
    NormalArgs A{};
    const double h1 = lengths[0] / double(dims[0]), h2 = lengths[1] / double(dims[1]), h3 = lengths[2] / double(dims[2]);
    A.im = ImgView{di, dims[0], dims[1], dims[2], h1, h2, h3, w0};
    A.f1 = factors[0];
    A.f2 = factors[1];
    A.f3 = factors[2];
    A.b1 = b[0];
    A.b2 = b[1];
    A.b3 = b[2];
    A.bp0 = bp0;
    A.nbp = nbp;
    A.bl0 = lengths[0] / double(b[0]);
    A.bl1 = lengths[1] / double(b[1]);
    A.bl2 = lengths[2] / double(b[2]);
    A.r1 = h2 * h3 / h1;
    A.r2 = h1 * h3 / h2;
    A.r3 = h1 * h2 / h3;
    A.method = method;
    A.centering = centering;
    A.min_support = min_support;
    k_normals<<<grid_for(nb), 128, 0, c->stream>>>(A, dk, dn, df, ds.p);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    copy_back(c, normal3, dn, size_t(3 * nb), mem);
    copy_back(c, flags, df, size_t(nb), mem);
    unsigned long long hs[3];
    COMBO_CK(cudaMemcpyAsync(hs, ds.p, 24, cudaMemcpyDeviceToHost, c->stream));
    COMBO_CK(cudaStreamSynchronize(c->stream));
    if (stats) {
      stats->composite = int64_t(hs[0]);
      stats->degenerate_fallbacks = int64_t(hs[1]);
      stats->too_few_fallbacks = int64_t(hs[2]);
    }
  });
}

int combo_normals(combo_ctx* c, const uint8_t* img, const int64_t dims[3], const double lengths[3],
                  const int64_t factors[3], const uint8_t* kind, int method, int centering, int min_support,
                  double* normal3, uint8_t* flags, combo_normal_stats* stats, int mem) {
  if (!dims || !factors || factors[0] < 1 || dims[0] % factors[0] != 0) {
    if (c) c->err = "normals: factor does not divide image dims";
    return COMBO_ERR_NON_DIVIDING_FACTOR;
  }
  return combo_normals_slab(c, img, 0, dims[0], dims, lengths, factors, 0, dims[0] / factors[0], kind, method,
                            centering, min_support, normal3, flags, stats, mem);
}

int combo_laminate_solve(combo_ctx* c, const double fbox[9], const combo_law* plus, const combo_law* minus,
                         const double normal[3], double c_plus, const double a0[3], const combo_laminate_opts* lam,
                         double p9[9], double a3[3], int istate[4]) {
  return guarded(c, [&] {
    combo_dev::MatParams M{};
    DBuf<double> a9;
    a9.alloc(162);
    M.law[1] = combo_host::law_params(*plus, a9.p);
    M.law[0] = combo_host::law_params(*minus, a9.p + 81);
    combo_laminate_opts o{0.0, 1e-10, 0.0, 50, 1, 0.0};
    if (lam) o = *lam;
    M.lam.tol_abs = o.tol_abs;
    M.lam.tol_rel = o.tol_rel;
    M.lam.stress_floor = o.stress_floor;
    M.lam.max_iter = o.max_iter;
    M.lam.back_projection = o.back_projection;
    const double len = std::sqrt(normal[0] * normal[0] + normal[1] * normal[1] + normal[2] * normal[2]);
    double in[16];
    std::memcpy(in, fbox, 72);
    for (int i = 0; i < 3; ++i) in[9 + i] = normal[i] / len;
    in[12] = c_plus;
    for (int i = 0; i < 3; ++i) in[13 + i] = a0[i];
    DBuf<double> din, dout;
    DBuf<int> dist;
    din.alloc(16);
    dout.alloc(12);
    dist.alloc(4);
    COMBO_CK(cudaMemcpy(din.p, in, sizeof in, cudaMemcpyHostToDevice));
    k_laminate_one<<<1, 1, 0, c->stream>>>(M, din.p, dout.p, dist.p);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    double out[12];
    COMBO_CK(cudaMemcpyAsync(out, dout.p, sizeof out, cudaMemcpyDeviceToHost, c->stream));
    COMBO_CK(cudaMemcpyAsync(istate, dist.p, 16, cudaMemcpyDeviceToHost, c->stream));
    COMBO_CK(cudaStreamSynchronize(c->stream));
    std::memcpy(p9, out, 72);
    std::memcpy(a3, out + 9, 24);
    if (istate[3]) throw ComboError(COMBO_ERR_INADMISSIBLE_MACRO, "admissibility_bounds: det(F_box) <= 0");
  });
}

}  // extern "C"
