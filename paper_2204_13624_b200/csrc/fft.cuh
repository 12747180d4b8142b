// Hand-written fp64 batched 3D r2c/c2r FFT fused with the Gamma^0 projector.
//
// Replaces Fft3 (reference src/fft.cpp:23-60, FFTW many-plans) and
// GreenOperator::apply_fourier / project (src/green.cpp:59-151).
//
// Layout: real fields are component-major SoA [c][i][j][k] (field.hpp:32-70).
// The half spectrum is [c][i][j][k3] with k3 < n3/2+1 and a padded row
// stride n3p (multiple of 8 complex -> 128-byte aligned rows).
//
// Passes (each one HBM read + one HBM write of the spectrum):
//   Z-fwd : per tile of z-lines; a producer functor computes the 9 real
//           values of every cell; pairs of real lines are packed into one
//           complex line, transformed, and split into two half spectra.
//   Y     : per (component, k1-plane, column tile), c2c along axis 1.
//   X+G   : per (row group i, k2, column tile) the 3 components tau_i1..i3,
//           c2c along axis 0, Gamma applied per k-point, inverse c2c.
//   Y^-1, Z-inv : mirror images; Z-inv hands the real values (already scaled
//           by 1/n like fft.cpp:54-60) to a consumer functor.
// Line transforms run in shared memory as Stockham stages whose radix
// sequence is fixed at compile time from log2(n) (8,8,...,4/2); each thread
// holds one radix-8 butterfly (8 complex values) in registers across the
// stage barrier, so the transform is in place and the block size is tile/8.
// Non-power-of-two sizes (small test grids) take a runtime mixed-radix path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace combo_dev {

constexpr int kMaxFftThreads = 768;  // block size = tile / 8, <= 768
constexpr int kMaxRad = 16;
constexpr int kElems = 8;  // complex values held per thread per stage
constexpr int kGeneric = -1;

struct Axis {
  int n;
  int nrad;
  int rad[kMaxRad];
  const double2* tw;  // exp(-2 pi i k / n), k < n (host long double, rounded)
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 rot(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(double2* v) {
  const double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
template <bool INV>
__device__ __forceinline__ void dft4(double2* v) {
  const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  const double2 b0 = cadd(v[1], v[3]), b1 = rot<INV>(csub(v[1], v[3]));
  v[0] = cadd(a0, b0);
  v[2] = csub(a0, b0);
  v[1] = cadd(a1, b1);
  v[3] = csub(a1, b1);
}
template <bool INV>
__device__ __forceinline__ void dft8(double2* v) {
  constexpr double r2 = 0.70710678118654752440;
  const double2 a0 = cadd(v[0], v[4]), a1 = csub(v[0], v[4]);
  const double2 a2 = cadd(v[2], v[6]), a3 = rot<INV>(csub(v[2], v[6]));
  const double2 a4 = cadd(v[1], v[5]), a5 = csub(v[1], v[5]);
  const double2 a6 = cadd(v[3], v[7]), a7 = rot<INV>(csub(v[3], v[7]));
  const double2 e0 = cadd(a0, a2), e2 = csub(a0, a2), e1 = cadd(a1, a3), e3 = csub(a1, a3);
  const double2 o0 = cadd(a4, a6), o2 = rot<INV>(csub(a4, a6)), o1 = cadd(a5, a7), o3 = csub(a5, a7);
  // W8 = (1 -/+ i)/sqrt2 ; W8^3 = (-1 -/+ i)/sqrt2
  const double2 w1o1 = INV ? make_double2(r2 * (o1.x - o1.y), r2 * (o1.x + o1.y))
                           : make_double2(r2 * (o1.x + o1.y), r2 * (o1.y - o1.x));
  const double2 w3o3 = INV ? make_double2(-r2 * (o3.x + o3.y), r2 * (o3.x - o3.y))
                           : make_double2(r2 * (o3.y - o3.x), -r2 * (o3.x + o3.y));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[2] = cadd(e2, o2);
  v[6] = csub(e2, o2);
  v[1] = cadd(e1, w1o1);
  v[5] = csub(e1, w1o1);
  v[3] = cadd(e3, w3o3);
  v[7] = csub(e3, w3o3);
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2* v) {
  if constexpr (R == 2) dft2<INV>(v);
  if constexpr (R == 4) dft4<INV>(v);
  if constexpr (R == 8) dft8<INV>(v);
}

// ------------------------------------------------ compile-time pow2 stages
// radix sequence for n = 2^L: 8...8 then (4) or (4,4); n = 2 -> (2)
__host__ __device__ constexpr int pow2_nstages(int L) {
  return L == 0 ? 0 : (L == 1 ? 1 : (L % 3 == 0 ? L / 3 : L / 3 + 1));
}
__host__ __device__ constexpr int pow2_radix(int L, int s) {
  if (L == 1) return 2;
  const int k8 = L / 3, rem = L % 3;
  if (rem == 0) return 8;
  if (rem == 2) return s < k8 ? 8 : 4;
  return s < k8 - 1 ? 8 : 4;  // rem == 1, L >= 4: 8^(k8-1) 4 4
}

// One Stockham stage: buf[line*ls + e*es]; compile-time n, R, P (span).
// LF: consecutive threads -> consecutive lines (column tiles).
template <int N, int R, int P, bool INV, bool LF>
__device__ __forceinline__ void stage_ct(double2* buf, int nl, int es, int ls, const double2* __restrict__ tw) {
  constexpr int B = kElems / R;
  constexpr int M = N / R;
  constexpr int TS = N / (P * R);
  const int total = M * nl;
  const int tid = threadIdx.x, nthr = blockDim.x;
  double2 v[B][R];
  int lines[B], ts[B];
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int b = tid + q * nthr;
    lines[q] = -1;
    ts[q] = 0;
    if (b < total) {
      int line, t;
      if (LF) {
        line = b % nl;
        t = b / nl;
      } else {
        t = b % M;
        line = b / M;
      }
      lines[q] = line;
      ts[q] = t;
      const double2* base = buf + line * ls;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = base[(t + r * M) * es];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < B; ++q) {
    if (lines[q] >= 0) {
      const int t = ts[q];
      const int k = t % P;
      if constexpr (P > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = __ldg(tw + r * k * TS);
          if (INV) w.y = -w.y;
          v[q][r] = cmul(v[q][r], w);
        }
      }
      dftR<R, INV>(v[q]);
      const int j = (t - k) * R + k;
      double2* base = buf + lines[q] * ls;
#pragma unroll
      for (int r = 0; r < R; ++r) base[(j + r * P) * es] = v[q][r];
    }
  }
  __syncthreads();
}

template <int L, int S, int P, bool INV, bool LF>
__device__ __forceinline__ void pow2_stages(double2* buf, int nl, int es, int ls, const double2* tw) {
  if constexpr (S < pow2_nstages(L)) {
    constexpr int R = pow2_radix(L, S);
    stage_ct<(1 << L), R, P, INV, LF>(buf, nl, es, ls, tw);
    pow2_stages<L, S + 1, P * R, INV, LF>(buf, nl, es, ls, tw);
  }
}

// ------------------------------------------------- runtime mixed radix
template <bool INV, bool LF>
__device__ __noinline__ void stage_generic(double2* buf, int R, int n, int nl, int es, int ls, int p,
                                           const double2* __restrict__ tw) {
  constexpr int MAXV = 72;
  const int m = n / R;
  const int total = m * nl;
  const int tid = threadIdx.x, nthr = blockDim.x;
  double2 v[MAXV];
  int cnt = 0;
  for (int b = tid; b < total && cnt + R <= MAXV; b += nthr) {
    const int line = LF ? b % nl : b / m;
    const int t = LF ? b / nl : b % m;
    for (int r = 0; r < R; ++r) v[cnt + r] = buf[line * ls + (t + r * m) * es];
    cnt += R;
  }
  __syncthreads();
  cnt = 0;
  const int tstride = n / (p * R);
  const int wstep = n / R;
  for (int b = tid; b < total && cnt + R <= MAXV; b += nthr) {
    const int line = LF ? b % nl : b / m;
    const int t = LF ? b / nl : b % m;
    const int k = t % p;
    for (int r = 1; r < R; ++r) {
      double2 w = tw[r * k * tstride];
      if (INV) w.y = -w.y;
      v[cnt + r] = cmul(v[cnt + r], w);
    }
    double2 out[64];
    for (int s = 0; s < R; ++s) {
      double2 acc = make_double2(0.0, 0.0);
      for (int r = 0; r < R; ++r) {
        double2 w = tw[((r * s) % R) * wstep];
        if (INV) w.y = -w.y;
        acc = cadd(acc, cmul(v[cnt + r], w));
      }
      out[s] = acc;
    }
    const int j = (t - k) * R + k;
    for (int r = 0; r < R; ++r) buf[line * ls + (j + r * p) * es] = out[r];
    cnt += R;
  }
  __syncthreads();
}

// Transform nl lines of length ax.n held in shared memory (in place).
template <int L, bool INV, bool LF>
__device__ __forceinline__ void fft_lines(double2* buf, const Axis& ax, int nl, int es, int ls) {
  if constexpr (L >= 0) {
    pow2_stages<L, 0, 1, INV, LF>(buf, nl, es, ls, ax.tw);
  } else {
    int p = 1;
    for (int s = 0; s < ax.nrad; ++s) {
      const int R = ax.rad[s];
      stage_generic<INV, LF>(buf, R, ax.n, nl, es, ls, p, ax.tw);
      p *= R;
    }
  }
}

// --------------------------------------------------------- reductions
// Deterministic block reduction of NRED per-thread accumulators into
// partials[blockIdx.x * NRED + r] (fixed shuffle tree + warp order).
template <int NRED>
__device__ void block_reduce_store(double (&acc)[NRED], double* partials, int64_t block) {
  if constexpr (NRED > 0) {
    __shared__ double red[32][NRED > 0 ? NRED : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < NRED; ++r) {
      double v = acc[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][r] = v;
    }
    __syncthreads();
    if (threadIdx.x < NRED) {
      double s = 0.0;
      const int nw = (blockDim.x + 31) >> 5;
      for (int w = 0; w < nw; ++w) s += red[w][threadIdx.x];
      partials[block * NRED + threadIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------- passes
// Half spectrum: rows of n3p complex.
//
// Single slab (blocked = 0): row (c, i, j) at c cs + i si + j sj, with
// i-major (si = n2 n3p, sj = n3p) or j-major (si = n3p, sj = n1 n3p) rows.
//
// Slab decomposition over R ranks (blocked = 1; ni = n1 / R planes per slab,
// nj = n2 / R k2-columns per pencil): the slab side (z and y passes) keeps
// planes [i0, i0 + ni) of every k2 and stores them blocked by destination
// pencil s = j / nj:  A(c, il, j) = s blk + c cs + (il nj + j mod nj) n3p;
// the pencil side (x pass + Gamma) keeps k2 in [j0, j0 + nj) of every plane,
// blocked by source slab r = i / ni:  B(c, i, jl) = r blk + c cs +
// ((i mod ni) nj + jl) n3p, with blk = 9 ni nj n3p and cs = ni nj n3p. Block s
// of A on rank q is block q of B on rank s, so the transpose is one
// all-to-all of equal contiguous blocks; with R = 1 both reduce to the
// i-major single-slab layout.
struct SpecView {
  double2* spec;
  int64_t n1, n2, n3, n3c, n3p;  // global grid, row length
  int64_t cs;                    // component stride
  int64_t si, sj;                // single-slab row strides
  int64_t ni, nj, i0, j0, blk;   // slab / pencil extents and offsets
  int blocked;
  int swap;  // blocked: rows j-major inside each block (x lines contiguous), else i-major
  // slab side: local plane il, global k2 j
  __host__ __device__ __forceinline__ int64_t rowA(int64_t il, int64_t j) const {
    if (!blocked) return il * si + j * sj;
    const int s = int(j) / int(nj);
    const int64_t jl = j - int64_t(s) * nj;
    return s * blk + (swap ? jl * ni + il : il * nj + jl) * n3p;
  }
  // pencil side: global plane i, local k2 jl
  __host__ __device__ __forceinline__ int64_t rowB(int64_t i, int64_t jl) const {
    if (!blocked) return i * si + jl * sj;
    const int r = int(i) / int(ni);
    const int64_t il = i - int64_t(r) * ni;
    return r * blk + (swap ? jl * ni + il : il * nj + jl) * n3p;
  }
  // row of component c on local z-line `line` = il n2 + j
  __host__ __device__ __forceinline__ int64_t zrow(int64_t c, int64_t line) const {
    const int64_t il = line / n2;
    return c * cs + rowA(il, line - il * n2);
  }
};

template <int LOG2N>
__device__ __forceinline__ int line_len(const Axis& ax) {
  if constexpr (LOG2N >= 0)
    return 1 << LOG2N;
  else
    return ax.n;
}

// Z-forward: producer(cell, v[9], acc) -> spectrum. L z-lines per block.
template <class Prod, int LOG2N>
static __global__ void __launch_bounds__(kMaxFftThreads)
    zfwd_kernel(SpecView sv, Axis ax, int L, int ls, Prod prod, double* partials) {
  extern __shared__ double2 sm[];
  const int n = line_len<LOG2N>(ax);
  const int64_t nlines_tot = sv.ni * sv.n2;  // local z-lines
  const int64_t line0 = int64_t(blockIdx.x) * L;
  const int nlines = int(min(int64_t(L), nlines_tot - line0));
  const int nreal = 9 * nlines;
  const int npair = (nreal + 1) >> 1;
  constexpr int NR = Prod::NRED > 0 ? Prod::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = 0.0;
  for (int t = threadIdx.x; t < nlines * n; t += blockDim.x) {
    const int li = t / n, k = t - li * n;
    const int64_t cell = (line0 + li) * n + k;
    double v[9];
    prod(cell, v, acc);
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const int rl = li * 9 + c;
      reinterpret_cast<double*>(sm + (rl >> 1) * ls + k)[rl & 1] = v[c];
    }
  }
  if (nreal & 1)
    for (int k = threadIdx.x; k < n; k += blockDim.x) reinterpret_cast<double*>(sm + (npair - 1) * ls + k)[1] = 0.0;
  __syncthreads();
  fft_lines<LOG2N, false, false>(sm, ax, npair, 1, ls);
  const int nc = int(sv.n3c);
  for (int t = threadIdx.x; t < npair * nc; t += blockDim.x) {
    const int pp = t / nc, k = t - pp * nc;
    const double2 zk = sm[pp * ls + k];
    const double2 zm = sm[pp * ls + (k == 0 ? 0 : n - k)];
    int rl = 2 * pp;
    int li = rl / 9, c = rl - 9 * li;
    sv.spec[sv.zrow(c, line0 + li) + k] =
        make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    ++rl;
    if (rl < nreal) {
      li = rl / 9;
      c = rl - 9 * li;
      sv.spec[sv.zrow(c, line0 + li) + k] =
          make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    }
  }
  if constexpr (Prod::NRED > 0) block_reduce_store<Prod::NRED>(acc, partials, blockIdx.x);
}

// Z-inverse: spectrum -> consumer(cell, v[9] (scaled by 1/n_total), acc)
template <class Cons, int LOG2N>
static __global__ void __launch_bounds__(kMaxFftThreads)
    zinv_kernel(SpecView sv, Axis ax, int L, int ls, double scale, Cons cons, double* partials) {
  extern __shared__ double2 sm[];
  const int n = line_len<LOG2N>(ax);
  const int64_t nlines_tot = sv.ni * sv.n2;  // local z-lines
  const int64_t line0 = int64_t(blockIdx.x) * L;
  const int nlines = int(min(int64_t(L), nlines_tot - line0));
  const int nreal = 9 * nlines;
  const int npair = (nreal + 1) >> 1;
  const int nc = int(sv.n3c);
  for (int t = threadIdx.x; t < npair * nc; t += blockDim.x) {
    const int pp = t / nc, k = t - pp * nc;
    int rl = 2 * pp;
    int li = rl / 9, c = rl - 9 * li;
    double2 xa = sv.spec[sv.zrow(c, line0 + li) + k];
    double2 xb = make_double2(0.0, 0.0);
    ++rl;
    if (rl < nreal) {
      li = rl / 9;
      c = rl - 9 * li;
      xb = sv.spec[sv.zrow(c, line0 + li) + k];
    }
    const bool selfconj = (k == 0) || (2 * k == n);
    if (selfconj) {
      // halfcomplex c2r: imaginary parts of DC / Nyquist are ignored
      xa.y = 0.0;
      xb.y = 0.0;
    }
    sm[pp * ls + k] = make_double2(xa.x - xb.y, xa.y + xb.x);
    if (!selfconj) sm[pp * ls + (n - k)] = make_double2(xa.x + xb.y, xb.x - xa.y);
  }
  __syncthreads();
  fft_lines<LOG2N, true, false>(sm, ax, npair, 1, ls);
  constexpr int NR = Cons::NRED > 0 ? Cons::NRED : 1;
  double acc[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = 0.0;
  for (int t = threadIdx.x; t < nlines * n; t += blockDim.x) {
    const int li = t / n, k = t - li * n;
    const int64_t cell = (line0 + li) * n + k;
    double v[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const int rl = li * 9 + c;
      v[c] = reinterpret_cast<const double*>(sm + (rl >> 1) * ls + k)[rl & 1] * scale;
    }
    cons(cell, v, acc);
  }
  if constexpr (Cons::NRED > 0) block_reduce_store<Cons::NRED>(acc, partials, blockIdx.x);
}

// Y pass: c2c along axis 1; grid (column tiles, n1, ncomp)
template <int LOG2N, bool INV>
static __global__ void __launch_bounds__(kMaxFftThreads) ypass_kernel(SpecView sv, Axis ax, int W) {
  extern __shared__ double2 sm[];
  const int n2 = line_len<LOG2N>(ax);
  const int c = blockIdx.z, i = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  double2* base = sv.spec + int64_t(c) * sv.cs + kc0;
  for (int t = threadIdx.x; t < n2 * W; t += blockDim.x) {
    const int j = t / W, col = t - j * W;
    if (col < w) sm[t] = base[sv.rowA(i, j) + col];
  }
  __syncthreads();
  fft_lines<LOG2N, INV, true>(sm, ax, W, W, 1);
  for (int t = threadIdx.x; t < n2 * W; t += blockDim.x) {
    const int j = t / W, col = t - j * W;
    if (col < w) base[sv.rowA(i, j) + col] = sm[t];
  }
}

// Green operator symbol tables (green.cpp:16-57), computed on the host.
struct GreenTables {
  int kind;  // 0 continuous, 1 rotated, 2 staggered
  const double2* fwd[3];
  const double2* avg[3];
  const double* xi[3];
};

// Gamma row i applied to (t1, t2, t3) = tau_i1..i3 at (k1, k2, k3)
// (green.cpp:67-130).
__device__ __forceinline__ void gamma_row(const GreenTables& G, int row, int64_t k1, int64_t k2, int64_t k3,
                                          int64_t n1, int64_t n2, int64_t n3, double2* t) {
  double2 g[3];
  if (G.kind == 0) {
    if (2 * k1 == n1 || 2 * k2 == n2 || 2 * k3 == n3) {
      t[0] = t[1] = t[2] = make_double2(0.0, 0.0);
      return;
    }
    g[0] = make_double2(0.0, G.xi[0][k1]);
    g[1] = make_double2(0.0, G.xi[1][k2]);
    g[2] = make_double2(0.0, G.xi[2][k3]);
  } else if (G.kind == 1) {
    const double2 a1 = G.avg[0][k1], a2 = G.avg[1][k2], a3 = G.avg[2][k3];
    g[0] = cmul(cmul(G.fwd[0][k1], a2), a3);
    g[1] = cmul(cmul(G.fwd[1][k2], a1), a3);
    g[2] = cmul(cmul(G.fwd[2][k3], a1), a2);
  } else {
    g[0] = G.fwd[0][k1];
    g[1] = G.fwd[1][k2];
    g[2] = G.fwd[2][k3];
  }
  const double den = (g[0].x * g[0].x + g[0].y * g[0].y) + (g[1].x * g[1].x + g[1].y * g[1].y) +
                     (g[2].x * g[2].x + g[2].y * g[2].y);
  if (den == 0.0) {
    t[0] = t[1] = t[2] = make_double2(0.0, 0.0);
    return;
  }
  double2 gr[3];
#pragma unroll
  for (int J = 0; J < 3; ++J) gr[J] = (G.kind == 2 && J != row) ? make_double2(-g[J].x, g[J].y) : g[J];
  double sx = 0.0, sy = 0.0;
#pragma unroll
  for (int L = 0; L < 3; ++L) {
    // conj(gr) * t
    sx += gr[L].x * t[L].x + gr[L].y * t[L].y;
    sy += gr[L].x * t[L].y - gr[L].y * t[L].x;
  }
  sx /= den;
  sy /= den;
  const double2 s = make_double2(sx, sy);
#pragma unroll
  for (int J = 0; J < 3; ++J) t[J] = cmul(gr[J], s);
}

// X pass fused with Gamma: grid (column tiles, n2, 3 row groups)
template <int LOG2N>
static __global__ void __launch_bounds__(kMaxFftThreads) xgamma_kernel(SpecView sv, Axis ax, int W, GreenTables G,
                                                                       int rg0) {
  extern __shared__ double2 sm[];
  const int n1 = line_len<LOG2N>(ax);
  const int rg = rg0 + blockIdx.z, j = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  const int W3 = 3 * W;
  const int64_t plane = sv.cs;  // component stride
  double2* base = sv.spec + int64_t(3 * rg) * plane + kc0;  // pencil side, local k2 j
  for (int t = threadIdx.x; t < n1 * W3; t += blockDim.x) {
    const int i = t / W3, rem = t - i * W3, cc = rem / W, col = rem - cc * W;
    if (col < w) sm[t] = base[int64_t(cc) * plane + sv.rowB(i, j) + col];
  }
  __syncthreads();
  fft_lines<LOG2N, false, true>(sm, ax, W3, W3, 1);
  for (int t = threadIdx.x; t < n1 * W; t += blockDim.x) {
    const int k1 = t / W, col = t - k1 * W;
    if (col < w) {
      double2 v[3];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) v[cc] = sm[k1 * W3 + cc * W + col];
      gamma_row(G, rg, k1, sv.j0 + j, kc0 + col, sv.n1, sv.n2, sv.n3, v);
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) sm[k1 * W3 + cc * W + col] = v[cc];
    }
  }
  __syncthreads();
  fft_lines<LOG2N, true, true>(sm, ax, W3, W3, 1);
  for (int t = threadIdx.x; t < n1 * W3; t += blockDim.x) {
    const int i = t / W3, rem = t - i * W3, cc = rem / W, col = rem - cc * W;
    if (col < w) base[int64_t(cc) * plane + sv.rowB(i, j) + col] = sm[t];
  }
}

// Plain X pass (no Gamma), used by the raw FFT test entry point.
template <int LOG2N, bool INV>
static __global__ void __launch_bounds__(kMaxFftThreads) xpass_kernel(SpecView sv, Axis ax, int W) {
  extern __shared__ double2 sm[];
  const int n1 = line_len<LOG2N>(ax);
  const int c = blockIdx.z, j = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  double2* base = sv.spec + int64_t(c) * sv.cs + kc0;
  for (int t = threadIdx.x; t < n1 * W; t += blockDim.x) {
    const int i = t / W, col = t - i * W;
    if (col < w) sm[t] = base[sv.rowB(i, j) + col];
  }
  __syncthreads();
  fft_lines<LOG2N, INV, true>(sm, ax, W, W, 1);
  for (int t = threadIdx.x; t < n1 * W; t += blockDim.x) {
    const int i = t / W, col = t - i * W;
    if (col < w) base[sv.rowB(i, j) + col] = sm[t];
  }
}

}  // namespace combo_dev
