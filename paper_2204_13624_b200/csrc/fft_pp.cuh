// Persistent, double-buffered versions of the register-resident passes.
//
// Each block loops over tiles (tile = blockIdx.x + k * gridDim.x, a static
// assignment, so reductions stay deterministic). The global->shared copy of
// the next tile is issued with cp.async (LDGSTS, 16 B) before the current
// tile is transformed, so HBM reads are continuously in flight while the FP64
// butterflies and the shared-memory exchanges of the current tile run. The
// tile buffer doubles as the exchange buffer once its stage-0 operands are in
// registers. Outputs are stored straight from registers.
#pragma once

#include "fft_rr.cuh"

namespace combo_dev {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// --------------------------------------------------------------- Y pass
// tile = (column tile kt, plane i, component c); buffer [pad8(row)][W]
template <int L, bool INV>
static __global__ void __launch_bounds__(512, 1) ypass_pp(SpecView sv, const double2* __restrict__ tw, int W,
                                                          int64_t ntiles, int bufsz) {
  constexpr int N = 1 << L;
  extern __shared__ double2 sm[];
  const int ntk = int((sv.n3c + W - 1) / W);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  auto base_of = [&](int64_t tile, int& w) {
    const int kt = int(tile % ntk);
    const int64_t rest = tile / ntk;
    const int64_t i = rest % sv.n1, c = rest / sv.n1;
    w = min(W, int(sv.n3c) - kt * W);
    return sv.spec + c * sv.cs + i * sv.si + int64_t(kt) * W;
  };
  auto prefetch = [&](double2* buf, int64_t tile) {
    int w;
    const double2* g = base_of(tile, w);
    for (int idx = threadIdx.x; idx < N * W; idx += blockDim.x) {
      const int row = idx / W, col = idx - row * W;
      if (col < w) cp_async16(buf + pad8(row) * W + col, g + int64_t(row) * sv.sj + col);
    }
    cp_async_commit();
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prefetch(sm, tile);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double2* buf = sm + (it & 1) * bufsz;
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) {
      prefetch(sm + ((it + 1) & 1) * bufsz, next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    int w;
    double2* g = base_of(tile, w);
    const bool active = line < w && u < N / 8;
    double2 v[1][8];
    if (active) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[0][q] = buf[pad8(rr_first_pos<L, false>(u, q)) * W + line];
    }
    __syncthreads();
    auto addr = [&](int, int pos) { return pad8(pos) * W + line; };
    rr_stages<L, INV, false, 0, 1>(v, u, active, buf, tw, addr);
    if (active) {
#pragma unroll
      for (int q = 0; q < 8; ++q) g[int64_t(rr_final_pos<L, false>(u, q)) * sv.sj + line] = v[0][q];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- X + Gamma
// tile = (column tile kt, k2 = j, row group rg); buffer [ch][pad8(row)][W]
template <int L>
static __global__ void __launch_bounds__(256, 1) xgamma_pp(SpecView sv, const double2* __restrict__ tw, int W,
                                                           GreenTables G, int64_t ntiles, int bufsz) {
  constexpr int N = 1 << L;
  extern __shared__ double2 sm[];
  const int ntk = int((sv.n3c + W - 1) / W);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  const int64_t plane = sv.cs;  // single slab only (pipelines are off when blocked)
  const int64_t rowstride = sv.si;
  const int chs = (N + N / 8) * W;
  auto base_of = [&](int64_t tile, int& w, int64_t& j, int& rg, int& kc0) {
    const int kt = int(tile % ntk);
    const int64_t rest = tile / ntk;
    j = rest % sv.n2;
    rg = int(rest / sv.n2);
    kc0 = kt * W;
    w = min(W, int(sv.n3c) - kc0);
    return sv.spec + int64_t(3 * rg) * plane + j * sv.sj + kc0;
  };
  auto prefetch = [&](double2* buf, int64_t tile) {
    int w, rg, kc0;
    int64_t j;
    const double2* g = base_of(tile, w, j, rg, kc0);
    for (int idx = threadIdx.x; idx < 3 * N * W; idx += blockDim.x) {
      const int col = idx % W, rest = idx / W, row = rest % N, ch = rest / N;
      if (col < w) cp_async16(buf + ch * chs + pad8(row) * W + col, g + int64_t(ch) * plane + row * rowstride + col);
    }
    cp_async_commit();
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prefetch(sm, tile);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double2* buf = sm + (it & 1) * bufsz;
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) {
      prefetch(sm + ((it + 1) & 1) * bufsz, next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    int w, rg, kc0;
    int64_t j;
    double2* g = base_of(tile, w, j, rg, kc0);
    const bool active = line < w && u < N / 8;
    double2 v[3][8];
    if (active) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
#pragma unroll
        for (int q = 0; q < 8; ++q) v[ch][q] = buf[ch * chs + pad8(rr_first_pos<L, false>(u, q)) * W + line];
    }
    __syncthreads();
    auto addr = [&](int ch, int pos) { return ch * chs + pad8(pos) * W + line; };
    rr_stages<L, false, false, 0, 3>(v, u, active, buf, tw, addr);
    if (active) {
      const int64_t k3 = kc0 + line;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t k1 = rr_final_pos<L, false>(u, q);
        double2 t[3] = {v[0][q], v[1][q], v[2][q]};
        gamma_row(G, rg, k1, j, k3, sv.n1, sv.n2, sv.n3, t);
        v[0][q] = t[0];
        v[1][q] = t[1];
        v[2][q] = t[2];
      }
    }
    rr_stages<L, true, true, 0, 3>(v, u, active, buf, tw, addr);
    if (active) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
#pragma unroll
        for (int q = 0; q < 8; ++q) g[int64_t(ch) * plane + rr_final_pos<L, true>(u, q) * rowstride + line] = v[ch][q];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ Z pass
// tile = nlb consecutive z-lines; 9 nlb real lines packed in pairs.
// Buffer: input region [rl][N + N/8] doubles, exchange region [pair][pad8(N)]
// complex (same memory, used after the stage-0 operands are in registers).
template <class Prod, int L>
static __global__ void __launch_bounds__(384, 2)
    zfwd_pp(SpecView sv, const double2* __restrict__ tw, int nlb, int64_t ntiles, int bufsz, Prod prod) {
  constexpr int N = 1 << L, TL = N / 8, LS = N + N / 8;
  constexpr int LSD = (LS + 1) & ~1;  // even double stride: 16-byte aligned rows
  extern __shared__ double2 sm[];
  const int64_t nlines_tot = sv.ni * sv.n2;  // local z-lines
  const int u = threadIdx.x % TL, p = threadIdx.x / TL;
  const int rla = 2 * p, rlb = 2 * p + 1;
  const int la = rla / 9, ca = rla - 9 * la, lb = rlb / 9, cb = rlb - 9 * lb;
  auto prefetch = [&](double2* buf, int64_t tile) {
    const int64_t line0 = tile * nlb;
    const int nl = int(min(int64_t(nlb), nlines_tot - line0));
    double* dbuf = reinterpret_cast<double*>(buf);
    const int chunks = N / 2;  // 16-byte chunks per real line
    for (int idx = threadIdx.x; idx < 9 * nl * chunks; idx += blockDim.x) {
      const int rl = idx / chunks, ck = idx - rl * chunks;
      const int li = rl / 9, c = rl - 9 * li;
      cp_async16(dbuf + rl * LSD + 2 * ck, prod.src + c * prod.N + (line0 + li) * N + 2 * ck);
    }
    cp_async_commit();
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prefetch(sm, tile);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double2* buf = sm + (it & 1) * bufsz;
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) {
      prefetch(sm + ((it + 1) & 1) * bufsz, next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t line0 = tile * nlb;
    const int nlines = int(min(int64_t(nlb), nlines_tot - line0));
    const int nreal = 9 * nlines;
    const int npair = (nreal + 1) >> 1;
    const bool active = p < npair;
    const bool hasb = rlb < nreal;
    const double* dbuf = reinterpret_cast<const double*>(buf);
    double2 v[1][8];
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = rr_first_pos<L, false>(u, i);
        v[0][i].x = dbuf[rla * LSD + e];
        v[0][i].y = hasb ? dbuf[rlb * LSD + e] : 0.0;
      }
    }
    __syncthreads();
    auto addr = [&](int, int pos) { return p * LS + pad8(pos); };
    rr_stages<L, false, false, 0, 1>(v, u, active, buf, tw, addr);
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i) buf[p * LS + pad8(rr_final_pos<L, false>(u, i))] = v[0][i];
    }
    __syncthreads();
    const int nc = int(sv.n3c);
    for (int t = threadIdx.x; t < npair * nc; t += blockDim.x) {
      const int pp = t / nc, k = t - pp * nc;
      const double2 zk = buf[pp * LS + pad8(k)];
      const double2 zm = buf[pp * LS + pad8(k == 0 ? 0 : N - k)];
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
    __syncthreads();
  }
  (void)la;
  (void)lb;
  (void)ca;
  (void)cb;
}

// Z inverse: input region [rl][n3p] complex (half spectra), Hermitian
// completion read straight into the stage-0 registers; consumer applied per
// component from the final registers; per-block reduction once at the end.
template <class Cons, int L>
static __global__ void __launch_bounds__(384, 2) zinv_pp(SpecView sv, const double2* __restrict__ tw, int nlb,
                                                         int64_t ntiles, int bufsz, double scale, Cons cons,
                                                         double* partials) {
  constexpr int N = 1 << L, TL = N / 8, LS = N + N / 8;
  extern __shared__ double2 sm[];
  const int64_t nlines_tot = sv.ni * sv.n2;  // local z-lines
  const int nc = int(sv.n3c);
  const int u = threadIdx.x % TL, p = threadIdx.x / TL;
  const int rla = 2 * p, rlb = 2 * p + 1;
  const int la = rla / 9, ca = rla - 9 * la, lb = rlb / 9, cb = rlb - 9 * lb;
  auto prefetch = [&](double2* buf, int64_t tile) {
    const int64_t line0 = tile * nlb;
    const int nl = int(min(int64_t(nlb), nlines_tot - line0));
    for (int idx = threadIdx.x; idx < 9 * nl * nc; idx += blockDim.x) {
      const int rl = idx / nc, k = idx - rl * nc;
      const int li = rl / 9, c = rl - 9 * li;
      cp_async16(buf + rl * int(sv.n3p) + k, sv.spec + sv.zrow(c, line0 + li) + k);
    }
    cp_async_commit();
  };
  double sc[Cons::NSC > 0 ? Cons::NSC : 1];
#pragma unroll
  for (int i = 0; i < (Cons::NSC > 0 ? Cons::NSC : 1); ++i) sc[i] = 0.0;
  double pa = 0.0, pb = 0.0;
  bool any_b = false;
  int64_t tile = blockIdx.x;
  if (tile < ntiles) prefetch(sm, tile);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    double2* buf = sm + (it & 1) * bufsz;
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) {
      prefetch(sm + ((it + 1) & 1) * bufsz, next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int64_t line0 = tile * nlb;
    const int nlines = int(min(int64_t(nlb), nlines_tot - line0));
    const int nreal = 9 * nlines;
    const int npair = (nreal + 1) >> 1;
    const bool active = p < npair;
    const bool hasb = rlb < nreal;
    double2 v[1][8];
    if (active) {
      const int n3p = int(sv.n3p);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = rr_first_pos<L, false>(u, i);
        const bool upper = 2 * e > N;
        const int k = upper ? N - e : e;
        double2 xa = buf[rla * n3p + k];
        double2 xb = hasb ? buf[rlb * n3p + k] : make_double2(0.0, 0.0);
        if (k == 0 || 2 * k == N) {  // halfcomplex c2r: DC/Nyquist imaginary parts ignored
          xa.y = 0.0;
          xb.y = 0.0;
        }
        v[0][i] = upper ? make_double2(xa.x + xb.y, xb.x - xa.y) : make_double2(xa.x - xb.y, xa.y + xb.x);
      }
    }
    __syncthreads();
    auto addr = [&](int, int pos) { return p * LS + pad8(pos); };
    rr_stages<L, true, false, 0, 1>(v, u, active, buf, tw, addr);
    if (active) {
      any_b = any_b || hasb;
      const int64_t cella = (line0 + la) * N, cellb = (line0 + lb) * N;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = rr_final_pos<L, false>(u, i);
        pa += cons.comp(ca, cella + e, v[0][i].x * scale, sc);
        if (hasb) pb += cons.comp(cb, cellb + e, v[0][i].y * scale, sc);
      }
    }
    __syncthreads();
  }
  if constexpr (Cons::NSC > 0 || Cons::PERCOMP) {
    group_reduce_store<Cons::NSC, Cons::PERCOMP>(sc, pa, pb, ca, any_b ? cb : -1, TL,
                                                 reinterpret_cast<double*>(sm), partials, blockIdx.x);
  }
}

}  // namespace combo_dev
