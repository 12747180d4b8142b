// Register-resident Stockham passes for power-of-two line lengths >= 8.
//
// Each thread owns one radix-8 butterfly position u of a line (8 complex
// values in registers; two radix-4 butterflies on radix-4 stages). The first
// stage reads its operands straight from global memory, intermediate stages
// exchange through a padded shared-memory tile (conflict-free 128-byte
// phases), and the last stage leaves the natural-order outputs
// X[u + r N/8] in registers, from where they are stored to global memory (or,
// in the X pass, projected by Gamma and fed directly to the inverse transform,
// whose radix order is reversed so its first stage consumes exactly those
// registers). Compared with the staged version this halves shared-memory
// traffic and keeps 8-24 independent 16-byte loads per thread in flight.
#pragma once

#include "fft.cuh"
#include "stage.cuh"

namespace combo_dev {

template <int L, bool REV>
struct Seq {
  static constexpr int N = 1 << L;
  static constexpr int NS = pow2_nstages(L);
  static constexpr int R(int s) { return pow2_radix(L, REV ? NS - 1 - s : s); }
  static constexpr int P(int s) {
    int p = 1;
    for (int i = 0; i < s; ++i) p *= R(i);
    return p;
  }
};

// Base twiddles of one stage: w^(k TS) per butterfly (k = t mod P); the
// R - 1 twiddles of a butterfly are its powers, formed in registers (depth-3
// product tree, <= 4 ulp) so a stage issues one 16-byte L1 load per
// butterfly instead of R - 1, and the load can be hoisted above the
// preceding exchange barrier.
template <int N, int R, int P>
__device__ __forceinline__ void rr_twload(double2 (&w)[8 / R], int u, const double2* __restrict__ tw) {
  constexpr int TS = N / (P * R);
#pragma unroll
  for (int q = 0; q < 8 / R; ++q) {
    if constexpr (P > 1) {
      const int k = (u + q * (N / 8)) & (P - 1);
      w[q] = __ldg(tw + k * TS);
    } else {
      w[q] = make_double2(1.0, 0.0);
    }
  }
}

// butterflies of one stage on the 8 register values of a channel
template <int N, int R, int P, bool INV>
__device__ __forceinline__ void rr_bfly(double2 (&v)[8], const double2 (&w)[8 / R]) {
  constexpr int B = 8 / R;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    if constexpr (P > 1) {
      double2 p[8];
      p[1] = w[q];
      if (INV) p[1].y = -p[1].y;
      if constexpr (R >= 4) {
        p[2] = cmul(p[1], p[1]);
        p[3] = cmul(p[2], p[1]);
      }
      if constexpr (R == 8) {
        p[4] = cmul(p[2], p[2]);
        p[5] = cmul(p[4], p[1]);
        p[6] = cmul(p[3], p[3]);
        p[7] = cmul(p[4], p[3]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[q * R + r] = cmul(v[q * R + r], p[r]);
    }
    dftR<R, INV>(&v[q * R]);
  }
}

// output position of register (q, r) after stage (N, R, P)
template <int N, int R, int P>
__device__ __forceinline__ int rr_out(int u, int q, int r) {
  const int t = u + q * (N / 8);
  const int k = t & (P - 1);
  return (t - k) * R + k + r * P;
}
// input position of register (q, r) for stage (N, R)
template <int N, int R>
__device__ __forceinline__ int rr_in(int u, int q, int r) {
  return u + q * (N / 8) + r * (N / R);
}

// barrier of the threads that exchange through sm: the whole block, or a
// named barrier over a warp-aligned group of it
struct BlockSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct GroupSync {
  int id, count;  // barrier 1..15, threads (a multiple of 32)
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
};

// Stages S.. of the transform on C channels held in v. addr(ch, pos) gives
// the shared-memory slot of channel ch at line position pos (per thread's
// line). All threads of the block (of the sync group) must call this
// (barriers inside).
template <int L, bool INV, bool REV, int S, int C, class Addr, class Sync = BlockSync>
__device__ __forceinline__ void rr_stages_w(double2 (&v)[C][8], int u, bool active, double2* sm,
                                            const double2* __restrict__ tw, const Addr& addr,
                                            const double2 (&w)[8 / Seq<L, REV>::R(S)], const Sync& sync = Sync()) {
  using Q = Seq<L, REV>;
  constexpr int N = Q::N, R = Q::R(S), P = Q::P(S);
  if (active) {
#pragma unroll
    for (int ch = 0; ch < C; ++ch) rr_bfly<N, R, P, INV>(v[ch], w);
  }
  if constexpr (S + 1 < Q::NS) {
    constexpr int R2 = Q::R(S + 1), P2 = Q::P(S + 1);
    double2 wn[8 / R2];
    rr_twload<N, R2, P2>(wn, u, tw);  // latency overlaps the exchange
    if (active) {
#pragma unroll
      for (int ch = 0; ch < C; ++ch)
#pragma unroll
        for (int q = 0; q < 8 / R; ++q)
#pragma unroll
          for (int r = 0; r < R; ++r) sm[addr(ch, rr_out<N, R, P>(u, q, r))] = v[ch][q * R + r];
    }
    sync();
    if (active) {
#pragma unroll
      for (int ch = 0; ch < C; ++ch)
#pragma unroll
        for (int q = 0; q < 8 / R2; ++q)
#pragma unroll
          for (int r = 0; r < R2; ++r) v[ch][q * R2 + r] = sm[addr(ch, rr_in<N, R2>(u, q, r))];
    }
    sync();
    rr_stages_w<L, INV, REV, S + 1, C>(v, u, active, sm, tw, addr, wn, sync);
  }
}

// Stages S.. of the transform on C channels held in v. addr(ch, pos) gives
// the shared-memory slot of channel ch at line position pos (per thread's
// line). All threads of the block must call this (barriers inside).
template <int L, bool INV, bool REV, int S, int C, class Addr, class Sync = BlockSync>
__device__ __forceinline__ void rr_stages(double2 (&v)[C][8], int u, bool active, double2* sm,
                                          const double2* __restrict__ tw, const Addr& addr,
                                          const Sync& sync = Sync()) {
  using Q = Seq<L, REV>;
  if constexpr (S < Q::NS) {
    double2 w[8 / Q::R(S)];
    rr_twload<Q::N, Q::R(S), Q::P(S)>(w, u, tw);
    rr_stages_w<L, INV, REV, S, C>(v, u, active, sm, tw, addr, w, sync);
  }
}

// natural-order output position of register i after the last stage
template <int L, bool REV>
__device__ __forceinline__ int rr_final_pos(int u, int i) {
  using Q = Seq<L, REV>;
  constexpr int R = Q::R(Q::NS - 1);
  return rr_in<Q::N, R>(u, i / R, i % R);  // last stage: P = N/R, k = t -> t + r N/R
}
// input position of register i for the first stage
template <int L, bool REV>
__device__ __forceinline__ int rr_first_pos(int u, int i) {
  using Q = Seq<L, REV>;
  constexpr int R = Q::R(0);
  return rr_in<Q::N, R>(u, i / R, i % R);
}

// padded element index (one spare slot per 8 elements)
__device__ __forceinline__ int pad8(int e) { return e + (e >> 3); }

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---------------------------------------------------------------- reductions
// Threads are grouped in power-of-two groups of G lanes sharing the same
// (component a, component b) pair; per group: NSC scalars, plus per-component
// sums of a and b when PERCOMP. Deterministic fixed-order combination into
// partials[block][NSC + (PERCOMP ? 9 : 0)].
template <int NSC, bool PERCOMP, class Sync = BlockSync>
__device__ void group_reduce_store(double (&sc)[NSC > 0 ? NSC : 1], double pa, double pb, int ca, int cb, int G,
                                   double* red_sm, double* partials, int64_t block, int tid = threadIdx.x,
                                   int nthreads = blockDim.x, const Sync& sync = Sync()) {
  constexpr int NV = NSC + (PERCOMP ? 2 : 0);
  if constexpr (NV > 0) {
    double v[NV > 0 ? NV : 1];
#pragma unroll
    for (int i = 0; i < NSC; ++i) v[i] = sc[i];
    if constexpr (PERCOMP) {
      v[NSC] = pa;
      v[NSC + 1] = pb;
    }
    const int lane = tid & 31;
    const int g = G < 32 ? G : 32;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      for (int o = g >> 1; o > 0; o >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], o, g);
    const int ngroups = (nthreads + g - 1) / g;
    const int grp = tid / g;
    // red_sm: [ngroups][NV + 2] (values, ca, cb)
    if ((lane & (g - 1)) == 0) {
#pragma unroll
      for (int i = 0; i < NV; ++i) red_sm[grp * (NV + 2) + i] = v[i];
      red_sm[grp * (NV + 2) + NV] = double(ca);
      red_sm[grp * (NV + 2) + NV + 1] = double(cb);
    }
    sync();
    constexpr int NOUT = NSC + (PERCOMP ? 9 : 0);
    if (tid < NOUT) {
      double s = 0.0;
      const int o = tid;
      for (int gi = 0; gi < ngroups; ++gi) {
        const double* e = red_sm + gi * (NV + 2);
        if (o < NSC) {
          s += e[o];
        } else if constexpr (PERCOMP) {
          const int c = o - NSC;
          if (int(e[NV]) == c) s += e[NSC];
          if (int(e[NV + 1]) == c) s += e[NSC + 1];
        }
      }
      partials[block * NOUT + o] = s;
    }
  }
}

// ------------------------------------------------------------------ Z pass
constexpr int kMaxZRows = 1024;  // 9 x lines per block (T <= 512 bounds it)
// Pairs of real lines (comp c of z-line l, enumerated rl = 9 l + c) are packed
// as one complex line; T = npair * N/8 threads, thread -> (pair, u).
// one tile: z-lines [line0, line0 + nlines) of the slab
template <class Prod, int L>
__device__ __forceinline__ void zfwd_tile(const SpecView& sv, const double2* __restrict__ tw, int64_t line0,
                                          int nlines, const Prod& prod) {
  constexpr int N = 1 << L, TL = N / 8, LS = N + N / 8;
  extern __shared__ double2 sm[];
  const int nreal = 9 * nlines;
  const int npair = (nreal + 1) >> 1;
  const int u = threadIdx.x % TL, p = threadIdx.x / TL;
  const bool active = p < npair;
  const int rla = 2 * p, rlb = 2 * p + 1;
  const int la = rla / 9, ca = rla - 9 * la, lb = rlb / 9, cb = rlb - 9 * lb;
  const bool hasb = rlb < nreal;
  double2 v[1][8];
  if (active) {
    const int64_t cella = (line0 + la) * N, cellb = (line0 + lb) * N;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = rr_first_pos<L, false>(u, i);
      v[0][i].x = prod.comp(ca, cella + e);
      v[0][i].y = hasb ? prod.comp(cb, cellb + e) : 0.0;
    }
  }
  // spectrum row offsets of the block's real lines (read after the barriers
  // inside rr_stages)
  __shared__ int64_t zr[kMaxZRows];
  for (int t = threadIdx.x; t < nreal; t += blockDim.x) zr[t] = sv.zrow(t % 9, line0 + t / 9);
  auto addr = [&](int, int pos) { return p * LS + pad8(pos); };
  rr_stages<L, false, false, 0, 1>(v, u, active, sm, tw, addr);
  // natural order to smem, then split the pair into two half spectra
  if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i) sm[p * LS + pad8(rr_final_pos<L, false>(u, i))] = v[0][i];
  }
  __syncthreads();
  const int nc = int(sv.n3c);
  // warp-aligned k ranges per pair: the 8-lane phases of the 16-byte shared
  // loads then never straddle a pad slot (bank conflicts otherwise)
  const int ncr = (nc + 31) & ~31;
  for (int t = threadIdx.x; t < npair * ncr; t += blockDim.x) {
    const int pp = t / ncr, k = t - pp * ncr;
    if (k >= nc) continue;
    const double2 zk = sm[pp * LS + pad8(k)];
    const double2 zm = sm[pp * LS + pad8(k == 0 ? 0 : N - k)];
    const int rl = 2 * pp;
    sv.spec[zr[rl] + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    if (rl + 1 < nreal) sv.spec[zr[rl + 1] + k] = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
  }
}

template <class Prod, int L>
static __global__ void __launch_bounds__(512, 2)
    zfwd_rr(SpecView sv, const double2* __restrict__ tw, int nl_per_block, Prod prod, double*) {
  const int64_t nlines_tot = sv.ni * sv.n2;  // local z-lines
  const int64_t line0 = int64_t(blockIdx.x) * nl_per_block;
  zfwd_tile<Prod, L>(sv, tw, line0, int(min(int64_t(nl_per_block), nlines_tot - line0)), prod);
}

// Second half of a z-inverse tile: the completed natural-order pair lines
// are in sm; inverse stages, then the consumer on the real outputs.
template <class Cons, int L, class Sync = BlockSync>
__device__ __forceinline__ void zinv_finish(double2* sm, const double2* __restrict__ tw, int64_t line0, int nreal,
                                            int npair, double scale, const Cons& cons, double* partials,
                                            int64_t slot, int tid = threadIdx.x, int nthreads = blockDim.x,
                                            const Sync& sync = Sync()) {
  constexpr int N = 1 << L, TL = N / 8, LS = N + N / 8;
  const int u = tid % TL, p = tid / TL;
  const bool active = p < npair;
  const int rla = 2 * p, rlb = 2 * p + 1;
  const int la = rla / 9, ca = rla - 9 * la, lb = rlb / 9, cb = rlb - 9 * lb;
  const bool hasb = rlb < nreal;
  const int64_t cella = (line0 + la) * N, cellb = (line0 + lb) * N;
  double2 v[1][8];
  if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[0][i] = sm[p * LS + pad8(rr_first_pos<L, false>(u, i))];
  }
  // PRELOAD consumers: the field values the epilogue combines with the
  // outputs are requested now, so their latency hides behind the stages
  // (registers or, under pressure, L1-resident local memory)
  [[maybe_unused]] double pre[2][8];
  if constexpr (Cons::PRELOAD) {
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = rr_final_pos<L, false>(u, i);
        pre[0][i] = cons.load(ca, cella + e);
        pre[1][i] = hasb ? cons.load(cb, cellb + e) : 0.0;
      }
    }
  }
  sync();
  auto addr = [&](int, int pos) { return p * LS + pad8(pos); };
  rr_stages<L, true, false, 0, 1>(v, u, active, sm, tw, addr, sync);
  double sc[Cons::NSC > 0 ? Cons::NSC : 1];
#pragma unroll
  for (int i = 0; i < (Cons::NSC > 0 ? Cons::NSC : 1); ++i) sc[i] = 0.0;
  double pa = 0.0, pb = 0.0;
  if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = rr_final_pos<L, false>(u, i);
      if constexpr (Cons::PRELOAD) {
        pa += cons.comp_pre(ca, cella + e, v[0][i].x * scale, pre[0][i], sc);
        if (hasb) pb += cons.comp_pre(cb, cellb + e, v[0][i].y * scale, pre[1][i], sc);
      } else {
        pa += cons.comp(ca, cella + e, v[0][i].x * scale, sc);
        if (hasb) pb += cons.comp(cb, cellb + e, v[0][i].y * scale, sc);
      }
    }
  }
  if constexpr (Cons::NSC > 0 || Cons::PERCOMP) {
    sync();  // sm reused for the group reduction
    group_reduce_store<Cons::NSC, Cons::PERCOMP>(sc, pa, pb, ca, active && hasb ? cb : -1, TL,
                                                 reinterpret_cast<double*>(sm), partials, slot, tid, nthreads, sync);
  }
}

// one tile: z-lines [line0, line0 + nlines); partial sums -> partials[slot].
// CG: spectrum loads bypass L1 (the fused Y/Z kernel reads rows other SMs
// just wrote); DISCARD: the consumed spectrum rows are dropped from L2
// without write-back (dead after this pass).
template <class Cons, int L, bool CG = false, bool DISCARD = false>
__device__ __forceinline__ void zinv_tile(const SpecView& sv, const double2* __restrict__ tw, int64_t line0,
                                          int nlines, double scale, const Cons& cons, double* partials,
                                          int64_t slot, bool discard = true) {
  constexpr int N = 1 << L, LS = N + N / 8;
  extern __shared__ double2 sm[];
  const int nreal = 9 * nlines;
  const int npair = (nreal + 1) >> 1;
  const int nc = int(sv.n3c);
  const int ncr = (nc + 31) & ~31;  // warp-aligned k ranges (see zfwd_rr)
  // the consumer's field rows of this block (read after the transform) go
  // to L2 now, so the epilogue loads hit L2 instead of HBM latency
  if (threadIdx.x < 9) cons.prefetch(int(threadIdx.x), line0 * N, int64_t(nlines) * N);
  __shared__ int64_t zr[kMaxZRows];
  for (int t = threadIdx.x; t < nreal; t += blockDim.x) zr[t] = sv.zrow(t % 9, line0 + t / 9);
  __syncthreads();
  // Hermitian completion of the pair (halfcomplex c2r: DC/Nyquist imaginary
  // parts ignored) into natural-order smem lines
  // kZU rows of the loop are loaded before any is completed: 2 kZU
  // independent 16-byte loads in flight per thread (one pair at a time left
  // the pass latency-bound)
  constexpr int kZU = 4;
  const int total = npair * ncr;
  for (int t0 = 0; t0 < total; t0 += kZU * int(blockDim.x)) {
    double2 xa[kZU], xb[kZU];
#pragma unroll
    for (int r = 0; r < kZU; ++r) {
      const int t = t0 + r * int(blockDim.x) + int(threadIdx.x);
      const int pp = t / ncr, k = t - pp * ncr;
      const int rl = 2 * pp;
      xa[r] = xb[r] = make_double2(0.0, 0.0);
      if (t < total && k < nc) {
        if (CG) {
          xa[r] = __ldcg(sv.spec + zr[rl] + k);
          if (rl + 1 < nreal) xb[r] = __ldcg(sv.spec + zr[rl + 1] + k);
        } else {
          xa[r] = sv.spec[zr[rl] + k];
          if (rl + 1 < nreal) xb[r] = sv.spec[zr[rl + 1] + k];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kZU; ++r) {
      const int t = t0 + r * int(blockDim.x) + int(threadIdx.x);
      const int pp = t / ncr, k = t - pp * ncr;
      if (t >= total || k >= nc) continue;
      const bool selfconj = (k == 0) || (2 * k == N);
      if (selfconj) {
        xa[r].y = 0.0;
        xb[r].y = 0.0;
      }
      sm[pp * LS + pad8(k)] = make_double2(xa[r].x - xb[r].y, xa[r].y + xb[r].x);
      if (!selfconj) sm[pp * LS + pad8(N - k)] = make_double2(xa[r].x + xb[r].y, xb[r].x - xa[r].y);
    }
  }
  __syncthreads();
  if (DISCARD && discard) {
    // every row of the tile has been read by the whole block (barrier above)
    const int lpr = int((nc * 16 + 127) / 128);  // 128-byte lines per row (rows are 128-byte aligned)
    for (int t = threadIdx.x; t < nreal * lpr; t += blockDim.x) {
      const int rl = t / lpr, q = t - rl * lpr;
      const char* a = reinterpret_cast<const char*>(sv.spec + zr[rl]) + 128 * q;
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
    }
  }
  zinv_finish<Cons, L>(sm, tw, line0, nreal, npair, scale, cons, partials, slot);
}

template <class Cons, int L>
static __global__ void __launch_bounds__(512, 2)
    zinv_rr(SpecView sv, const double2* __restrict__ tw, int nl_per_block, double scale, Cons cons,
            double* partials) {
  const int64_t nlines_tot = sv.ni * sv.n2;  // local z-lines
  const int64_t line0 = int64_t(blockIdx.x) * nl_per_block;
  zinv_tile<Cons, L>(sv, tw, line0, int(min(int64_t(nl_per_block), nlines_tot - line0)), scale, cons, partials,
                     blockIdx.x);
}

// Persistent ring-staged z-inverse for z-lines of 512 cells (one line per
// tile): one block per SM, two consumer groups of 5 N/8 threads and no
// producer warp (20 warps: 96 registers per thread, so a PRELOAD consumer
// keeps its prefetched field values in registers). The 9 spectrum rows of a
// tile reach a ring of kStages shared-memory stages by cp.async.bulk on the
// stage's mbarrier; the group that has consumed a stage (Hermitian completion
// into its own pair lines) re-arms it at once with the tile kStages ahead and
// L2-prefetches that tile's consumer rows. The groups take alternate tiles,
// so completion / inverse stages / epilogue of one tile overlap the other
// group's and the loads in flight. armed[s] (the tile last armed on stage s)
// keeps a group from polling a stage's barrier before its previous use was
// re-armed -- an mbarrier only distinguishes two consecutive phases.
// Partials are indexed by tile: same values and order as zinv_rr.
template <int L>
struct ZRing {
  static constexpr int N = 1 << L, LS = N + N / 8, NP = 5, GT = NP * (N / 8);  // threads per consumer group
  static constexpr int kStages = 3;
  static constexpr int kHead = 128;           // full[kStages] barriers, armed[kStages]
  static constexpr int kWork = NP * LS * 16;  // pair lines of one group
  static constexpr int kThreads = 2 * GT;
};

template <class Cons, int L>
static __global__ void __launch_bounds__(ZRing<L>::kThreads, 1)
    zinv_ring(SpecView sv, const double2* __restrict__ tw, double scale, Cons cons, double* partials) {
  using Z = ZRing<L>;
  constexpr int N = Z::N, LS = Z::LS, NP = Z::NP, GT = Z::GT, S = Z::kStages;
  extern __shared__ __align__(128) unsigned char zr_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(zr_raw);
  volatile long long* armed = reinterpret_cast<volatile long long*>(zr_raw + 64);
  const int n3p = int(sv.n3p), nc = int(sv.n3c);
  const int ncr = (nc + 31) & ~31;  // warp-aligned k ranges (see zfwd_rr)
  const uint32_t stage_bytes = uint32_t(9 * n3p) * 16u;
  const uint32_t rb = uint32_t(nc) * 16u;
  unsigned char* stages = zr_raw + Z::kHead + 2 * Z::kWork;
  const int64_t ntiles = sv.ni * sv.n2;  // local z-lines
  const int64_t stride = gridDim.x;
  // k-th tile of this block: blockIdx.x + k stride, on stage k % S, group k % 2
  auto arm = [&](int64_t k) {  // one thread: loads of the block's k-th tile
    const int64_t tile = blockIdx.x + k * stride;
    const int s = int(k % S);
    double2* rows = reinterpret_cast<double2*>(stages + size_t(s) * stage_bytes);
    mbar_expect_tx(&full[s], 9u * rb);
#pragma unroll 1
    for (int rl = 0; rl < 9; ++rl) bulk_g2s(rows + rl * n3p, sv.spec + sv.zrow(rl, tile), rb, &full[s]);
    __threadfence_block();
    armed[s] = k;
#pragma unroll 1
    for (int c = 0; c < 9; ++c) cons.prefetch(c, tile * N, N);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      armed[s] = -1;
    }
    mbar_fence_init();
    for (int64_t k = 0; k < S && blockIdx.x + k * stride < ntiles; ++k) arm(k);
  }
  __syncthreads();
  const int g = int(threadIdx.x) / GT, tid = int(threadIdx.x) - g * GT;
  const GroupSync gsync{1 + g, GT};
  double2* work = reinterpret_cast<double2*>(zr_raw + Z::kHead + g * Z::kWork);
  for (int64_t k = g; blockIdx.x + k * stride < ntiles; k += 2) {
    const int64_t tile = blockIdx.x + k * stride;
    const int s = int(k % S);
    gsync();  // the previous tile's reduction has left the pair lines
    while (armed[s] != k) {
    }
    mbar_wait(&full[s], uint32_t((k / S) & 1));
    const double2* rows = reinterpret_cast<const double2*>(stages + size_t(s) * stage_bytes);
    // Hermitian completion of the pairs (see zinv_tile) from the staged rows
    for (int t = tid; t < NP * ncr; t += GT) {
      const int pp = t / ncr, kk = t - pp * ncr;
      if (kk >= nc) continue;
      const int rl = 2 * pp;
      double2 xa = rows[rl * n3p + kk];
      double2 xb = rl + 1 < 9 ? rows[(rl + 1) * n3p + kk] : make_double2(0.0, 0.0);
      const bool selfconj = (kk == 0) || (2 * kk == N);
      if (selfconj) {
        xa.y = 0.0;
        xb.y = 0.0;
      }
      work[pp * LS + pad8(kk)] = make_double2(xa.x - xb.y, xa.y + xb.x);
      if (!selfconj) work[pp * LS + pad8(N - kk)] = make_double2(xa.x + xb.y, xb.x - xa.y);
    }
    gsync();  // stage consumed, pair lines complete
    if (tid == 0 && blockIdx.x + (k + S) * stride < ntiles) arm(k + S);
    zinv_finish<Cons, L>(work, tw, tile, 9, NP, scale, cons, partials, tile, tid, GT, gsync);
  }
}

// ------------------------------------------------------------------ Y pass
// W columns (lines) per block, thread -> (line = tid % W, u = tid / W)
// one tile: columns [kc0, kc0 + W) of component c, local plane i
template <int L, bool INV, bool CG = false>
__device__ __forceinline__ void ypass_tile(const SpecView& sv, const double2* __restrict__ tw, int W, int c,
                                           int64_t i, int kc0) {
  constexpr int N = 1 << L;
  extern __shared__ double2 sm[];
  const int w = min(W, int(sv.n3c) - kc0);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  const bool active = line < w && u < N / 8;
  double2* base = sv.spec + int64_t(c) * sv.cs + kc0 + line;
  double2 v[1][8];
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t o = sv.rowA(i, rr_first_pos<L, false>(u, q));
      v[0][q] = CG ? __ldcg(base + o) : base[o];
    }
  }
  auto addr = [&](int, int pos) { return pad8(pos) * W + line; };
  rr_stages<L, INV, false, 0, 1>(v, u, active, sm, tw, addr);
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) base[sv.rowA(i, rr_final_pos<L, false>(u, q))] = v[0][q];
  }
}

template <int L, bool INV, int MAXT = 512, int MINB = 2>
static __global__ void __launch_bounds__(MAXT, MINB)
    ypass_rr(SpecView sv, const double2* __restrict__ tw, int W) {
  ypass_tile<L, INV>(sv, tw, W, blockIdx.z, blockIdx.y, blockIdx.x * W);
}

// ---------------------------------------------------------------- X + Gamma
// ------------------------------------------------ X + Gamma, rank-1 variant
// Gamma^0 row rg at k is rank one: tau_J <- gr_J s / den with
// s = sum_L conj(gr_L) tau_L (green.cpp:67-130). In all three schemes the
// column symbols gr_1, gr_2 factor as (per-k1 scalar a) x (per-(k2, k3)
// constant), so along an x line
//   s(k1)  = conj(gr_0(k1)) T_0(k1) + conj(a(k1)) FFT_x(e_1 t_1 + e_2 t_2)
//   out_J  = o_J IFFT_x(a s / den)   for J = 1, 2
// with e_J = conj(o_J) constant on the line. The pass therefore transforms
// two channels forward and two back instead of three: 1/3 less FP64 work,
// 16 instead of 24 complex registers and two shared-memory channel regions
// (three blocks per SM). Equal to gamma_row up to floating-point
// reassociation (linearity of the DFT).
__device__ __forceinline__ double drcp(double d) {
  // MUFU seed + three Newton steps (no slow-path call in the hot loop)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

template <int KIND>
struct RankCol {
  double2 o1, o2;  // output column factors (row's gr_1, gr_2 without a(k1))
  double2 c0;      // rotated: a2 a3
  double d12;      // |o1|^2 + |o2|^2
  bool zero;       // continuous: the column lies on a Nyquist plane
};

template <int KIND>
__device__ __forceinline__ RankCol<KIND> rank_col(const GreenTables& G, int row, int64_t k2, int64_t k3, int64_t n2,
                                                  int64_t n3) {
  RankCol<KIND> c;
  c.c0 = make_double2(0.0, 0.0);
  c.zero = false;
  if constexpr (KIND == 0) {
    c.o1 = make_double2(G.xi[1][k2], 0.0);
    c.o2 = make_double2(G.xi[2][k3], 0.0);
    c.zero = 2 * k2 == n2 || 2 * k3 == n3;
  } else if constexpr (KIND == 1) {
    const double2 a2 = __ldg(G.avg[1] + k2), a3 = __ldg(G.avg[2] + k3);
    c.c0 = cmul(a2, a3);
    c.o1 = cmul(__ldg(G.fwd[1] + k2), a3);
    c.o2 = cmul(__ldg(G.fwd[2] + k3), a2);
  } else {
    const double2 f1 = __ldg(G.fwd[1] + k2), f2 = __ldg(G.fwd[2] + k3);
    c.o1 = row == 1 ? f1 : make_double2(-f1.x, f1.y);
    c.o2 = row == 2 ? f2 : make_double2(-f2.x, f2.y);
  }
  c.d12 = (c.o1.x * c.o1.x + c.o1.y * c.o1.y) + (c.o2.x * c.o2.x + c.o2.y * c.o2.y);
  return c;
}

// (T0, U) at k1 -> (out_0, H) with out_1,2 = o_1,2 H
template <int KIND>
__device__ __forceinline__ void rank_gamma(const GreenTables& G, const RankCol<KIND>& c, int row, int64_t k1,
                                           int64_t n1, double2& t0, double2& u) {
  double2 g0, a;
  if constexpr (KIND == 0) {
    if (c.zero || 2 * k1 == n1) {
      t0 = u = make_double2(0.0, 0.0);
      return;
    }
    g0 = make_double2(__ldg(G.xi[0] + k1), 0.0);  // real form of g = i xi
    a = make_double2(1.0, 0.0);
  } else if constexpr (KIND == 1) {
    g0 = cmul(__ldg(G.fwd[0] + k1), c.c0);
    a = __ldg(G.avg[0] + k1);
  } else {
    const double2 f0 = __ldg(G.fwd[0] + k1);
    g0 = row == 0 ? f0 : make_double2(-f0.x, f0.y);
    a = make_double2(1.0, 0.0);
  }
  const double aa = a.x * a.x + a.y * a.y;
  const double den = (g0.x * g0.x + g0.y * g0.y) + aa * c.d12;
  if (den == 0.0) {
    t0 = u = make_double2(0.0, 0.0);
    return;
  }
  const double2 s0 = cmulc(g0, t0), s1 = cmulc(a, u);
  const double r = drcp(den);
  const double2 h = make_double2((s0.x + s1.x) * r, (s0.y + s1.y) * r);
  t0 = cmul(g0, h);
  u = cmul(a, h);
}

template <int L, int KIND, int MAXT, int MINB>
static __global__ void __launch_bounds__(MAXT, MINB)
    xgamma_v4(SpecView sv, const double2* __restrict__ tw, int W, GreenTables G, int rg0) {
  constexpr int N = 1 << L;
  extern __shared__ double2 sm[];
  const int rg = rg0 + blockIdx.z, j = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  const bool active = line < w && u < N / 8;
  const int64_t plane = sv.cs;
  double2* base = sv.spec + int64_t(3 * rg) * plane + kc0 + line;  // pencil side, local k2 j
  const RankCol<KIND> col = rank_col<KIND>(G, rg, sv.j0 + j, kc0 + line, sv.n2, sv.n3);
  double2 v[2][8];
  if (active) {
    double2 t1[8], t2[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t o = sv.rowB(rr_first_pos<L, false>(u, q), j);
      v[0][q] = base[o];
      t1[q] = base[plane + o];
      t2[q] = base[2 * plane + o];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 a = cmulc(col.o1, t1[q]), b = cmulc(col.o2, t2[q]);
      v[1][q] = make_double2(a.x + b.x, a.y + b.y);
    }
  }
  const int chs = (N + N / 8) * W;
  auto addr = [&](int ch, int pos) { return ch * chs + pad8(pos) * W + line; };
  rr_stages<L, false, false, 0, 2>(v, u, active, sm, tw, addr);
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) rank_gamma<KIND>(G, col, rg, rr_final_pos<L, false>(u, q), sv.n1, v[0][q], v[1][q]);
  }
  rr_stages<L, true, true, 0, 2>(v, u, active, sm, tw, addr);
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t o = sv.rowB(rr_final_pos<L, true>(u, q), j);
      base[o] = v[0][q];
      base[plane + o] = cmul(col.o1, v[1][q]);
      base[2 * plane + o] = cmul(col.o2, v[1][q]);
    }
  }
}

// plain X pass (raw FFT test entry point)
template <int L, bool INV>
static __global__ void __launch_bounds__(512, 2) xpass_rr(SpecView sv, const double2* __restrict__ tw, int W) {
  constexpr int N = 1 << L;
  extern __shared__ double2 sm[];
  const int c = blockIdx.z, j = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  const bool active = line < w && u < N / 8;
  double2* base = sv.spec + int64_t(c) * sv.cs + kc0 + line;
  double2 v[1][8];
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) v[0][q] = base[sv.rowB(rr_first_pos<L, false>(u, q), j)];
  }
  auto addr = [&](int, int pos) { return pad8(pos) * W + line; };
  rr_stages<L, INV, false, 0, 1>(v, u, active, sm, tw, addr);
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) base[sv.rowB(rr_final_pos<L, false>(u, q), j)] = v[0][q];
  }
}

}  // namespace combo_dev
