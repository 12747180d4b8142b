// Pointwise kernels of the LS iteration and the FFT producer/consumer
// functors that fuse the solver updates into the first / last FFT pass.
//
// Reference loops replaced (file:line in /root/reference/proj/src):
//   stress_sweep            cell_material.cpp:104-168   -> k_sweep
//   tangent_matvec + p-upd. cell_material.cpp:170-194,
//                           solver.cpp:194-197          -> k_matvec (matrix free)
//   F update + residual     solver.cpp:135-149          -> ConsBasic (Z-inverse)
//   b = -Pi(P), rms         solver.cpp:209-225          -> ConsResid
//   pap = dot(pdir, Pi(q))  solver.cpp:180-181          -> ConsCg
//   x += s p, r -= s ap, rr solver.cpp:186-190          -> k_cg_update
//   ftrial = F + s x, mean  solver.cpp:241-243          -> k_trial
//   Field9::mean / pin_mean field.cpp:18-38             -> k_sum9 / lazy shift
#pragma once

#include "fft.cuh"
#include "fft_rr.cuh"
#include "material.cuh"
#include "stage.cuh"

namespace combo_dev {

constexpr int kEwThreads = 256;

// cid encoding: -1 pure matrix, -2 pure inclusion, >= 0 composite id
struct CellData {
  const int32_t* cid;
  const double* nrm;  // [3][ncomp]
  const double* cp;   // [ncomp]
  const double* cm;   // [ncomp]
  double* warm;       // [3][ncomp]
  int64_t ncomp;
  const int64_t* ccell;  // cell index per composite id
  const double* t45;     // [45][ncomp] packed composite tangents (or null)
};

struct Stats {  // device counters (SweepStats)
  unsigned long long inadmissible, failures, backproj, iter_max;
};

__device__ __forceinline__ void warp_stats(Stats* st, unsigned long long inad, unsigned long long fail,
                                           unsigned long long bp, unsigned int itmax) {
  const unsigned mask = __activemask();
  const unsigned a = __reduce_add_sync(mask, unsigned(inad));
  const unsigned f = __reduce_add_sync(mask, unsigned(fail));
  const unsigned b = __reduce_add_sync(mask, unsigned(bp));
  const unsigned m = __reduce_max_sync(mask, itmax);
  if ((threadIdx.x & 31) == __ffs(mask) - 1) {
    if (a) atomicAdd(&st->inadmissible, (unsigned long long)a);
    if (f) atomicAdd(&st->failures, (unsigned long long)f);
    if (b) atomicAdd(&st->backproj, (unsigned long long)b);
    if (m) atomicMax(&st->iter_max, (unsigned long long)m);
  }
}

// P(F) for one cell; returns false when inadmissible. Writes back the warm
// start of composite cells when `writeback`.
__device__ __forceinline__ bool cell_stress(const MatParams& M, const CellData& cd, int64_t cell,
                                            const double* f, double* p, bool writeback, unsigned long long& fail,
                                            unsigned long long& bp, unsigned int& itmax) {
  const int32_t id = cd.cid[cell];
  if (id >= 0) {
    const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
    const double a0[3] = {cd.warm[id], cd.warm[cd.ncomp + id], cd.warm[2 * cd.ncomp + id]};
    LamResult R;
    laminate_solve(M, f, n, cd.cp[id], cd.cm[id], a0, R);
    if (R.inadmissible) {
#pragma unroll
      for (int c = 0; c < 9; ++c) p[c] = 0.0;
      return false;
    }
    if (!R.converged) ++fail;
    bp += (unsigned long long)R.back_projections;
    itmax = max(itmax, (unsigned)R.iterations);
    if (writeback) {
      cd.warm[id] = R.a[0];
      cd.warm[cd.ncomp + id] = R.a[1];
      cd.warm[2 * cd.ncomp + id] = R.a[2];
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) p[c] = R.p[c];
    return true;
  }
  NhState s;
  const LawP L = id == -2 ? M.law[1] : M.law[0];
  if (!law_eval(L, f, p, s)) {
#pragma unroll
    for (int c = 0; c < 9; ++c) p[c] = 0.0;
    return false;
  }
  return true;
}

struct Shift9 {
  double v[9];
};

// Deterministic, decomposition-invariant reductions: block b of a chunked
// launch owns cells [p plane + k C, min(p plane + (k + 1) C, (p + 1) plane))
// of local plane p = b / cpp (k = b mod cpp, C = kChunk). Chunks never
// straddle a plane, so a slab of whole planes owns a contiguous range of the
// global chunk list and the fixed-order combination of all chunk partials is
// the same for any number of slabs (reference: deterministic chunk-4096
// reductions, parallel.hpp:40-104).
constexpr int kChunk = 2048;
struct Chunks {
  int64_t plane;  // cells per plane (n2 n3)
  int cpp;        // chunks per plane
};
__device__ __forceinline__ void chunk_range(const Chunks& k, int64_t& beg, int64_t& end) {
  const int64_t p = blockIdx.x / k.cpp;
  const int64_t j = blockIdx.x - p * k.cpp;
  beg = p * k.plane + j * kChunk;
  end = min(beg + kChunk, (p + 1) * k.plane);
}

// out = P(F_in + shift) - alpha (F_in + shift); partial sums of P (P-bar).
static __global__ void __launch_bounds__(kEwThreads) k_sweep(MatParams M, CellData cd, const double* __restrict__ fin,
                                                      Shift9 sh, double alpha, double* __restrict__ out,
                                                      int64_t N, Chunks ch, int writeback, Stats* st,
                                                      double* partials) {
  double acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0;
  unsigned long long inad = 0, fail = 0, bp = 0;
  unsigned int itmax = 0;
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
    double f[9], p[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell] + sh.v[c];
    if (!cell_stress(M, cd, cell, f, p, writeback != 0, fail, bp, itmax)) ++inad;
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      acc[c] += p[c];
      out[c * N + cell] = alpha != 0.0 ? p[c] + (-alpha) * f[c] : p[c];
    }
  }
  warp_stats(st, inad, fail, bp, itmax);
  block_reduce_store<9>(acc, partials, blockIdx.x);
}

// Split sweep, pass 1: the laminate Newton of every composite cell
// (finite_strain_solve, cell_material.cpp:139-145), one composite per
// thread over the compact composite list, so the per-cell Newton no longer
// serialises the pure cells of mixed warps. Writes the raw P of each
// composite cell (0 when inadmissible) into out; pass 2 folds it in.
// 3 blocks of 128 threads per SM (168 registers): 41.1 ms per sweep at 512^3
// against 49.8 ms at 2 blocks (255 registers) and 40.0 ms at 4 (128)
static __global__ void __launch_bounds__(128, 3)
    k_sweep_comp(MatParams M, CellData cd, const double* __restrict__ fin, Shift9 sh, double* __restrict__ out,
                 int64_t N, int writeback, Stats* st) {
  unsigned long long inad = 0, fail = 0, bp = 0;
  unsigned int itmax = 0;
  for (int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; id < cd.ncomp;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cell = cd.ccell[id];
    double f[9], p[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell] + sh.v[c];
    if (!cell_stress(M, cd, cell, f, p, writeback != 0, fail, bp, itmax)) ++inad;
#pragma unroll
    for (int c = 0; c < 9; ++c) out[c * N + cell] = p[c];
  }
  warp_stats(st, inad, fail, bp, itmax);
}

// Split sweep, pass 2: NH stress of the pure cells, composite P read back
// from pass 1; out = P - alpha F; chunk partial sums of P in the same order
// as k_sweep (bitwise the same results).
static __global__ void __launch_bounds__(kEwThreads) k_sweep_pure(MatParams M, CellData cd,
                                                                  const double* __restrict__ fin, Shift9 sh,
                                                                  double alpha, double* __restrict__ out, int64_t N,
                                                                  Chunks ch, Stats* st, double* partials) {
  double acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0;
  unsigned long long inad = 0;
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
    const int32_t id = cd.cid[cell];
    double f[9], p[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell] + sh.v[c];
    if (id >= 0) {
#pragma unroll
      for (int c = 0; c < 9; ++c) p[c] = out[c * N + cell];
    } else {
      NhState s;
      if (!law_eval(id == -2 ? M.law[1] : M.law[0], f, p, s)) {
#pragma unroll
        for (int c = 0; c < 9; ++c) p[c] = 0.0;
        ++inad;
      }
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      acc[c] += p[c];
      out[c * N + cell] = alpha != 0.0 ? p[c] + (-alpha) * f[c] : p[c];
    }
  }
  warp_stats(st, inad, 0, 0, 0);
  block_reduce_store<9>(acc, partials, blockIdx.x);
}

// recover_phase_fields (postprocess.cpp:13-38): every composite re-solves
// its laminate at F from the stored warm start (not written back); the
// phase stresses P+ / P- of the returned state go to pp / pm [9][ncomp].
// per-composite recovered laminate state for interface tractions
// (recover_phase_fields, postprocess.cpp:13-36; LaminateResult traction,
// laminate.cpp:258-266): F+, F- and T = P+ n (converged) or the mean of the
// two phase tractions (best iterate), by composite id
static __global__ void __launch_bounds__(128) k_recover_state(MatParams M, CellData cd, const double* __restrict__ fin,
                                                              int64_t N, int64_t* __restrict__ cell_out,
                                                              double* __restrict__ fpo, double* __restrict__ fmo,
                                                              double* __restrict__ tro, Stats* st) {
  unsigned long long inad = 0;
  unsigned int itmax = 0;
  for (int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; id < cd.ncomp;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cell = cd.ccell[id];
    double f[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell];
    const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
    const double a0[3] = {cd.warm[id], cd.warm[cd.ncomp + id], cd.warm[2 * cd.ncomp + id]};
    LamResult R;
    laminate_solve(M, f, n, cd.cp[id], cd.cm[id], a0, R);
    double fp[9], fm[9], p1[9], p2[9], t[3];
    if (R.inadmissible) {
      ++inad;
#pragma unroll
      for (int c = 0; c < 9; ++c) fp[c] = fm[c] = 0.0;
      t[0] = t[1] = t[2] = 0.0;
    } else {
      itmax = max(itmax, (unsigned)R.iterations);
      form_phases(f, n, cd.cp[id], cd.cm[id], R.a, fp, fm);
      NhState s1, s2;
      if (!law_eval(M.law[1], fp, p1, s1))
#pragma unroll
        for (int c = 0; c < 9; ++c) p1[c] = 0.0;
      if (!law_eval(M.law[0], fm, p2, s2))
#pragma unroll
        for (int c = 0; c < 9; ++c) p2[c] = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double tp = p1[3 * i] * n[0] + p1[3 * i + 1] * n[1] + p1[3 * i + 2] * n[2];
        const double tm = p2[3 * i] * n[0] + p2[3 * i + 1] * n[1] + p2[3 * i + 2] * n[2];
        t[i] = R.converged ? tp : 0.5 * (tp + tm);
      }
    }
    cell_out[id] = cell;
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      fpo[c * cd.ncomp + id] = fp[c];
      fmo[c * cd.ncomp + id] = fm[c];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) tro[i * cd.ncomp + id] = t[i];
  }
  warp_stats(st, inad, 0, 0, itmax);
}

static __global__ void __launch_bounds__(128) k_recover(MatParams M, CellData cd, const double* __restrict__ fin,
                                                        int64_t N, double* __restrict__ pp, double* __restrict__ pm,
                                                        Stats* st) {
  unsigned long long inad = 0;
  unsigned int itmax = 0;
  for (int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; id < cd.ncomp;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cell = cd.ccell[id];
    double f[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell];
    const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
    const double a0[3] = {cd.warm[id], cd.warm[cd.ncomp + id], cd.warm[2 * cd.ncomp + id]};
    LamResult R;
    laminate_solve(M, f, n, cd.cp[id], cd.cm[id], a0, R);
    double fp[9], fm[9], p1[9], p2[9];
    if (R.inadmissible) {
      ++inad;
#pragma unroll
      for (int c = 0; c < 9; ++c) p1[c] = p2[c] = 0.0;
    } else {
      itmax = max(itmax, (unsigned)R.iterations);
      // the phases of the returned state, as the last update_phases
      form_phases(f, n, cd.cp[id], cd.cm[id], R.a, fp, fm);
      NhState s1, s2;
      if (!law_eval(M.law[1], fp, p1, s1))
#pragma unroll
        for (int c = 0; c < 9; ++c) p1[c] = 0.0;
      if (!law_eval(M.law[0], fm, p2, s2))
#pragma unroll
        for (int c = 0; c < 9; ++c) p2[c] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      pp[c * cd.ncomp + id] = p1[c];
      pm[c * cd.ncomp + id] = p2[c];
    }
  }
  warp_stats(st, inad, 0, 0, itmax);
}

// phase_averages (postprocess.cpp:49-106): chunk partials of
// [sum+ (9), weight+, sum- (9), weight-]
static __global__ void __launch_bounds__(kEwThreads) k_phase_sum(MatParams M, CellData cd,
                                                                 const double* __restrict__ fin, int64_t N,
                                                                 const double* __restrict__ pp,
                                                                 const double* __restrict__ pm, Chunks ch,
                                                                 double* partials) {
  double acc[20];
#pragma unroll
  for (int c = 0; c < 20; ++c) acc[c] = 0.0;
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
    const int32_t id = cd.cid[cell];
    if (id >= 0) {
      const double cpl = cd.cp[id], cmi = cd.cm[id];
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        acc[c] += cpl * pp[c * cd.ncomp + id];
        acc[10 + c] += cmi * pm[c * cd.ncomp + id];
      }
      acc[9] += cpl;
      acc[19] += cmi;
    } else {
      double f[9], p[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell];
      NhState s;
      if (!law_eval(id == -2 ? M.law[1] : M.law[0], f, p, s))
#pragma unroll
        for (int c = 0; c < 9; ++c) p[c] = 0.0;
      const int o = id == -2 ? 0 : 10;
#pragma unroll
      for (int c = 0; c < 9; ++c) acc[o + c] += p[c];
      acc[o + 9] += 1.0;
    }
  }
  block_reduce_store<20>(acc, partials, blockIdx.x);
}

// CG step P1 (solver.cpp:186-197, deferred): x += step_prev * pdir_old (the
// x update of the previous iteration, applied where pdir_old is read anyway),
// pdir = first ? r : r + beta * pdir_old ; y = A(F) : pdir (matrix free NH,
// packed tangent for composites) for one cell. x may be null (operator-level
// calls).
struct MatvecArgs {
  MatParams M;
  CellData cd;
  const double* fin;
  Shift9 sh;
  const double* r;
  double* pdir;
  double beta;
  int first;
  int64_t N;
  double* xv;
  double step_prev;
  // bulk kernel only: per-tile sums of pdir . q (pdir^T A pdir; equals
  // pdir^T Pi(q) of solver.cpp:181 because pdir lies in the range of the
  // self-adjoint projection Pi), one value per warp of each kMvT-cell tile
  // ([tile][warp]); may be null
  double* pq_part;
};

__device__ __forceinline__ void mv_cell(const MatvecArgs& a, int64_t cell, double* y) {
  const int64_t N = a.N;
  // all loads are issued before any store (pdir / xv may not be reordered
  // across stores by the compiler otherwise)
  double f[9], x[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) x[c] = __ldg(a.r + c * N + cell);
#pragma unroll
  for (int c = 0; c < 9; ++c) f[c] = __ldg(a.fin + c * N + cell) + a.sh.v[c];
  if (!a.first) {
    double po[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) po[c] = a.pdir[c * N + cell];
    if (a.xv) {
      double xo[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) xo[c] = a.xv[c * N + cell];
#pragma unroll
      for (int c = 0; c < 9; ++c) a.xv[c * N + cell] = xo[c] + a.step_prev * po[c];
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) x[c] += a.beta * po[c];
  }
#pragma unroll
  for (int c = 0; c < 9; ++c) a.pdir[c * N + cell] = x[c];
  const int32_t id = a.cd.cid[cell];
  if (id >= 0) {
    // composite: packed effective tangent of this Newton iteration
    packed45_apply(a.cd.t45 + id, a.cd.ncomp, x, y);
  } else {
    const LawP L = id == -2 ? a.M.law[1] : a.M.law[0];
    NhState s;
    double p[9];
    if (law_eval(L, f, p, s))
      law_apply(L, s, x, y);
    else
      for (int c = 0; c < 9; ++c) y[c] = x[c];
  }
}

template <int MINB = 1>
static __global__ void __launch_bounds__(kEwThreads, MINB) k_matvec(MatvecArgs a, double* __restrict__ q) {
  for (int64_t cell = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < a.N;
       cell += int64_t(gridDim.x) * blockDim.x) {
    double y[9];
    mv_cell(a, cell, y);
#pragma unroll
    for (int c = 0; c < 9; ++c) q[c * a.N + cell] = y[c];
  }
}

// Bulk-staged matvec (same arithmetic as k_matvec, bitwise): a producer warp
// streams the tile's component rows (r, F, pdir, x: 9 rows of kMvT cells
// each, plus the cell ids) into a ring of shared-memory stages with
// cp.async.bulk; 8 consumer warps compute one cell per thread from shared
// memory and store pdir, x and q. Cells past the last full tile are done by
// block 0 with direct loads. Requires N even and 16-byte aligned rows.
constexpr int kMvT = 256;
constexpr int kMvHead = 128;  // barriers ahead of the ring

template <bool FIRST, bool HASX>
struct MvStage {
  static constexpr int kRows = 18 + (FIRST ? 0 : 9) + ((!FIRST && HASX) ? 9 : 0);
  static constexpr int kBytes = kRows * kMvT * 8 + kMvT * 4;
};

template <bool FIRST, bool HASX>
static __global__ void __launch_bounds__(kMvT + 32, 1) k_matvec_bulk(MatvecArgs a, double* __restrict__ q,
                                                                      int nstages) {
  using S = MvStage<FIRST, HASX>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 8;
  unsigned char* buf = smem_raw + kMvHead;
  const int64_t N = a.N;
  const int64_t nfull = N / kMvT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMvT / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == kMvT / 32) {  // producer
    if (lane == 0) {
      Ring rg(nstages);
      int k = 0;
      for (int64_t t = blockIdx.x; t < nfull; t += gridDim.x, ++k, rg.next()) {
        if (k >= nstages) mbar_wait(&empty[rg.s], rg.phase ^ 1u);
        double* d = reinterpret_cast<double*>(buf + size_t(rg.s) * S::kBytes);
        const int64_t off = t * kMvT;
        constexpr uint32_t rb = kMvT * 8;
        mbar_expect_tx(&full[rg.s], S::kBytes);
#pragma unroll 1
        for (int c = 0; c < 9; ++c) {
          bulk_g2s(d + c * kMvT, a.r + c * N + off, rb, &full[rg.s]);
          bulk_g2s(d + (9 + c) * kMvT, a.fin + c * N + off, rb, &full[rg.s]);
          if (!FIRST) bulk_g2s(d + (18 + c) * kMvT, a.pdir + c * N + off, rb, &full[rg.s]);
          if (!FIRST && HASX) bulk_g2s(d + (27 + c) * kMvT, a.xv + c * N + off, rb, &full[rg.s]);
        }
        bulk_g2s(d + S::kRows * kMvT, a.cd.cid + off, kMvT * 4, &full[rg.s]);
      }
    }
    return;
  }
  const int tid = threadIdx.x;
  Ring rg(nstages);
  for (int64_t t = blockIdx.x; t < nfull; t += gridDim.x, rg.next()) {
    mbar_wait(&full[rg.s], rg.phase);
    const double* d = reinterpret_cast<const double*>(buf + size_t(rg.s) * S::kBytes);
    const int64_t cell = t * kMvT + tid;
    double x[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) x[c] = d[c * kMvT + tid];
    if (!FIRST) {
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        const double po = d[(18 + c) * kMvT + tid];
        if (HASX) a.xv[c * N + cell] = d[(27 + c) * kMvT + tid] + a.step_prev * po;
        x[c] += a.beta * po;
      }
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) a.pdir[c * N + cell] = x[c];
    const int32_t id = reinterpret_cast<const int32_t*>(d + S::kRows * kMvT)[tid];
    double y[9];
    if (id >= 0) {
      packed45_apply(a.cd.t45 + id, a.cd.ncomp, x, y);
    } else {
      double f[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) f[c] = d[(9 + c) * kMvT + tid] + a.sh.v[c];
      const LawP L = id == -2 ? a.M.law[1] : a.M.law[0];
      NhState s;
      if (law_state(L, f, s))
        law_apply(L, s, x, y);
      else
#pragma unroll
        for (int c = 0; c < 9; ++c) y[c] = x[c];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rg.s]);
#pragma unroll
    for (int c = 0; c < 9; ++c) q[c * N + cell] = y[c];
    if (a.pq_part) {
      // fixed-order sum per warp of the tile (9 products per cell, warp
      // tree); no block barrier: the consumer warps stay decoupled
      double dq = 0.0;
#pragma unroll
      for (int c = 0; c < 9; ++c) dq += x[c] * y[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dq += __shfl_down_sync(0xffffffffu, dq, o);
      if (lane == 0) a.pq_part[t * (kMvT / 32) + warp] = dq;
    }
  }
  if (blockIdx.x == 0) {
    for (int64_t cell = nfull * kMvT + tid; cell < N; cell += kMvT) {
      double y[9];
      mv_cell(a, cell, y);
#pragma unroll
      for (int c = 0; c < 9; ++c) q[c * N + cell] = y[c];
    }
  }
}

// Packed effective tangents of all composite cells at (F, warm starts): the
// tangent half of stress_sweep(tangents45) (cell_material.cpp:146-160),
// evaluated once per Newton iteration.
// 2 blocks per SM (255 registers): 32.2 ms at 512^3; 3 blocks 32.2, 4 blocks 38.0
static __global__ void __launch_bounds__(128, 2)
    k_comp_tangent(MatParams M, CellData cd, const double* __restrict__ fin, Shift9 sh, double* __restrict__ t45,
                   int64_t N) {
  for (int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; id < cd.ncomp;
       id += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cell = cd.ccell[id];
    double f[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell] + sh.v[c];
    const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
    const double a[3] = {cd.warm[id], cd.warm[cd.ncomp + id], cd.warm[2 * cd.ncomp + id]};
    LamTangent S;
    if (det3(f) > 0.0) {
      laminate_prepare(M, f, n, cd.cp[id], cd.cm[id], a, S);
    } else {
      S.ok = false;  // inadmissible macro state: identity (cell_material.cpp:134)
    }
    laminate_tangent45(M, S, t45 + id, cd.ncomp);
  }
}

// CG step P6 (solver.cpp:187-190): r -= step * ap ; partial sum of r^2
static __global__ void __launch_bounds__(kEwThreads) k_cg_update(double* __restrict__ r,
                                                          const double* __restrict__ ap, double step,
                                                          int64_t N, Chunks ch, double* partials) {
  double acc[1] = {0.0};
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const int64_t i = c * N + cell;
      const double rv = r[i] + (-step) * ap[i];
      r[i] = rv;
      acc[0] += rv * rv;
    }
  }
  block_reduce_store<1>(acc, partials, blockIdx.x);
}

// pending x += step * pdir of the last CG iteration (solver.cpp:186)
static __global__ void k_axpy(double* __restrict__ x, const double* __restrict__ p, double step, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] += step * p[i];
}

// ftrial = (F + shiftF) + s x ; per-component sums for pin_mean
static __global__ void __launch_bounds__(kEwThreads) k_trial(const double* __restrict__ f, Shift9 sh,
                                                      const double* __restrict__ x, double s,
                                                      double* __restrict__ ft, int64_t N, Chunks ch,
                                                      double* partials) {
  double acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0;
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const double v = (f[c * N + cell] + sh.v[c]) + s * x[c * N + cell];
      ft[c * N + cell] = v;
      acc[c] += v;
    }
  }
  block_reduce_store<9>(acc, partials, blockIdx.x);
}

// f = f + shift (materialize), per-component sums of the result
static __global__ void __launch_bounds__(kEwThreads) k_materialize(double* __restrict__ f, Shift9 sh, int64_t N,
                                                            Chunks ch, double* partials) {
  double acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0;
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const double v = f[c * N + cell] + sh.v[c];
      f[c * N + cell] = v;
      acc[c] += v;
    }
  }
  block_reduce_store<9>(acc, partials, blockIdx.x);
}

static __global__ void k_fill9(double* f, Shift9 val, int64_t N) {
  for (int64_t cell = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < N;
       cell += int64_t(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 9; ++c) f[c * N + cell] = val.v[c];
  }
}

// y_cell = A x_cell with packed 45 tangents (API compatibility path)
static __global__ void k_t45_matvec(const double* __restrict__ t45, const double* __restrict__ x, double* __restrict__ y,
                             int64_t N) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += int64_t(gridDim.x) * blockDim.x) {
    const double* a = t45 + 45 * i;
    double xv[9], yv[9];
    for (int c = 0; c < 9; ++c) {
      xv[c] = x[c * N + i];
      yv[c] = 0.0;
    }
    int t = 0;
    for (int r = 0; r < 9; ++r) {
      yv[r] += a[t] * xv[r];
      ++t;
      for (int c = r + 1; c < 9; ++c, ++t) {
        yv[r] += a[t] * xv[c];
        yv[c] += a[t] * xv[r];
      }
    }
    for (int c = 0; c < 9; ++c) y[c * N + i] = yv[c];
  }
}

// packed tangent = columns of A applied to unit vectors (matrix free), sym.
static __global__ void k_tangent45(MatParams M, CellData cd, const double* __restrict__ fin, double* __restrict__ t45,
                            int64_t N) {
  for (int64_t cell = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < N;
       cell += int64_t(gridDim.x) * blockDim.x) {
    double f[9];
    for (int c = 0; c < 9; ++c) f[c] = fin[c * N + cell];
    double A[81];
    const int32_t id = cd.cid[cell];
    for (int col = 0; col < 9; ++col) {
      double x[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, y[9];
      x[col] = 1.0;
      if (id >= 0) {
        const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
        const double a[3] = {cd.warm[id], cd.warm[cd.ncomp + id], cd.warm[2 * cd.ncomp + id]};
        if (det3(f) > 0.0)
          laminate_apply(M, f, n, cd.cp[id], cd.cm[id], a, x, y);
        else
          for (int c = 0; c < 9; ++c) y[c] = x[c];
      } else {
        const LawP L = id == -2 ? M.law[1] : M.law[0];
        NhState s;
        double p[9];
        if (law_eval(L, f, p, s))
          law_apply(L, s, x, y);
        else
          for (int c = 0; c < 9; ++c) y[c] = x[c];
      }
      for (int r = 0; r < 9; ++r) A[9 * r + col] = y[r];
    }
    int t = 0;
    for (int r = 0; r < 9; ++r)
      for (int c = r; c < 9; ++c) t45[45 * cell + (t++)] = 0.5 * (A[9 * r + c] + A[9 * c + r]);
  }
}

// Deterministic final reduction: one block per value, fixed strided
// assignment + fixed tree.
static __global__ void k_reduce_partials(const double* __restrict__ partials, int64_t nblocks, int nred,
                                  double* __restrict__ out) {
  __shared__ double sm[1024];
  const int r = blockIdx.x;
  double s = 0.0;
  for (int64_t b = threadIdx.x; b < nblocks; b += blockDim.x) s += partials[b * nred + r];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x >> 1; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = sm[0];
}

// First level for long partial vectors: block b sums partials
// [b chunk, (b + 1) chunk) of every value in a fixed order (strided
// assignment + fixed tree) -> out[b][nred]; k_reduce_partials finishes.
static __global__ void k_reduce_chunks(const double* __restrict__ partials, int64_t nblocks, int nred, int chunk,
                                       double* __restrict__ out) {
  __shared__ double sm[256];
  const int64_t b0 = int64_t(blockIdx.x) * chunk;
  const int64_t b1 = min(b0 + int64_t(chunk), nblocks);
  for (int r = 0; r < nred; ++r) {
    double s = 0.0;
    for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) s += partials[b * nred + r];
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x >> 1; w > 0; w >>= 1) {
      if (int(threadIdx.x) < w) sm[threadIdx.x] += sm[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[int64_t(blockIdx.x) * nred + r] = sm[0];
    __syncthreads();
  }
}

// ------------------------------------------------------------ FFT functors
// FIELDS = real 9N-field streams (reads + writes) besides the spectrum; used
// for the algorithmic-bytes bookkeeping of the profiler.
// Two interfaces: operator() works on all 9 components of a cell (staged
// generic-size path), comp() on one component (register-resident pow2 path,
// NSC scalar accumulators + optional per-component sums, see fft_rr.cuh).
struct ProdLoad9 {
  static constexpr int NRED = 0;
  static constexpr int FIELDS = 1;
  const double* src;
  int64_t N;
  __device__ __forceinline__ void operator()(int64_t cell, double* v, double*) const {
#pragma unroll
    for (int c = 0; c < 9; ++c) v[c] = src[c * N + cell];
  }
  __device__ __forceinline__ double comp(int c, int64_t cell) const { return src[c * N + cell]; }
};

struct ConsStore9 {
  static constexpr int NRED = 0;
  static constexpr int NSC = 0;
  static constexpr bool PERCOMP = false;
  static constexpr int FIELDS = 1;
  static constexpr bool LOADS = false;  // the epilogue reads fields (ring kernel: latency exposed)
  static constexpr bool PRELOAD = false;  // fields requested ahead of the inverse stages (zinv_finish)
  double* dst;
  int64_t N;
  __device__ __forceinline__ void operator()(int64_t cell, const double* v, double*) const {
#pragma unroll
    for (int c = 0; c < 9; ++c) dst[c * N + cell] = v[c];
  }
  __device__ __forceinline__ void prefetch(int, int64_t, int64_t) const {}
  __device__ __forceinline__ double comp(int c, int64_t cell, double v, double*) const {
    dst[c * N + cell] = v;
    return 0.0;
  }
};

// CG with the step length known before the projection (pdir^T A pdir comes
// from the matvec, MatvecArgs::pq_part): the z-inverse applies
// r' = r - s Pi(q) itself and sums r'^T r' (solver.cpp:186-190), so
// ap = Pi(q) is never stored and k_cg_update's pass over r and ap
// disappears. r' goes to a second field (the host swaps the slots).
struct ConsCgUpdate {
  static constexpr int NRED = 1;
  static constexpr int NSC = 1;
  static constexpr bool PERCOMP = false;
  static constexpr int FIELDS = 2;
  static constexpr bool LOADS = true;
  static constexpr bool PRELOAD = true;
  const double* r;
  double* rnew;
  double step;
  int64_t N;
  __device__ __forceinline__ double load(int c, int64_t cell) const { return r[c * N + cell]; }
  __device__ __forceinline__ double comp_pre(int c, int64_t cell, double v, double rold, double* sc) const {
    const double rn = rold - step * v;
    rnew[c * N + cell] = rn;
    sc[0] += rn * rn;
    return 0.0;
  }
  __device__ __forceinline__ void operator()(int64_t cell, const double* v, double* acc) const {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const double rn = r[c * N + cell] - step * v[c];
      rnew[c * N + cell] = rn;
      acc[0] += rn * rn;
    }
  }
  __device__ __forceinline__ void prefetch(int c, int64_t cell0, int64_t n) const {
    bulk_prefetch_l2(r + c * N + cell0, size_t(n) * 8);
  }
  __device__ __forceinline__ double comp(int c, int64_t cell, double v, double* sc) const {
    const double rn = r[c * N + cell] - step * v;
    rnew[c * N + cell] = rn;
    sc[0] += rn * rn;
    return 0.0;
  }
};

// run_basic F update (solver.cpp:135-149): F_new = fbar - Pi(tau)/alpha,
// diff against the pinned F_old; sums of diff^2 and of F_new.
struct ConsBasic {
  static constexpr int NRED = 10;
  static constexpr int FIELDS = 2;
  static constexpr bool LOADS = true;  // the epilogue reads fields (ring kernel: latency exposed)
  static constexpr bool PRELOAD = false;  // fields requested ahead of the inverse stages (zinv_finish)
  const double* fold;
  Shift9 fold_shift;
  double* fnew;
  Shift9 fbar;
  double alpha;
  int64_t N;
  __device__ __forceinline__ void operator()(int64_t cell, const double* v, double* acc) const {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const double fn = fbar.v[c] - v[c] / alpha;
      const double d = fn - (fold[c * N + cell] + fold_shift.v[c]);
      acc[0] += d * d;
      acc[1 + c] += fn;
      fnew[c * N + cell] = fn;
    }
  }
  static constexpr int NSC = 1;
  static constexpr bool PERCOMP = true;
  // the old F rows of cells [cell0, cell0 + n) into L2 ahead of comp()
  __device__ __forceinline__ void prefetch(int c, int64_t cell0, int64_t n) const {
    bulk_prefetch_l2(fold + c * N + cell0, size_t(n) * 8);
  }
  __device__ __forceinline__ double comp(int c, int64_t cell, double v, double* sc) const {
    const double fn = fbar.v[c] - v / alpha;
    const double d = fn - (fold[c * N + cell] + fold_shift.v[c]);
    sc[0] += d * d;
    fnew[c * N + cell] = fn;
    return fn;
  }
};

// Newton residual (solver.cpp:209-225): r = -Pi(P), sum of Pi(P)^2
struct ConsResid {
  static constexpr int NRED = 1;
  static constexpr int NSC = 1;
  static constexpr bool PERCOMP = false;
  static constexpr int FIELDS = 1;
  static constexpr bool LOADS = false;  // the epilogue reads fields (ring kernel: latency exposed)
  static constexpr bool PRELOAD = false;  // fields requested ahead of the inverse stages (zinv_finish)
  double* r;
  int64_t N;
  __device__ __forceinline__ void operator()(int64_t cell, const double* v, double* acc) const {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      r[c * N + cell] = -v[c];
      acc[0] += v[c] * v[c];
    }
  }
  __device__ __forceinline__ void prefetch(int, int64_t, int64_t) const {}
  __device__ __forceinline__ double comp(int c, int64_t cell, double v, double* sc) const {
    r[c * N + cell] = -v;
    sc[0] += v * v;
    return 0.0;
  }
};

// CG (solver.cpp:180-181): ap = Pi(q), sum of pdir . ap
struct ConsCg {
  static constexpr int NRED = 1;
  static constexpr int NSC = 1;
  static constexpr bool PERCOMP = false;
  static constexpr int FIELDS = 2;
  static constexpr bool LOADS = true;  // the epilogue reads fields (ring kernel: latency exposed)
  static constexpr bool PRELOAD = false;  // fields requested ahead of the inverse stages (zinv_finish)
  double* ap;
  const double* pdir;
  int64_t N;
  __device__ __forceinline__ void operator()(int64_t cell, const double* v, double* acc) const {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      ap[c * N + cell] = v[c];
      acc[0] += pdir[c * N + cell] * v[c];
    }
  }
  __device__ __forceinline__ void prefetch(int c, int64_t cell0, int64_t n) const {
    bulk_prefetch_l2(pdir + c * N + cell0, size_t(n) * 8);
  }
  __device__ __forceinline__ double comp(int c, int64_t cell, double v, double* sc) const {
    ap[c * N + cell] = v;
    sc[0] += pdir[c * N + cell] * v;
    return 0.0;
  }
};

}  // namespace combo_dev
