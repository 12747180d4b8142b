// Doubly-fine material grid (DFMG) on the GPU (reference src/dfmg.cpp).
//
// Every staggered stress component is the average over its 8 adjacent
// doubly-fine cells (dfc) of the host cell's law evaluated on the locally
// assembled F (gather_dfc, dfmg.cpp:27-47). The reference evaluates each dfc
// four times (once per position class, dfmg.cpp:138-174, identical inputs);
// here each dfc (host cell, code) is evaluated exactly once:
//   k_dfmg_eval   one thread per dfc -> P_dfc [9][8][N], warm start per dfc
//   k_dfmg_gather per cell, per component: sum over codes 0..7 (reference
//                 order) of P_dfc at the class's host cell, / 8
// The linearization (dfmg_tangent_pass + dfmg_tangent_matvec,
// dfmg.cpp:178-253) is matrix free for pure hosts and uses per-dfc packed
// tangents (pack45) for composite hosts, built once per Newton iteration.
// Sweep statistics reproduce the reference's multiplicities: inadmissible and
// failure counts are incremented by every one of the 4 evaluations, back
// projections and the iteration maximum by the owner only (dfmg.cpp:69-109).
#include "context.hpp"

using namespace combo_dev;
using namespace combo_host;

namespace {

struct Dims3 {
  int64_t n1, n2, n3;
  __device__ __forceinline__ int64_t at(int64_t i, int64_t j, int64_t k) const {
    i %= n1;
    j %= n2;
    k %= n3;
    if (i < 0) i += n1;
    if (j < 0) j += n2;
    if (k < 0) k += n3;
    return (i * n2 + j) * n3 + k;
  }
};

// gather_dfc (dfmg.cpp:27-47)
__device__ __forceinline__ void gather_dfc(const double* __restrict__ f, const Shift9& sh, int64_t N, const Dims3& d,
                                           int64_t i, int64_t j, int64_t k, int code, double* m) {
  const int s1 = code & 1, s2 = (code >> 1) & 1, s3 = (code >> 2) & 1;
  const int64_t c0 = d.at(i, j, k);
  const int64_t c12 = d.at(i + s1, j + s2, k);
  const int64_t c13 = d.at(i + s1, j, k + s3);
  const int64_t c23 = d.at(i, j + s2, k + s3);
  m[0] = f[0 * N + c0] + sh.v[0];
  m[4] = f[4 * N + c0] + sh.v[4];
  m[8] = f[8 * N + c0] + sh.v[8];
  m[1] = f[1 * N + c12] + sh.v[1];
  m[3] = f[3 * N + c12] + sh.v[3];
  m[2] = f[2 * N + c13] + sh.v[2];
  m[6] = f[6 * N + c13] + sh.v[6];
  m[5] = f[5 * N + c23] + sh.v[5];
  m[7] = f[7 * N + c23] + sh.v[7];
}

// mode 0: stress sweep (dfmg_stress); mode 1: tangent pass re-solve
// (dfmg_tangent_pass) -- warm starts read from the pre-launch state and
// written back per dfc (each dfc has exactly one writer).
static __global__ void __launch_bounds__(256) k_dfmg_eval(MatParams M, CellData cd, const double* __restrict__ fin,
                                                          Shift9 sh, Dims3 d, double* __restrict__ warm8,
                                                          double* __restrict__ pd, int mode, Stats* st) {
  const int64_t N = d.n1 * d.n2 * d.n3;
  const int64_t nw = 8 * cd.ncomp;
  unsigned long long inad = 0, fail = 0, bp = 0;
  unsigned int itmax = 0;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < 8 * N; t += int64_t(gridDim.x) * blockDim.x) {
    const int code = int(t / N);
    const int64_t cell = t - code * N;
    const int64_t k = cell % d.n3, j = (cell / d.n3) % d.n2, i = cell / (d.n2 * d.n3);
    double f[9], p[9];
    gather_dfc(fin, sh, N, d, i, j, k, code, f);
    const int32_t id = cd.cid[cell];
    if (id >= 0) {
      const int64_t w = int64_t(id) * 8 + code;
      const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
      const double a0[3] = {warm8[w], warm8[nw + w], warm8[2 * nw + w]};
      LamResult R;
      laminate_solve(M, f, n, cd.cp[id], cd.cm[id], a0, R);
      if (R.inadmissible) {
        inad += mode == 0 ? 4 : 1;
#pragma unroll
        for (int c = 0; c < 9; ++c) p[c] = 0.0;
      } else {
        if (!R.converged) fail += mode == 0 ? 4 : 1;
        bp += (unsigned long long)R.back_projections;
        itmax = max(itmax, (unsigned)R.iterations);
        warm8[w] = R.a[0];
        warm8[nw + w] = R.a[1];
        warm8[2 * nw + w] = R.a[2];
#pragma unroll
        for (int c = 0; c < 9; ++c) p[c] = R.p[c];
      }
    } else {
      NhState s;
      const LawP L = id == -2 ? M.law[1] : M.law[0];
      if (!law_eval(L, f, p, s)) {
        inad += mode == 0 ? 4 : 1;
#pragma unroll
        for (int c = 0; c < 9; ++c) p[c] = 0.0;
      }
    }
    if (mode == 0) {
#pragma unroll
      for (int c = 0; c < 9; ++c) pd[(int64_t(c) * 8 + code) * N + cell] = p[c];
    }
  }
  if (mode == 1) fail = 0;  // the tangent pass's failures are not reported (solver.cpp:76-78)
  warp_stats(st, inad, fail, mode == 0 ? bp : 0, itmax);
}

// P[c](cell) = (1/8) sum_code pd[c][code](host(cell, class(c), code)); out =
// P - alpha F; P sums -> partials (P-bar).
static __global__ void __launch_bounds__(256) k_dfmg_gather(const double* __restrict__ pd, Dims3 d,
                                                            const double* __restrict__ fin, Shift9 sh, double alpha,
                                                            double* __restrict__ out, double* partials, int reduce) {
  const int64_t N = d.n1 * d.n2 * d.n3;
  double acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0;
  for (int64_t cell = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < N;
       cell += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = cell % d.n3, j = (cell / d.n3) % d.n2, i = cell / (d.n2 * d.n3);
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      // position classes (dfmg.cpp:119-124): diagonal, (0,1), (0,2), (1,2)
      const int cls = (c == 0 || c == 4 || c == 8) ? 0 : (c == 1 || c == 3) ? 1 : (c == 2 || c == 6) ? 2 : 3;
      double s = 0.0;
#pragma unroll
      for (int code = 0; code < 8; ++code) {
        const int l1 = code & 1, l2 = (code >> 1) & 1, l3 = (code >> 2) & 1;
        int64_t hi = i, hj = j, hk = k;
        if (cls == 1) {
          hi -= l1;
          hj -= l2;
        } else if (cls == 2) {
          hi -= l1;
          hk -= l3;
        } else if (cls == 3) {
          hj -= l2;
          hk -= l3;
        }
        s += pd[(int64_t(c) * 8 + code) * N + d.at(hi, hj, hk)];
      }
      const double p = s / 8.0;
      acc[c] += p;
      out[c * N + cell] = alpha != 0.0 ? p + (-alpha) * (fin[c * N + cell] + sh.v[c]) : p;
    }
  }
  if (reduce) block_reduce_store<9>(acc, partials, blockIdx.x);
}

// per-dfc packed tangents of composite hosts: t8[t][id*8+code]
static __global__ void __launch_bounds__(128) k_dfmg_comp_tangent(MatParams M, CellData cd,
                                                                  const double* __restrict__ fin, Shift9 sh, Dims3 d,
                                                                  const double* __restrict__ warm8,
                                                                  double* __restrict__ t8) {
  const int64_t N = d.n1 * d.n2 * d.n3;
  const int64_t nw = 8 * cd.ncomp;
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < nw; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t id = w / 8;
    const int code = int(w - id * 8);
    const int64_t cell = cd.ccell[id];
    const int64_t k = cell % d.n3, j = (cell / d.n3) % d.n2, i = cell / (d.n2 * d.n3);
    double f[9];
    gather_dfc(fin, sh, N, d, i, j, k, code, f);
    const double n[3] = {cd.nrm[id], cd.nrm[cd.ncomp + id], cd.nrm[2 * cd.ncomp + id]};
    const double a[3] = {warm8[w], warm8[nw + w], warm8[2 * nw + w]};
    LamTangent S;
    if (det3(f) > 0.0)
      laminate_prepare(M, f, n, cd.cp[id], cd.cm[id], a, S);
    else
      S.ok = false;
    laminate_tangent45(M, S, t8 + w, nw);
  }
}

// y_dfc = A_dfc x_dfc for every dfc -> yd [9][8][N]
static __global__ void __launch_bounds__(256) k_dfmg_apply(MatParams M, CellData cd, const double* __restrict__ fin,
                                                           Shift9 sh, Dims3 d, const double* __restrict__ x,
                                                           const double* __restrict__ t8, double* __restrict__ yd) {
  const int64_t N = d.n1 * d.n2 * d.n3;
  const int64_t nw = 8 * cd.ncomp;
  Shift9 zero;
#pragma unroll
  for (int c = 0; c < 9; ++c) zero.v[c] = 0.0;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < 8 * N; t += int64_t(gridDim.x) * blockDim.x) {
    const int code = int(t / N);
    const int64_t cell = t - code * N;
    const int64_t k = cell % d.n3, j = (cell / d.n3) % d.n2, i = cell / (d.n2 * d.n3);
    double xv[9], y[9];
    gather_dfc(x, zero, N, d, i, j, k, code, xv);
    const int32_t id = cd.cid[cell];
    if (id >= 0) {
      packed45_apply(t8 + int64_t(id) * 8 + code, nw, xv, y);
    } else {
      double f[9], p[9];
      gather_dfc(fin, sh, N, d, i, j, k, code, f);
      NhState s;
      const LawP L = id == -2 ? M.law[1] : M.law[0];
      if (law_eval(L, f, p, s))
        law_apply(L, s, xv, y);
      else
        for (int c = 0; c < 9; ++c) y[c] = xv[c];
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) yd[(int64_t(c) * 8 + code) * N + cell] = y[c];
  }
}

// pdir = first ? r : r + beta pdir
static __global__ void k_pdir(const double* __restrict__ r, double* __restrict__ pdir, double beta, int first,
                              int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    pdir[i] = first ? r[i] : r[i] + beta * pdir[i];
}

Dims3 dims3(const combo_ctx* c) { return Dims3{c->dims[0], c->dims[1], c->dims[2]}; }

void ensure_dfmg(combo_ctx* c) {
  const size_t nw = size_t(8 * std::max<int64_t>(c->ncomp, 1));
  if (c->dfmg_warm.n != 3 * nw) {
    c->dfmg_warm.alloc(3 * nw);
    COMBO_CK(cudaMemsetAsync(c->dfmg_warm.p, 0, 3 * nw * 8, c->stream));
  }
  c->dfmg_pd.alloc(size_t(72 * c->N));
}

int grid8(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

}  // namespace

namespace combo_host {

// dfmg_stress (dfmg.cpp:128-176): out = P - alpha F, P sums -> slot
void dfmg_sweep(combo_ctx* c, const double* fin, const Shift9& sh, double alpha, double* out, int slot) {
  ensure_dfmg(c);
  const int64_t N = c->N;
  {
    ProfScope ps(c, kTagSweep, 8.0 * 72.0 * double(N) * 2.0 + 8.0 * 112.0 * double(c->ncomp));
    k_dfmg_eval<<<grid8(8 * N), 256, 0, c->stream>>>(c->mp, c->cell_data(), fin, sh, dims3(c), c->dfmg_warm.p,
                                                      c->dfmg_pd.p, 0, c->dstats.p);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
  }
  const int g = ew_grid(N);
  ensure_partials(c, int64_t(g) * 9);
  {
    ProfScope ps(c, kTagSweep, 8.0 * 72.0 * double(N) + 144.0 * double(N));
    k_dfmg_gather<<<g, kEwThreads, 0, c->stream>>>(c->dfmg_pd.p, dims3(c), fin, sh, alpha, out, c->partials.p, 1);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
  }
  reduce_partials(c, g, 9, slot);
}

// dfmg_tangent_pass (dfmg.cpp:178-207): re-solve from the current warm
// starts, then per-dfc packed tangents of the composite hosts.
void dfmg_tangent_prepare(combo_ctx* c, const double* fin, const Shift9& sh) {
  ensure_dfmg(c);
  const int64_t N = c->N;
  {
    ProfScope ps(c, kTagOther, 8.0 * 72.0 * double(N) + 8.0 * 112.0 * double(c->ncomp));
    k_dfmg_eval<<<grid8(8 * N), 256, 0, c->stream>>>(c->mp, c->cell_data(), fin, sh, dims3(c), c->dfmg_warm.p,
                                                      nullptr, 1, c->dstats.p);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
  }
  if (c->ncomp) {
    c->dfmg_t8.alloc(size_t(45 * 8 * c->ncomp));
    ProfScope ps(c, kTagOther, 8.0 * double(c->ncomp) * (72.0 + 64.0 + 360.0));
    k_dfmg_comp_tangent<<<unsigned(std::min<int64_t>((8 * c->ncomp + 127) / 128, 148 * 32)), 128, 0, c->stream>>>(
        c->mp, c->cell_data(), fin, sh, dims3(c), c->dfmg_warm.p, c->dfmg_t8.p);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
  }
}

// q = d dfmg_stress / dF [pdir] with pdir = first ? r : r + beta pdir
// (dfmg_tangent_matvec, dfmg.cpp:209-253)
void dfmg_matvec(combo_ctx* c, const double* fin, const Shift9& sh, const double* r, double* pdir, double beta,
                 bool first, double* q) {
  const int64_t N = c->N;
  {
    ProfScope ps(c, kTagMatvec, (first ? 144.0 : 216.0) * double(N));
    k_pdir<<<ew_grid(9 * N), kEwThreads, 0, c->stream>>>(r, pdir, beta, first ? 1 : 0, 9 * N);
    ++c->launches;
  }
  {
    ProfScope ps(c, kTagMatvec, 8.0 * 72.0 * double(N) * 3.0 + 8.0 * 360.0 * double(c->ncomp));
    k_dfmg_apply<<<grid8(8 * N), 256, 0, c->stream>>>(c->mp, c->cell_data(), fin, sh, dims3(c), pdir, c->dfmg_t8.p,
                                                       c->dfmg_pd.p);
    ++c->launches;
  }
  {
    ProfScope ps(c, kTagMatvec, 8.0 * 72.0 * double(N) + 72.0 * double(N));
    Shift9 z{};
    k_dfmg_gather<<<ew_grid(N), kEwThreads, 0, c->stream>>>(c->dfmg_pd.p, dims3(c), fin, z, 0.0, q, nullptr, 0);
    ++c->launches;
  }
  COMBO_CK(cudaGetLastError());
}

}  // namespace combo_host

// ====================================================================== C-ABI
namespace {
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

const double* stage_in(combo_ctx* c, const double* p, int mem, int slot) {
  if (mem == COMBO_MEM_DEVICE) return p;
  c->scratch[slot].alloc(size_t(9 * c->N));
  COMBO_CK(cudaMemcpyAsync(c->scratch[slot].p, p, size_t(9 * c->N) * 8, cudaMemcpyHostToDevice, c->stream));
  return c->scratch[slot].p;
}
double* stage_out(combo_ctx* c, double* p, int mem, int slot) {
  if (mem == COMBO_MEM_DEVICE) return p;
  c->scratch[slot].alloc(size_t(9 * c->N));
  return c->scratch[slot].p;
}
void finish_out(combo_ctx* c, double* host, const double* dev, int mem) {
  if (mem != COMBO_MEM_DEVICE)
    COMBO_CK(cudaMemcpyAsync(host, dev, size_t(9 * c->N) * 8, cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaStreamSynchronize(c->stream));
}
}  // namespace

extern "C" {

int combo_dfmg_stress(combo_ctx* c, const double* F, double* P, combo_sweep_stats* st, int mem) {
  return guarded(c, [&] {
    if (!c->bound) throw ComboError(COMBO_ERR_STATE, "materials not bound (combo_bind_materials)");
    require_single(c);
    ensure_scratch(c);
    const double* f = stage_in(c, F, mem, 0);
    double* p = stage_out(c, P, mem, 1);
    COMBO_CK(cudaMemsetAsync(c->dstats.p, 0, sizeof(Stats), c->stream));
    Shift9 z{};
    dfmg_sweep(c, f, z, 0.0, p, 0);
    fetch_results(c);
    finish_out(c, P, p, mem);
    if (st) {
      const Stats* s = reinterpret_cast<const Stats*>(c->hres + 64);
      st->inadmissible_cells = int64_t(s->inadmissible);
      st->laminate_failures = int64_t(s->failures);
      st->back_projections = int64_t(s->backproj);
      st->laminate_iter_max = int64_t(s->iter_max);
    }
  });
}

// dfmg_tangent_pass at F (from the current warm starts) + dfmg_tangent_matvec
int combo_dfmg_tangent_matvec(combo_ctx* c, const double* F, const double* x, double* y, int mem) {
  return guarded(c, [&] {
    if (!c->bound) throw ComboError(COMBO_ERR_STATE, "materials not bound (combo_bind_materials)");
    require_single(c);
    ensure_scratch(c);
    const double* f = stage_in(c, F, mem, 0);
    const double* xx = stage_in(c, x, mem, 1);
    double* yy = stage_out(c, y, mem, 2);
    c->scratch[3].alloc(size_t(9 * c->N));
    Shift9 z{};
    COMBO_CK(cudaMemsetAsync(c->dstats.p, 0, sizeof(Stats), c->stream));
    dfmg_tangent_prepare(c, f, z);
    dfmg_matvec(c, f, z, xx, c->scratch[3].p, 0.0, true, yy);
    finish_out(c, y, yy, mem);
  });
}

int combo_dfmg_get_warm_starts(combo_ctx* c, double* warm3, int mem) {
  return guarded(c, [&] {
    if (!c->bound) throw ComboError(COMBO_ERR_STATE, "materials not bound (combo_bind_materials)");
    require_single(c);
    ensure_dfmg(c);
    const int64_t nw = 8 * c->ncomp;
    if (!nw) return;
    std::vector<double> soa(size_t(3 * nw)), aos(size_t(3 * nw));
    COMBO_CK(cudaMemcpy(soa.data(), c->dfmg_warm.p, soa.size() * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < nw; ++i)
      for (int d = 0; d < 3; ++d) aos[size_t(3 * i + d)] = soa[size_t(d * nw + i)];
    if (mem == COMBO_MEM_DEVICE)
      COMBO_CK(cudaMemcpy(warm3, aos.data(), aos.size() * 8, cudaMemcpyHostToDevice));
    else
      std::memcpy(warm3, aos.data(), aos.size() * 8);
  });
}

}  // extern "C"
