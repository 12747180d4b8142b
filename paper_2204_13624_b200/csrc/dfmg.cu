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

// a slab of ni planes (the whole grid: ni = n1)
struct Dims3 {
  int64_t n1, n2, n3;  // n1: this slab's planes
  __device__ __forceinline__ int64_t jk(int64_t j, int64_t k) const {
    j %= n2;
    k %= n3;
    if (j < 0) j += n2;
    if (k < 0) k += n3;
    return j * n3 + k;
  }
};

// One axis-0 neighbour plane of a field (DFMG needs a
// one-plane halo, gather_dfc reads i + 1, the stress assembly i - 1,
// dfmg.cpp:27-47, 148-156): component q of that plane at p[q * stride + jk].
// A single slab points it at its own plane 0 (upper) or n1 - 1 (lower) with
// stride N, which is the reference's periodic wrap.
struct Halo {
  const double* p;
  int64_t stride;
};

// component q of a [.][N] field at local plane i in [-1, n1] (the planes
// -1 and n1 come from the halo h)
__device__ __forceinline__ double fld(const double* __restrict__ f, const Halo& h, int64_t N, const Dims3& d, int q,
                                      int64_t i, int64_t j, int64_t k) {
  const int64_t jk = d.jk(j, k);
  if (i < 0 || i >= d.n1) return h.p[q * h.stride + jk];
  return f[q * N + i * d.n2 * d.n3 + jk];
}

// gather_dfc (dfmg.cpp:27-47); fh: the plane above the slab
__device__ __forceinline__ void gather_dfc(const double* __restrict__ f, const Halo& fh, const Shift9& sh, int64_t N,
                                           const Dims3& d, int64_t i, int64_t j, int64_t k, int code, double* m) {
  const int s1 = code & 1, s2 = (code >> 1) & 1, s3 = (code >> 2) & 1;
  m[0] = fld(f, fh, N, d, 0, i, j, k) + sh.v[0];
  m[4] = fld(f, fh, N, d, 4, i, j, k) + sh.v[4];
  m[8] = fld(f, fh, N, d, 8, i, j, k) + sh.v[8];
  m[1] = fld(f, fh, N, d, 1, i + s1, j + s2, k) + sh.v[1];
  m[3] = fld(f, fh, N, d, 3, i + s1, j + s2, k) + sh.v[3];
  m[2] = fld(f, fh, N, d, 2, i + s1, j, k + s3) + sh.v[2];
  m[6] = fld(f, fh, N, d, 6, i + s1, j, k + s3) + sh.v[6];
  m[5] = fld(f, fh, N, d, 5, i, j + s2, k + s3) + sh.v[5];
  m[7] = fld(f, fh, N, d, 7, i, j + s2, k + s3) + sh.v[7];
}

// mode 0: stress sweep (dfmg_stress); mode 1: tangent pass re-solve
// (dfmg_tangent_pass) -- warm starts read from the pre-launch state and
// written back per dfc (each dfc has exactly one writer).
static __global__ void __launch_bounds__(256) k_dfmg_eval(MatParams M, CellData cd, const double* __restrict__ fin,
                                                          Halo fh, Shift9 sh, Dims3 d, double* __restrict__ warm8,
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
    gather_dfc(fin, fh, sh, N, d, i, j, k, code, f);
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
// P - alpha F. ph: the plane below the slab of pd [9][8]. With partials:
// chunked (plane-aligned) P sums -> partials[chunk] (P-bar, decomposition
// invariant like every other reduction).
static __global__ void __launch_bounds__(256) k_dfmg_gather(const double* __restrict__ pd, Halo ph, Dims3 d,
                                                            const double* __restrict__ fin, Shift9 sh, double alpha,
                                                            double* __restrict__ out, Chunks ch, double* partials) {
  const int64_t N = d.n1 * d.n2 * d.n3;
  double acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0.0;
  int64_t beg, end;
  chunk_range(ch, beg, end);
  for (int64_t cell = beg + threadIdx.x; cell < end; cell += blockDim.x) {
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
        s += fld(pd, ph, N, d, c * 8 + code, hi, hj, hk);
      }
      const double p = s / 8.0;
      acc[c] += p;
      out[c * N + cell] = alpha != 0.0 ? p + (-alpha) * (fin[c * N + cell] + sh.v[c]) : p;
    }
  }
  if (partials) block_reduce_store<9>(acc, partials, blockIdx.x);
}

// per-dfc packed tangents of composite hosts: t8[t][id*8+code]
static __global__ void __launch_bounds__(128) k_dfmg_comp_tangent(MatParams M, CellData cd,
                                                                  const double* __restrict__ fin, Halo fh, Shift9 sh,
                                                                  Dims3 d, const double* __restrict__ warm8,
                                                                  double* __restrict__ t8) {
  const int64_t N = d.n1 * d.n2 * d.n3;
  const int64_t nw = 8 * cd.ncomp;
  for (int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < nw; w += int64_t(gridDim.x) * blockDim.x) {
    const int64_t id = w / 8;
    const int code = int(w - id * 8);
    const int64_t cell = cd.ccell[id];
    const int64_t k = cell % d.n3, j = (cell / d.n3) % d.n2, i = cell / (d.n2 * d.n3);
    double f[9];
    gather_dfc(fin, fh, sh, N, d, i, j, k, code, f);
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
                                                           Halo fh, Shift9 sh, Dims3 d, const double* __restrict__ x,
                                                           Halo xh, const double* __restrict__ t8,
                                                           double* __restrict__ yd) {
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
    gather_dfc(x, xh, zero, N, d, i, j, k, code, xv);
    const int32_t id = cd.cid[cell];
    if (id >= 0) {
      packed45_apply(t8 + int64_t(id) * 8 + code, nw, xv, y);
    } else {
      double f[9], p[9];
      gather_dfc(fin, fh, sh, N, d, i, j, k, code, f);
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

Dims3 dims3(const combo_ctx* c) { return Dims3{c->N / (c->dims[1] * c->dims[2]), c->dims[1], c->dims[2]}; }

void ensure_dfmg(combo_ctx* c) {
  const size_t nw = size_t(8 * std::max<int64_t>(c->ncomp, 1));
  if (c->dfmg_warm.n != 3 * nw) {
    c->dfmg_warm.alloc(3 * nw);
    COMBO_CK(cudaMemsetAsync(c->dfmg_warm.p, 0, 3 * nw * 8, c->stream));
  }
  c->dfmg_pd.alloc(size_t(72 * c->N));
}

int grid8(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

// Halo exchange along axis 0 (ranks in slab order, periodic): `up` fills
// every rank's buffer with plane 0 of the next rank's field (the plane
// above its slab), else with the last plane of the previous rank's (below).
// fields[k] / bufs[k]: rank k of the group (one per process with NCCL).
// A single slab needs no exchange (the halo points into its own field).
std::vector<Halo> halo_exchange(combo_ctx* L, const std::vector<const double*>& fields, int ncomp, bool up,
                                int which) {
  const auto ms = combo_host::members(L);
  const int64_t plane = L->dims[1] * L->dims[2];
  const int64_t N = L->N;
  const int64_t ni = N / plane;
  std::vector<Halo> h(ms.size());
  if (L->R == 1) {
    h[0] = Halo{fields[0] + (up ? 0 : (ni - 1) * plane), N};
    return h;
  }
  for (size_t k = 0; k < ms.size(); ++k) ms[k]->halo[which].alloc(size_t(ncomp * plane));
  ProfScope ps(L, kTagExchange, double(L->R) * double(ncomp) * double(plane) * 16.0);
  if (L->nccl) {
    // pack my boundary plane, send it to the neighbour that needs it
    combo_ctx* c = ms[0];
    c->halo_send.alloc(size_t(ncomp * plane));
    const double* src = fields[0] + (up ? 0 : (ni - 1) * plane);
    COMBO_CK(cudaMemcpy2DAsync(c->halo_send.p, size_t(plane) * 8, src, size_t(N) * 8, size_t(plane) * 8,
                               size_t(ncomp), cudaMemcpyDeviceToDevice, c->stream));
    const int to = up ? (c->q + c->R - 1) % c->R : (c->q + 1) % c->R;
    const int from = up ? (c->q + 1) % c->R : (c->q + c->R - 1) % c->R;
    combo_host::nccl_sendrecv(c, c->halo_send.p, to, c->halo[which].p, from, size_t(ncomp * plane));
  } else {
    const int R = int(ms.size());
    for (int q = 0; q < R; ++q) {
      const int from = up ? (q + 1) % R : (q + R - 1) % R;
      const double* src = fields[size_t(from)] + (up ? 0 : (ni - 1) * plane);
      COMBO_CK(cudaMemcpy2DAsync(ms[size_t(q)]->halo[which].p, size_t(plane) * 8, src, size_t(N) * 8,
                                 size_t(plane) * 8, size_t(ncomp), cudaMemcpyDeviceToDevice, L->stream));
    }
  }
  for (size_t k = 0; k < ms.size(); ++k) h[k] = Halo{ms[k]->halo[which].p, plane};
  return h;
}

}  // namespace

namespace combo_host {

// dfmg_stress (dfmg.cpp:128-176) over every rank hosted by the leader c:
// out = P - alpha F, P sums -> slot
void dfmg_sweep(combo_ctx* c, const std::vector<const double*>& fin, const Shift9& sh, double alpha,
                const std::vector<double*>& out, int slot) {
  const auto ms = members(c);
  const auto fh = halo_exchange(c, fin, 9, true, 0);
  for (size_t k = 0; k < ms.size(); ++k) {
    combo_ctx* m = ms[k];
    ensure_dfmg(m);
    ProfScope ps(m, kTagSweep, 8.0 * 72.0 * double(m->N) * 2.0 + 8.0 * 112.0 * double(m->ncomp));
    k_dfmg_eval<<<grid8(8 * m->N), 256, 0, m->stream>>>(m->mp, m->cell_data(), fin[k], fh[k], sh, dims3(m),
                                                        m->dfmg_warm.p, m->dfmg_pd.p, 0, stats_ptr(m));
    ++m->launches;
    COMBO_CK(cudaGetLastError());
  }
  std::vector<const double*> pds;
  for (auto* m : ms) pds.push_back(m->dfmg_pd.p);
  const auto ph = halo_exchange(c, pds, 72, false, 1);
  const int64_t nb = chunk_blocks(c);
  for (size_t k = 0; k < ms.size(); ++k) {
    combo_ctx* m = ms[k];
    double* part = part_ptr(m, nb, 9);
    ProfScope ps(m, kTagSweep, 8.0 * 72.0 * double(m->N) + 144.0 * double(m->N));
    k_dfmg_gather<<<unsigned(nb), kEwThreads, 0, m->stream>>>(m->dfmg_pd.p, ph[k], dims3(m), fin[k], sh, alpha,
                                                              out[k], chunks_of(m), part);
    ++m->launches;
    COMBO_CK(cudaGetLastError());
  }
  group_reduce(c, nb, 9, slot);
}

// dfmg_tangent_pass (dfmg.cpp:178-207): re-solve from the current warm
// starts, then per-dfc packed tangents of the composite hosts.
void dfmg_tangent_prepare(combo_ctx* c, const std::vector<const double*>& fin, const Shift9& sh) {
  const auto ms = members(c);
  const auto fh = halo_exchange(c, fin, 9, true, 0);
  for (size_t k = 0; k < ms.size(); ++k) {
    combo_ctx* m = ms[k];
    ensure_dfmg(m);
    {
      ProfScope ps(m, kTagOther, 8.0 * 72.0 * double(m->N) + 8.0 * 112.0 * double(m->ncomp));
      k_dfmg_eval<<<grid8(8 * m->N), 256, 0, m->stream>>>(m->mp, m->cell_data(), fin[k], fh[k], sh, dims3(m),
                                                          m->dfmg_warm.p, nullptr, 1, stats_ptr(m));
      ++m->launches;
      COMBO_CK(cudaGetLastError());
    }
    if (m->ncomp) {
      m->dfmg_t8.alloc(size_t(45 * 8 * m->ncomp));
      ProfScope ps(m, kTagOther, 8.0 * double(m->ncomp) * (72.0 + 64.0 + 360.0));
      k_dfmg_comp_tangent<<<unsigned(std::min<int64_t>((8 * m->ncomp + 127) / 128, 148 * 32)), 128, 0,
                            m->stream>>>(m->mp, m->cell_data(), fin[k], fh[k], sh, dims3(m), m->dfmg_warm.p,
                                         m->dfmg_t8.p);
      ++m->launches;
      COMBO_CK(cudaGetLastError());
    }
  }
}

// q = d dfmg_stress / dF [pdir] with pdir = first ? r : r + beta pdir
// (dfmg_tangent_matvec, dfmg.cpp:209-253)
void dfmg_matvec(combo_ctx* c, const std::vector<const double*>& fin, const Shift9& sh,
                 const std::vector<const double*>& r, const std::vector<double*>& pdir, double beta, bool first,
                 const std::vector<double*>& q) {
  const auto ms = members(c);
  for (size_t k = 0; k < ms.size(); ++k) {
    combo_ctx* m = ms[k];
    ProfScope ps(m, kTagMatvec, (first ? 144.0 : 216.0) * double(m->N));
    k_pdir<<<ew_grid(9 * m->N), kEwThreads, 0, m->stream>>>(r[k], pdir[k], beta, first ? 1 : 0, 9 * m->N);
    ++m->launches;
  }
  const auto fh = halo_exchange(c, fin, 9, true, 0);
  const auto xh = halo_exchange(c, std::vector<const double*>(pdir.begin(), pdir.end()), 9, true, 2);
  for (size_t k = 0; k < ms.size(); ++k) {
    combo_ctx* m = ms[k];
    ensure_dfmg(m);
    ProfScope ps(m, kTagMatvec, 8.0 * 72.0 * double(m->N) * 3.0 + 8.0 * 360.0 * double(m->ncomp));
    k_dfmg_apply<<<grid8(8 * m->N), 256, 0, m->stream>>>(m->mp, m->cell_data(), fin[k], fh[k], sh, dims3(m),
                                                          pdir[k], xh[k], m->dfmg_t8.p, m->dfmg_pd.p);
    ++m->launches;
  }
  std::vector<const double*> pds;
  for (auto* m : ms) pds.push_back(m->dfmg_pd.p);
  const auto ph = halo_exchange(c, pds, 72, false, 1);
  for (size_t k = 0; k < ms.size(); ++k) {
    combo_ctx* m = ms[k];
    ProfScope ps(m, kTagMatvec, 8.0 * 72.0 * double(m->N) + 72.0 * double(m->N));
    Shift9 z{};
    k_dfmg_gather<<<unsigned(chunk_blocks(m)), kEwThreads, 0, m->stream>>>(m->dfmg_pd.p, ph[k], dims3(m), fin[k], z,
                                                                         0.0, q[k], chunks_of(m), nullptr);
    ++m->launches;
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
    dfmg_sweep(c, {f}, z, 0.0, {p}, 0);
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
    dfmg_tangent_prepare(c, {f}, z);
    dfmg_matvec(c, {f}, z, {xx}, {c->scratch[3].p}, 0.0, true, {yy});
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
