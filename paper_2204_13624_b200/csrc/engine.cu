// B200 ComBo engine: FFT/Gamma plans, fused projection pipeline, stress /
// tangent sweeps and the Lippmann-Schwinger solver driver (basic fixed point
// and Newton-CG with line search and load-step bisection).
//
// Host control flow restates /root/reference/proj/src/solver.cpp:124-346
// line by line; every field-sized operation is a kernel of this library and
// only scalars (sums, stats) cross PCIe per iteration.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <thread>
#include <type_traits>

#include "context.hpp"
#include "fft_tma.cuh"

using namespace combo_dev;

namespace combo_host {

// ------------------------------------------------------------------ plans
namespace {
constexpr long double kPiL = 3.141592653589793238462643383279502884L;
constexpr double kPi = 3.141592653589793238462643383279502884;

std::vector<int> factor_radices(int n) {
  std::vector<int> r;
  int m = n;
  while (m % 8 == 0) {
    r.push_back(8);
    m /= 8;
  }
  while (m % 4 == 0) {
    r.push_back(4);
    m /= 4;
  }
  while (m % 2 == 0) {
    r.push_back(2);
    m /= 2;
  }
  for (int p = 3; m > 1; p += 2)
    while (m % p == 0) {
      if (p > 61) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "FFT: prime factor > 61 unsupported");
      r.push_back(p);
      m /= p;
    }
  if (r.size() > size_t(kMaxRad)) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "FFT: too many radix stages");
  return r;
}

void build_axis(AxisPlan& a, int n) {
  a.n = n;
  a.rad = factor_radices(n);
  std::vector<double2> tw(size_t(std::max(n, 1)));
  for (int k = 0; k < n; ++k) {
    const long double ph = -2.0L * kPiL * (long double)k / (long double)n;
    tw[size_t(k)] = make_double2(double(cosl(ph)), double(sinl(ph)));
  }
  a.tw.alloc(tw.size());
  COMBO_CK(cudaMemcpy(a.tw.p, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
}

// one radix-8 butterfly (8 complex values) per thread per stage
int pick_threads(int64_t tile) {
  const int64_t t = ((tile + kElems - 1) / kElems + 31) / 32 * 32;
  if (t > kMaxFftThreads) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "FFT tile too large");
  return int(std::max<int64_t>(t, 32));
}

// green.cpp:16-57 (identical double arithmetic to the reference)
void build_green(GreenPlan& g, int kind, const std::array<int64_t, 3>& dims,
                 const std::array<double, 3>& lengths) {
  g.kind = kind;
  for (int a = 0; a < 3; ++a) {
    const int64_t n = dims[a];
    const double h = lengths[a] / double(n);
    const double l = lengths[a];
    std::vector<double2> fwd(static_cast<size_t>(n)), avg(static_cast<size_t>(n));
    std::vector<double> xi(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
      const size_t sk = size_t(k);
      if (k == 0) {
        fwd[sk] = make_double2(0.0, 0.0);
        avg[sk] = make_double2(1.0, 0.0);
        xi[sk] = 0.0;
        continue;
      }
      if (2 * k == n) {
        fwd[sk] = make_double2(-2.0 / h, 0.0);
        avg[sk] = make_double2(0.0, 0.0);
        xi[sk] = 2.0 * kPi * double(k) / l;
        continue;
      }
      const double phi = 2.0 * kPi * double(k) / double(n);
      const double c = std::cos(phi), s = std::sin(phi);
      fwd[sk] = make_double2((c - 1.0) / h, s / h);
      avg[sk] = make_double2(0.5 * (c + 1.0), 0.5 * s);
      const int64_t ks = 2 * k < n ? k : k - n;
      xi[sk] = 2.0 * kPi * double(ks) / l;
    }
    g.fwd[a].alloc(size_t(n));
    g.avg[a].alloc(size_t(n));
    g.xi[a].alloc(size_t(n));
    COMBO_CK(cudaMemcpy(g.fwd[a].p, fwd.data(), size_t(n) * sizeof(double2), cudaMemcpyHostToDevice));
    COMBO_CK(cudaMemcpy(g.avg[a].p, avg.data(), size_t(n) * sizeof(double2), cudaMemcpyHostToDevice));
    COMBO_CK(cudaMemcpy(g.xi[a].p, xi.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice));
  }
}

GreenTables green_view(const GreenPlan& g) {
  GreenTables t;
  t.kind = g.kind;
  for (int a = 0; a < 3; ++a) {
    t.fwd[a] = g.fwd[a].p;
    t.avg[a] = g.avg[a].p;
    t.xi[a] = g.xi[a].p;
  }
  return t;
}
}  // namespace

int ew_grid(int64_t n) {
  const int64_t b = (n + kEwThreads - 1) / kEwThreads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

void ensure_scratch(combo_ctx* c) {
  if (!c->dres.p) {
    c->dres.alloc(64);
    c->dstats.alloc(1);
    COMBO_CK(cudaMallocHost(&c->hres, 64 * sizeof(double) + sizeof(Stats)));
  }
}

// 4-D tensor map over the single-slab spectrum for the TMA-staged strip
// passes (fft_tma.cuh): coordinates (column in doubles, row index with the
// smaller stride, the other row index, component); the box spans W columns
// and up to 256 rows of the transformed index.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    COMBO_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      throw ComboError(COMBO_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// returns lineFirst (the transformed index is coordinate 1)
int encode_strip_map(CUtensorMap* m, const FftPlan& p, bool xpass, int W) {
  const combo_dev::SpecView sv = p.sv();
  const bool i_first = sv.si < sv.sj;
  const int64_t n1 = p.dims[0], n2 = p.dims[1];
  const cuuint64_t gdim[4] = {cuuint64_t(2 * p.n3p), cuuint64_t(i_first ? n1 : n2), cuuint64_t(i_first ? n2 : n1), 9};
  const cuuint64_t gstr[3] = {cuuint64_t(16 * std::min(sv.si, sv.sj)), cuuint64_t(16 * std::max(sv.si, sv.sj)),
                              cuuint64_t(16 * sv.cs)};
  const bool line_first = xpass == i_first;
  const int64_t n = xpass ? n1 : n2;
  const cuuint32_t rb = cuuint32_t(std::min<int64_t>(n, 256));
  const cuuint32_t box[4] = {cuuint32_t(2 * W), line_first ? rb : 1u, line_first ? 1u : rb, xpass ? 3u : 1u};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = encode_tiled_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, p.spec.p, gdim, gstr, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       // 256-byte L2 promotion: y pass 3.674 -> 3.632 ms, nothing for the
                                       // 64-byte rows of the x pass (profiles/r2x_*)
                                       xpass ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw ComboError(COMBO_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return line_first ? 1 : 0;
}

bool pow2_between(int64_t n, int lo, int hi) {
  for (int l = lo; l <= hi; ++l)
    if (n == (int64_t(1) << l)) return true;
  return false;
}

void set_grid(combo_ctx* c, const int64_t* dims, const double* lengths) {
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 1) throw ComboError(COMBO_ERR_BAD_SHAPE, "grid dims must be >= 1");
    if (!(lengths[a] > 0.0)) throw ComboError(COMBO_ERR_BAD_SHAPE, "grid lengths must be positive");
  }
  const std::array<int64_t, 3> d{dims[0], dims[1], dims[2]};
  const std::array<double, 3> l{lengths[0], lengths[1], lengths[2]};
  const int R = c->R;
  if (R > 1 && (d[0] % R != 0 || d[1] % R != 0))
    throw ComboError(COMBO_ERR_BAD_SHAPE, "slab decomposition: the rank count must divide n1 and n2");
  c->has_grid = true;
  c->dims = d;
  c->lengths = l;
  c->Ng = d[0] * d[1] * d[2];
  c->N = (d[0] / R) * d[1] * d[2];
  if (c->plan && c->plan->dims == d && c->plan->lengths == l && c->plan->R == R && c->plan->q == c->q) return;
  auto p = std::make_unique<FftPlan>();
  p->dims = d;
  p->lengths = l;
  p->R = R;
  p->q = c->q;
  p->ni = d[0] / R;
  p->nj = d[1] / R;
  p->i0 = c->q * p->ni;
  p->j0 = c->q * p->nj;
  // z-line blocks never straddle a plane (decomposition-invariant partials)
  auto divisor_le = [&](int64_t L) {
    L = std::max<int64_t>(1, std::min(L, d[1]));
    while (d[1] % L != 0) --L;
    return L;
  };
  for (int a = 0; a < 3; ++a) build_axis(p->ax[a], int(d[a]));
  p->n3c = d[2] / 2 + 1;
  p->n3p = (p->n3c + 7) / 8 * 8;
  // z pass: L z-lines per block (~1024 cells), pairs of real lines packed
  const int64_t n3 = d[2];
  int64_t L = std::max<int64_t>(1, 1024 / n3);
  while (L > 1 && ((9 * L + 1) / 2) * n3 > 6144) --L;
  L = divisor_le(L);
  p->zL = int(L);
  p->zls = int(n3);
  const int64_t npair = (9 * L + 1) / 2;
  p->zT = pick_threads(npair * n3);
  p->zsmem = size_t(npair * n3) * sizeof(double2);
  // y pass
  int W = int(std::min<int64_t>(8, p->n3c));
  while (W > 1 && d[1] * W > 6144) W /= 2;
  p->yW = W;
  p->yT = pick_threads(d[1] * W);
  p->ysmem = size_t(d[1] * W) * sizeof(double2);
  // x pass + Gamma (3 components per tile)
  W = int(std::min<int64_t>(8, p->n3c));
  while (W > 1 && 3 * d[0] * W > 6144) W /= 2;
  p->xW = W;
  p->xT = pick_threads(3 * d[0] * W);
  p->xsmem = size_t(3 * d[0] * W) * sizeof(double2);
  // tuning knobs (benchmarks): COMBO_ZLINES / COMBO_YW / COMBO_XW the tile
  // shapes, COMBO_XMINB the x+Gamma residency
  auto knob = [](const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
  };
  p->xminb = knob("COMBO_XMINB", 2);
  p->pq_dot = knob("COMBO_PQ", 1) != 0;
  p->zring = knob("COMBO_ZRING", 2);
  p->mv_bulk = knob("COMBO_MV_BULK", 1) != 0;
  p->split_sweep = knob("COMBO_SPLIT_SWEEP", 1) != 0;
  // register-resident geometry (pow2 axes >= 8): T = lines * N/8
  if (n3 >= 8) {
    const int64_t tl = n3 / 8;
    auto lines_for = [&](int64_t tmax) {
      int64_t Lz = 1;
      while (((9 * (Lz + 1) + 1) / 2) * tl <= tmax && ((9 * (Lz + 1) + 1) / 2) * n3 * 18 <= 100 * 1024) ++Lz;
      return Lz;
    };
    int64_t Lz = lines_for(512);
    if (knob("COMBO_ZLINES", 0) > 0) Lz = std::min<int64_t>(knob("COMBO_ZLINES", 0), combo_dev::kMaxZRows / 9);
    Lz = divisor_le(Lz);
    p->rzL = int(Lz);
    const int64_t np = (9 * Lz + 1) / 2;
    p->rzT = int((np * tl + 31) / 32 * 32);
    p->rzsmem = size_t(np * (n3 + n3 / 8)) * sizeof(double2);
  }
  // j-major rows (single slab): x+Gamma 5.9 ms, y 4.05 / 4.09 ms; i-major: 6.8, 4.01 / 4.03 (512^3, round 1)
  p->swap = knob("COMBO_SWAP", 1) != 0;
  if (d[1] >= 8) {
    int Wy = int(std::min<int64_t>(8, p->n3c));
    // i-major rows: 256-thread tiles measured faster than 512 at n2 = 512
    // (4.5 vs 4.8 ms); j-major rows: y lines take the long stride and want
    // 128-byte row segments (W = 8)
    while (Wy > 1 && Wy * (d[1] / 8) > (p->swap ? 512 : 256)) Wy /= 2;
    if (knob("COMBO_YW", 0) > 0) Wy = knob("COMBO_YW", 0);
    p->ryW = Wy;
    p->ryT = int(std::max<int64_t>(32, (Wy * (d[1] / 8) + 31) / 32 * 32));
    p->rysmem = size_t((d[1] + d[1] / 8) * Wy) * sizeof(double2);
  }
  if (d[0] >= 8) {
    int Wx = int(std::min<int64_t>(8, p->n3c));
    while (Wx > 1 && Wx * (d[0] / 8) > 256) Wx /= 2;
    if (knob("COMBO_XW", 0) > 0) Wx = knob("COMBO_XW", 0);
    p->rxW = Wx;
    p->rxT = int(std::max<int64_t>(32, (Wx * (d[0] / 8) + 31) / 32 * 32));
    p->rxsmem = size_t(2 * (d[0] + d[0] / 8) * Wx) * sizeof(double2);
  }
  p->spec.alloc(size_t(9 * p->ni * d[1] * p->n3p));
  if (R > 1) {
    p->specB.alloc(size_t(9 * p->ni * d[1] * p->n3p));
  }
  // TMA-staged strip passes: single slab, lines of 64..1024 points
  if (R == 1 && p->n3c >= 8) {
    if (knob("COMBO_XTMA", 1) != 0 && pow2_between(d[0], 6, 10)) {
      p->tma_x_line_first = encode_strip_map(&p->xmap, *p, true, combo_dev::kTmaW);
      p->tma_x = true;
    }
    if (knob("COMBO_YTMA", 1) != 0 && pow2_between(d[1], 6, 10)) {
      p->tma_yw = d[1] >= 1024 ? 4 : 8;
      if (d[1] < 1024 && (knob("COMBO_YTMA_W", 0) == 4 || knob("COMBO_YTMA_W", 0) == 8))
        p->tma_yw = knob("COMBO_YTMA_W", 0);
      p->tma_y_line_first = encode_strip_map(&p->ymap, *p, false, p->tma_yw);
      p->tma_y = true;
    }
  }
  c->plan = std::move(p);
}

GreenPlan& green_plan(combo_ctx* c, int kind) {
  if (kind < 0 || kind > 2) throw ComboError(COMBO_ERR_CONFIG_INVALID, "unknown Green operator kind");
  GreenPlan& g = c->plan->green[kind];
  if (g.kind != kind) build_green(g, kind, c->plan->dims, c->plan->lengths);
  return g;
}

void reduce_partials(combo_ctx* c, int64_t nblocks, int nred, int slot) {
  ProfScope ps(c, kTagReduce, double(nblocks) * nred * 8.0);
  k_reduce_partials<<<nred, 1024, 0, c->stream>>>(c->partials.p, nblocks, nred, c->dres.p + slot);
  ++c->launches;
  COMBO_CK(cudaGetLastError());
}

void fetch_results(combo_ctx* c, bool with_stats) {
  const Stats* st = c->dstats.p;
  if (with_stats && c->nccl && c->R > 1) {
    // laminate statistics of all ranks: sums and the maximum iteration count
    c->gstats.alloc(1);
    nccl_allreduce_u64(c, reinterpret_cast<const unsigned long long*>(c->dstats.p),
                       reinterpret_cast<unsigned long long*>(c->gstats.p), 3, false);
    nccl_allreduce_u64(c, &c->dstats.p->iter_max, &c->gstats.p->iter_max, 1, true);
    st = c->gstats.p;
  }
  COMBO_CK(cudaMemcpyAsync(c->hres, c->dres.p, 64 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaMemcpyAsync(c->hres + 64, st, sizeof(Stats), cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaStreamSynchronize(c->stream));
}

void ensure_partials(combo_ctx* c, int64_t count) {
  if (c->partials.n < size_t(count)) c->partials.alloc(size_t(count));
}

// ------------------------------------------------- slab decomposition
combo_ctx* leader(combo_ctx* c) { return c->lead ? c->lead : c; }

std::vector<combo_ctx*> members(combo_ctx* c) {
  std::vector<combo_ctx*> v{c};
  for (auto& m : c->vm) v.push_back(m.get());
  return v;
}

// Block partials of rank q for a launch of nb blocks x nred values per rank:
// [global block][nred] in the leader's buffer (all ranks' blocks, rank order)
double* part_ptr(combo_ctx* c, int64_t nb, int nred) {
  combo_ctx* L = leader(c);
  const size_t need = size_t(c->R) * size_t(nb) * size_t(nred);
  if (L->gpart.n < need) L->gpart.alloc(need);
  return L->gpart.p + size_t(c->q) * size_t(nb) * size_t(nred);
}

Stats* stats_ptr(combo_ctx* c) { return leader(c)->dstats.p; }

// fixed-order combination of every rank's block partials -> dres[slot..]
void group_reduce(combo_ctx* c, int64_t nb, int nred, int slot) {
  combo_ctx* L = leader(c);
  const int64_t total = int64_t(L->R) * nb;
  constexpr int kChunkRed = 4096;
  const bool two_level = total > (int64_t(1) << 20);
  // long vectors (the matvec's per-warp sums): sums over fixed chunks of the
  // global block order first. Chunks that do not straddle ranks are summed
  // by their owner, so only the chunk sums cross NVLink.
  const bool local_chunks = two_level && nb % kChunkRed == 0;
  if (L->nccl && L->R > 1 && !local_chunks) nccl_allgather_inplace(L, L->gpart.p, size_t(nb) * size_t(nred));
  ProfScope ps(L, kTagReduce, double(L->R) * double(nb) * nred * 8.0);
  if (two_level) {
    const int64_t nch = (total + kChunkRed - 1) / kChunkRed;
    if (L->gpart2.n < size_t(nch * nred)) L->gpart2.alloc(size_t(nch * nred));
    if (L->nccl && L->R > 1 && local_chunks) {
      const int64_t nloc = nb / kChunkRed;
      k_reduce_chunks<<<unsigned(nloc), 256, 0, L->stream>>>(L->gpart.p + size_t(L->q) * size_t(nb) * nred, nb, nred,
                                                            kChunkRed, L->gpart2.p + size_t(L->q) * size_t(nloc) * nred);
      nccl_allgather_inplace(L, L->gpart2.p, size_t(nloc) * size_t(nred));
    } else {
      k_reduce_chunks<<<unsigned(nch), 256, 0, L->stream>>>(L->gpart.p, total, nred, kChunkRed, L->gpart2.p);
    }
    k_reduce_partials<<<nred, 1024, 0, L->stream>>>(L->gpart2.p, nch, nred, L->dres.p + slot);
    ++L->launches;
  } else {
    k_reduce_partials<<<nred, 1024, 0, L->stream>>>(L->gpart.p, total, nred, L->dres.p + slot);
  }
  ++L->launches;
  COMBO_CK(cudaGetLastError());
}

// chunked launches (decomposition-invariant partials, kernels.cuh)
Chunks chunks_of(const combo_ctx* c) {
  Chunks k;
  k.plane = c->dims[1] * c->dims[2];
  k.cpp = int((k.plane + kChunk - 1) / kChunk);
  return k;
}
int64_t chunk_blocks(const combo_ctx* c) { return (c->N / (c->dims[1] * c->dims[2])) * chunks_of(c).cpp; }

// slab <-> pencil transpose of the spectrum (SpecView): block s of rank q's
// slab side is block q of rank s's pencil side
// g >= 0: only the components of Gamma row group g (3 g .. 3 g + 2), on
// `stream` (default: the compute stream)
void exchange(combo_ctx* c, bool to_pencil, int g = -1, cudaStream_t stream = nullptr) {
  combo_ctx* L = leader(c);
  if (L->R == 1) return;
  if (!stream) stream = L->stream;
  const FftPlan& p0 = *L->plan;
  const size_t cs = size_t(p0.ni * p0.nj * p0.n3p);
  const size_t blk = 9 * cs;
  const size_t off = g < 0 ? 0 : size_t(3 * g) * cs, cnt = g < 0 ? blk : 3 * cs;
  ProfScope ps(L, kTagExchange, 2.0 * double(L->R - 1) * double(cnt) * 16.0 * (L->nccl ? 1.0 : double(L->R)), stream);
  if (L->nccl) {
    double2* src = to_pencil ? L->plan->spec.p : L->plan->specB.p;
    double2* dst = to_pencil ? L->plan->specB.p : L->plan->spec.p;
    nccl_alltoall_blocks(L, src, dst, blk, off, cnt, stream);
    return;
  }
  auto ms = members(L);
  for (int q = 0; q < L->R; ++q)
    for (int s = 0; s < L->R; ++s) {
      const double2* src = to_pencil ? ms[size_t(q)]->plan->spec.p + size_t(s) * blk
                                     : ms[size_t(s)]->plan->specB.p + size_t(q) * blk;
      double2* dst = to_pencil ? ms[size_t(s)]->plan->specB.p + size_t(q) * blk
                               : ms[size_t(q)]->plan->spec.p + size_t(s) * blk;
      COMBO_CK(cudaMemcpyAsync(dst + off, src + off, cnt * sizeof(double2), cudaMemcpyDeviceToDevice, stream));
    }
}

// ------------------------------------------------------------- profiler
namespace {
cudaEvent_t pool_event(combo_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  COMBO_CK(cudaEventCreate(&e));
  return e;
}
const char* kTagNames[kNumTags] = {"sweep",  "matvec",    "zfwd",      "yfwd",   "xgamma", "yinv",
                                   "zinv",   "cg_update", "trial",     "materialize", "reduce", "other", "matvec_zfwd", "exchange"};
}  // namespace

// emulated ranks record into the leader's profile (they share its stream)
ProfScope::ProfScope(combo_ctx* ctx, int tag, double bytes, cudaStream_t stream)
    : c(ctx->lead ? ctx->lead : ctx), st(stream ? stream : (ctx->lead ? ctx->lead : ctx)->stream) {
  if (!c->prof_on) return;
  combo_ctx::ProfRec r{tag, pool_event(c), pool_event(c), bytes};
  COMBO_CK(cudaEventRecord(r.a, st));
  idx = int(c->prof.size());
  c->prof.push_back(r);
}
ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(c->prof[size_t(idx)].b, st);
}

double spec_bytes(const combo_ctx* c) {
  return 9.0 * double(c->plan->ni * c->plan->dims[1] * c->plan->n3c) * 16.0;
}

// ------------------------------------------------------ launch helpers
// COMBO_CARVEOUT: shared-memory carveout percentage (default: driver's choice)
int carveout_knob() {
  static const int v = [] {
    const char* s = std::getenv("COMBO_CARVEOUT");
    return s ? std::atoi(s) : -1;
  }();
  return v;
}

template <class K>
void smem_attr(K kernel, size_t bytes) {
  // always opt in: static + dynamic above 48 KB needs the attribute too
  if (bytes > 0) COMBO_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  if (bytes > 0 && carveout_knob() >= 0)
    COMBO_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_knob()));
}

// compile-time line length: log2(n) for powers of two <= 1024, else generic
template <class F>
void dispatch_log2(int64_t n, F&& f) {
  int L = -1;
  for (int l = 0; l <= 10; ++l)
    if (n == (int64_t(1) << l)) L = l;
  switch (L) {
    case 0: f(std::integral_constant<int, 0>{}); break;
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 9: f(std::integral_constant<int, 9>{}); break;
    case 10: f(std::integral_constant<int, 10>{}); break;
    default: f(std::integral_constant<int, kGeneric>{}); break;
  }
}

// CG matvec: bulk-staged persistent kernel (one CTA per SM) when the rows
// are 16-byte aligned, else one cell per thread with direct loads.
template <bool FIRST, bool HASX>
void launch_matvec_bulk(combo_ctx* c, const MatvecArgs& a, double* q) {
  using S = combo_dev::MvStage<FIRST, HASX>;
  constexpr int kMaxSmem = 227 * 1024;
  const int stages = std::min(4, (kMaxSmem - combo_dev::kMvHead) / S::kBytes);
  const size_t smem = combo_dev::kMvHead + size_t(stages) * S::kBytes;
  auto kern = combo_dev::k_matvec_bulk<FIRST, HASX>;
  static bool attr = false;  // per instantiation
  if (!attr) {
    COMBO_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const int64_t tiles = std::max<int64_t>(1, a.N / combo_dev::kMvT);
  const int grid = int(std::min<int64_t>(tiles, c->num_sms));
  kern<<<grid, combo_dev::kMvT + 32, smem, c->stream>>>(a, q, stages);
}

bool mv_bulk_ok(const combo_ctx* c, const MatvecArgs& a) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return c->plan && c->plan->mv_bulk && a.N % 2 == 0 && al16(a.r) && al16(a.fin) && al16(a.pdir) &&
         (a.xv == nullptr || al16(a.xv)) && al16(a.cd.cid);
}

void launch_matvec(combo_ctx* c, const MatvecArgs& a, double* q) {
  const bool bulk = mv_bulk_ok(c, a);
  if (!bulk) {
    combo_dev::k_matvec<><<<ew_grid(a.N), kEwThreads, 0, c->stream>>>(a, q);
    return;
  }
  if (a.first)
    launch_matvec_bulk<true, false>(c, a, q);
  else if (a.xv)
    launch_matvec_bulk<false, true>(c, a, q);
  else
    launch_matvec_bulk<false, false>(c, a, q);
}

template <class Prod>
int64_t launch_zfwd(combo_ctx* c, const Prod& prod, double extra_bytes = 0.0) {
  FftPlan& p = *c->plan;
  int64_t nb = 0;
  ProfScope ps(c, kTagZfwd, spec_bytes(c) + 72.0 * double(c->N) * Prod::FIELDS + extra_bytes);
  dispatch_log2(p.dims[2], [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    if constexpr (L >= 3) {
      const int lz = p.rzL;
      nb = (p.ni * p.dims[1] + lz - 1) / lz;
      auto k = zfwd_rr<Prod, L>;
      smem_attr(k, p.rzsmem);
      k<<<unsigned(nb), p.rzT, p.rzsmem, c->stream>>>(p.sv(), p.ax[2].tw.p, lz, prod,
                                                                          nullptr);
    } else {
      nb = (p.ni * p.dims[1] + p.zL - 1) / p.zL;
      double* part = Prod::NRED ? part_ptr(c, nb, Prod::NRED) : nullptr;
      auto k = zfwd_kernel<Prod, L>;
      smem_attr(k, p.zsmem);
      k<<<unsigned(nb), p.zT, p.zsmem, c->stream>>>(p.sv(), p.ax[2].view(), p.zL, p.zls, prod, part);
    }
  });
  ++c->launches;
  COMBO_CK(cudaGetLastError());
  return nb;
}

template <class Cons>
int64_t launch_zinv(combo_ctx* c, const Cons& cons) {
  FftPlan& p = *c->plan;
  int64_t nb = 0;
  const double scale = 1.0 / double(c->Ng);
  ProfScope ps(c, kTagZinv, spec_bytes(c) + 72.0 * double(c->N) * Cons::FIELDS);
  dispatch_log2(p.dims[2], [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    if constexpr (L >= 3) {
      nb = (p.ni * p.dims[1] + p.rzL - 1) / p.rzL;
      double* part = Cons::NRED ? part_ptr(c, nb, Cons::NRED) : nullptr;
      const size_t rows = size_t(9 * p.rzL) * size_t(p.n3p) * sizeof(double2);
      bool ring = false;
      if constexpr (L == 9) {
        // persistent ring-staged kernel: one z-line per tile, two consumer groups
        using Z = combo_dev::ZRing<L>;
        const size_t smem = size_t(Z::kHead + 2 * Z::kWork) + size_t(Z::kStages) * rows;
        if (p.zring >= 2 && p.rzL == 1 && smem <= 227 * 1024 && !Cons::LOADS) {
          auto k = zinv_ring<Cons, L>;
          smem_attr(k, smem);
          const int grid = int(std::min<int64_t>(nb, c->num_sms));
          k<<<grid, Z::kThreads, smem, c->stream>>>(p.sv(), p.ax[2].tw.p, scale, cons, part);
          ring = true;
        }
      }
      if (ring) {
      } else {
        auto k = zinv_rr<Cons, L>;
        smem_attr(k, p.rzsmem);
        k<<<unsigned(nb), p.rzT, p.rzsmem, c->stream>>>(p.sv(), p.ax[2].tw.p, p.rzL, scale, cons, part);
      }
    } else {
      nb = (p.ni * p.dims[1] + p.zL - 1) / p.zL;
      double* part = Cons::NRED ? part_ptr(c, nb, Cons::NRED) : nullptr;
      auto k = zinv_kernel<Cons, L>;
      smem_attr(k, p.zsmem);
      k<<<unsigned(nb), p.zT, p.zsmem, c->stream>>>(p.sv(), p.ax[2].view(), p.zL, p.zls, scale, cons, part);
    }
  });
  ++c->launches;
  COMBO_CK(cudaGetLastError());
  return nb;
}

// components [c0, c0 + ncomp)
template <bool INV>
void launch_y(combo_ctx* c, int ncomp = 9, int c0 = 0) {
  FftPlan& p = *c->plan;
  ProfScope ps(c, INV ? kTagYinv : kTagYfwd, 2.0 * spec_bytes(c) * ncomp / 9.0);
  combo_dev::SpecView svy = p.sv();
  svy.spec += int64_t(c0) * svy.cs;
  dispatch_log2(p.dims[1], [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    if constexpr (L >= 6) {
      if (p.tma_y && c0 == 0) {
        auto go = [&](auto k, int W) {
          const size_t smem = size_t((p.dims[1] + p.dims[1] / 8) * W) * sizeof(double2);
          dim3 grid(unsigned((p.n3c + W - 1) / W), unsigned(p.ni), unsigned(ncomp));
          smem_attr(k, smem);
          k<<<grid, int(p.dims[1] / 8) * W, smem, c->stream>>>(p.ymap, p.sv(), p.ax[1].tw.p, p.tma_y_line_first);
        };
        if (p.tma_yw == 8) {
          if constexpr (L <= 9) go(ypass_tma<L, INV, 8>, 8);
        } else {
          go(ypass_tma<L, INV, 4>, 4);
        }
        return;
      }
    }
    if constexpr (L >= 3) {
      dim3 grid(unsigned((p.n3c + p.ryW - 1) / p.ryW), unsigned(p.ni), unsigned(ncomp));
      auto k = ypass_rr<L, INV>;
      smem_attr(k, p.rysmem);
      k<<<grid, p.ryT, p.rysmem, c->stream>>>(svy, p.ax[1].tw.p, p.ryW);
    } else {
      dim3 grid(unsigned((p.n3c + p.yW - 1) / p.yW), unsigned(p.ni), unsigned(ncomp));
      auto k = ypass_kernel<L, INV>;
      smem_attr(k, p.ysmem);
      k<<<grid, p.yT, p.ysmem, c->stream>>>(svy, p.ax[1].view(), p.yW);
    }
  });
  ++c->launches;
  COMBO_CK(cudaGetLastError());
}

// Gamma row groups [rg0, rg0 + nrg)
void launch_xgamma(combo_ctx* c, int kind, int rg0 = 0, int nrg = 3) {
  const GreenTables g = green_view(green_plan(c, kind));
  FftPlan& p = *c->plan;
  ProfScope ps(c, kTagXGamma, 2.0 * spec_bytes(c) * nrg / 3.0);
  dispatch_log2(p.dims[0], [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    if constexpr (L >= 6) {
      if (p.tma_x && rg0 == 0 && nrg == 3) {
        constexpr int W = combo_dev::kTmaW;
        const size_t smem = size_t(3 * p.dims[0] * W) * sizeof(double2);
        dim3 grid(unsigned((p.n3c + W - 1) / W), unsigned(p.nj), 3u);
        auto go = [&](auto k) {
          smem_attr(k, smem);
          k<<<grid, int(p.dims[0] / 8) * W, smem, c->stream>>>(p.xmap, p.svB(), p.ax[0].tw.p, g, p.tma_x_line_first);
        };
        if (kind == 0)
          go(xgamma_tma<L, 0>);
        else if (kind == 1)
          go(xgamma_tma<L, 1>);
        else
          go(xgamma_tma<L, 2>);
        return;
      }
    }
    if constexpr (L >= 3) {
      // rank-1 x + Gamma (fft_rr.cuh): two channels per thread
      dim3 grid(unsigned((p.n3c + p.rxW - 1) / p.rxW), unsigned(p.nj), unsigned(nrg));
      auto go = [&](auto k) {
        smem_attr(k, p.rxsmem);
        k<<<grid, p.rxT, p.rxsmem, c->stream>>>(p.svB(), p.ax[0].tw.p, p.rxW, g, rg0);
      };
      auto by_kind = [&](auto k0, auto k1, auto k2) {
        if (kind == 0)
          go(k0);
        else if (kind == 1)
          go(k1);
        else
          go(k2);
      };
      if (p.rxT > 256)
        by_kind(xgamma_v4<L, 0, 512, 1>, xgamma_v4<L, 1, 512, 1>, xgamma_v4<L, 2, 512, 1>);
      else if (p.xminb == 3)
        by_kind(xgamma_v4<L, 0, 256, 3>, xgamma_v4<L, 1, 256, 3>, xgamma_v4<L, 2, 256, 3>);
      else
        by_kind(xgamma_v4<L, 0, 256, 2>, xgamma_v4<L, 1, 256, 2>, xgamma_v4<L, 2, 256, 2>);
    } else {
      dim3 grid(unsigned((p.n3c + p.xW - 1) / p.xW), unsigned(p.nj), unsigned(nrg));
      auto k = xgamma_kernel<L>;
      smem_attr(k, p.xsmem);
      k<<<grid, p.xT, p.xsmem, c->stream>>>(p.svB(), p.ax[0].view(), p.xW, g, rg0);
    }
  });
  ++c->launches;
  COMBO_CK(cudaGetLastError());
}
template <bool INV>
void launch_x_plain(combo_ctx* c) {
  FftPlan& p = *c->plan;
  dispatch_log2(p.dims[0], [&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    if constexpr (L >= 3) {
      const size_t smem = size_t((p.dims[0] + p.dims[0] / 8) * p.rxW) * sizeof(double2);
      dim3 grid(unsigned((p.n3c + p.rxW - 1) / p.rxW), unsigned(p.nj), 9u);
      auto k = xpass_rr<L, INV>;
      smem_attr(k, smem);
      k<<<grid, p.rxT, smem, c->stream>>>(p.svB(), p.ax[0].tw.p, p.rxW);
    } else {
      // plain x pass: x tile geometry with a single component per block
      const size_t smem = size_t(p.dims[0] * p.xW) * sizeof(double2);
      dim3 grid(unsigned((p.n3c + p.xW - 1) / p.xW), unsigned(p.nj), 9u);
      auto k = xpass_kernel<L, INV>;
      smem_attr(k, smem);
      k<<<grid, pick_threads(p.dims[0] * p.xW), smem, c->stream>>>(p.svB(), p.ax[0].view(), p.xW);
    }
  });
  ++c->launches;
  COMBO_CK(cudaGetLastError());
}

// COMBO_OVERLAP=0: serial transposes (exchange -> x + Gamma -> exchange)
bool overlap_knob() {
  static const bool v = [] {
    const char* s = std::getenv("COMBO_OVERLAP");
    return s ? std::atoi(s) != 0 : true;
  }();
  return v;
}
void pipe_init(combo_ctx* c) {
  if (c->comm_stream) return;
  COMBO_CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  for (auto& e : c->pipe_ev) COMBO_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// Projection Pi(tau) = alpha Gamma^0 tau (green.cpp:133-151) with fused
// producer / consumer, over every rank hosted by the leader c: prodf(k) /
// consf(k) build member k's producer and consumer. z and y passes run on
// the slabs, the spectrum is transposed to pencils for the x pass + Gamma
// and back; the consumer's partials of all ranks are combined in global
// block order into dres[slot_cons..].
template <class PF, class CF>
void project_group(combo_ctx* c, int kind, PF&& prodf, CF&& consf, int slot_cons, double prod_bytes = 0.0) {
  const auto ms = members(c);
  using Prod = std::decay_t<decltype(prodf(size_t(0)))>;
  using Cons = std::decay_t<decltype(consf(size_t(0)))>;
  static_assert(Prod::NRED == 0, "producer reductions are not combined across ranks");
  for (size_t k = 0; k < ms.size(); ++k) launch_zfwd(ms[k], prodf(k), prod_bytes);
  if (c->R > 1 && overlap_knob()) {
    // Gamma couples only the components of one row group (green.cpp:114-127):
    // the transposes of group g run on the comm stream while the y / x
    // passes of the neighbouring groups run on the compute stream
    pipe_init(c);
    cudaStream_t cs = c->stream, xs = c->comm_stream;
    cudaEvent_t* ev = c->pipe_ev;  // [g]: y fwd done, [3+g]: to pencils done, [6+g]: x done, [9+g]: back done
    for (int g = 0; g < 3; ++g) {
      for (auto* m : ms) launch_y<false>(m, 3, 3 * g);
      COMBO_CK(cudaEventRecord(ev[g], cs));
      COMBO_CK(cudaStreamWaitEvent(xs, ev[g], 0));
      exchange(c, true, g, xs);
      COMBO_CK(cudaEventRecord(ev[3 + g], xs));
    }
    for (int g = 0; g < 3; ++g) {
      COMBO_CK(cudaStreamWaitEvent(cs, ev[3 + g], 0));
      for (auto* m : ms) launch_xgamma(m, kind, g, 1);
      COMBO_CK(cudaEventRecord(ev[6 + g], cs));
      COMBO_CK(cudaStreamWaitEvent(xs, ev[6 + g], 0));
      exchange(c, false, g, xs);
      COMBO_CK(cudaEventRecord(ev[9 + g], xs));
    }
    for (int g = 0; g < 3; ++g) {
      COMBO_CK(cudaStreamWaitEvent(cs, ev[9 + g], 0));
      for (auto* m : ms) launch_y<true>(m, 3, 3 * g);
    }
  } else {
    for (auto* m : ms) launch_y<false>(m);
    exchange(c, true);
    for (auto* m : ms) launch_xgamma(m, kind);
    exchange(c, false);
    for (auto* m : ms) launch_y<true>(m);
  }
  int64_t nbc = 0;
  for (size_t k = 0; k < ms.size(); ++k) nbc = launch_zinv(ms[k], consf(k));
  if (Cons::NRED) group_reduce(c, nbc, Cons::NRED, slot_cons);
}

void reset_stats(combo_ctx* c) {
  COMBO_CK(cudaMemsetAsync(leader(c)->dstats.p, 0, sizeof(Stats), leader(c)->stream));
}

// stress sweep: out = P(fin + sh) - alpha (fin + sh); P sums -> slot
// one rank's part: partials of its chunks, stats into the leader's counters
void sweep_launch(combo_ctx* c, const double* fin, const Shift9& sh, double alpha, double* out, bool writeback) {
  const int64_t nb = chunk_blocks(c);
  double* part = part_ptr(c, nb, 9);
  // F read + out write + cid, composite meta (n, c+, c-) and warm r/w
  ProfScope ps(c, kTagSweep, 148.0 * double(c->N) + 88.0 * double(c->ncomp));
  if (c->plan && c->plan->split_sweep && fin != out) {  // pass 1 writes out before pass 2 reads fin
    if (c->ncomp > 0) {
      const unsigned g = unsigned(std::min<int64_t>((c->ncomp + 127) / 128, int64_t(c->num_sms) * 64));
      k_sweep_comp<<<g, 128, 0, c->stream>>>(c->mp, c->cell_data(), fin, sh, out, c->N, writeback ? 1 : 0,
                                             stats_ptr(c));
      ++c->launches;
      COMBO_CK(cudaGetLastError());
    }
    k_sweep_pure<<<unsigned(nb), kEwThreads, 0, c->stream>>>(c->mp, c->cell_data(), fin, sh, alpha, out, c->N,
                                                             chunks_of(c), stats_ptr(c), part);
  } else {
    k_sweep<<<unsigned(nb), kEwThreads, 0, c->stream>>>(c->mp, c->cell_data(), fin, sh, alpha, out, c->N,
                                                        chunks_of(c), writeback ? 1 : 0, stats_ptr(c), part);
  }
  ++c->launches;
  COMBO_CK(cudaGetLastError());
}

void sweep(combo_ctx* c, const double* fin, const Shift9& sh, double alpha, double* out, bool writeback,
           int slot) {
  sweep_launch(c, fin, sh, alpha, out, writeback);
  group_reduce(c, chunk_blocks(c), 9, slot);
}

Shift9 zero_shift() {
  Shift9 s;
  for (double& v : s.v) v = 0.0;
  return s;
}

// packed effective tangents of every composite cell at (F + sh, warm starts)
void comp_tangents(combo_ctx* c, const double* F, const Shift9& sh) {
  if (!c->ncomp) return;
  c->t45.alloc(size_t(45 * c->ncomp));
  // F gather + meta + warm read, t45 write
  ProfScope ps(c, kTagOther, double(c->ncomp) * (72.0 + 64.0 + 360.0));
  const int64_t b = (c->ncomp + 127) / 128;
  k_comp_tangent<<<unsigned(std::min<int64_t>(b, 148 * 32)), 128, 0, c->stream>>>(c->mp, c->cell_data(), F, sh,
                                                                                     c->t45.p, c->N);
  ++c->launches;
  COMBO_CK(cudaGetLastError());
}

// ------------------------------------------------------- host tensors
// NH first elasticity tensor at F (closed form A_iJkL, see material.cuh)
// and Jacobi eigenvalues for the reference-medium choice
// (materials.cpp:112-125, cell_material.cpp:77-84, solver.cpp:99-104).
namespace {
double hdet3(const double* m) {
  return m[0] * (m[4] * m[8] - m[7] * m[5]) - m[3] * (m[1] * m[8] - m[7] * m[2]) + m[6] * (m[1] * m[5] - m[4] * m[2]);
}
bool nh_tangent_host(const combo_law& L, const double* f, double* A) {
  const double j = hdet3(f);
  if (!(j > 0.0)) return false;
  double g[9];
  g[0] = (f[4] * f[8] - f[5] * f[7]) / j;
  g[1] = (f[5] * f[6] - f[3] * f[8]) / j;
  g[2] = (f[3] * f[7] - f[4] * f[6]) / j;
  g[3] = (f[2] * f[7] - f[1] * f[8]) / j;
  g[4] = (f[0] * f[8] - f[2] * f[6]) / j;
  g[5] = (f[1] * f[6] - f[0] * f[7]) / j;
  g[6] = (f[1] * f[5] - f[2] * f[4]) / j;
  g[7] = (f[2] * f[3] - f[0] * f[5]) / j;
  g[8] = (f[0] * f[4] - f[1] * f[3]) / j;
  const double lnj = std::log(j);
  const double beta = L.mu - L.lambda * lnj;
  for (int i = 0; i < 3; ++i)
    for (int J = 0; J < 3; ++J)
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l)
          A[9 * (3 * i + J) + 3 * k + l] = (i == k && J == l ? L.mu : 0.0) + L.lambda * g[3 * i + J] * g[3 * k + l] +
                                           beta * g[3 * i + l] * g[3 * k + J];
  return true;
}

void jacobi_eigenvalues(int n, double* a, double* lam) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
    if (off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double app = a[p * n + p], aqq = a[q * n + q];
        const double g = 100.0 * std::fabs(apq);
        if (std::fabs(app) + g == std::fabs(app) && std::fabs(aqq) + g == std::fabs(aqq)) {
          a[p * n + q] = a[q * n + p] = 0.0;
          continue;
        }
        const double h = aqq - app;
        double t;
        if (std::fabs(h) + g == std::fabs(h)) {
          t = apq / h;
        } else {
          const double th = 0.5 * h / apq;
          t = 1.0 / (std::fabs(th) + std::sqrt(1.0 + th * th));
          if (th < 0.0) t = -t;
        }
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = t * cs, tau = sn / (1.0 + cs);
        a[p * n + p] = app - t * apq;
        a[q * n + q] = aqq + t * apq;
        a[p * n + q] = a[q * n + p] = 0.0;
        for (int r = 0; r < n; ++r) {
          if (r == p || r == q) continue;
          const double gr = a[r * n + p], hr = a[r * n + q];
          a[r * n + p] = a[p * n + r] = gr - sn * (hr + gr * tau);
          a[r * n + q] = a[q * n + r] = hr + sn * (gr - hr * tau);
        }
      }
  }
  for (int i = 0; i < n; ++i) lam[i] = a[i * n + i];
  std::sort(lam, lam + n);
}

void law_bounds(const combo_law& L, const double* f, double& lo, double& hi) {
  if (L.kind == COMBO_LAW_LINEAR) {
    double a[36], lam[6];
    std::memcpy(a, L.c6, sizeof a);
    jacobi_eigenvalues(6, a, lam);
    lo = std::min(0.0, lam[0]);
    hi = lam[5];
    return;
  }
  double A[81];
  if (!nh_tangent_host(L, f, A)) {
    lo = L.mu;
    hi = L.lambda + 2.0 * L.mu;
    return;
  }
  double s[81], lam[9];
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j < 9; ++j) s[9 * i + j] = 0.5 * (A[9 * i + j] + A[9 * j + i]);
  jacobi_eigenvalues(9, s, lam);
  lo = lam[0];
  hi = lam[8];
}
}  // namespace

void spectrum_bounds(const combo_ctx* c, const double* fbar, double& lo, double& hi) {
  double l0, h0, l1, h1;
  law_bounds(c->law_m, fbar, l0, h0);
  law_bounds(c->law_i, fbar, l1, h1);
  lo = std::min(l0, l1);
  hi = std::max(h0, h1);
}

// mandel_to_mat9 (tensor.cpp:127-136) for the linear law
void mandel_to_mat9(const double* c6, double* a9) {
  static const int pair[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
  const double s2 = 1.4142135623730951;
  double full[81] = {0};
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      const int i = pair[a][0], j = pair[a][1], k = pair[b][0], l = pair[b][1];
      const double v = c6[6 * a + b] / ((a < 3 ? 1.0 : s2) * (b < 3 ? 1.0 : s2));
      full[((i * 3 + j) * 3 + k) * 3 + l] = v;
      full[((j * 3 + i) * 3 + k) * 3 + l] = v;
      full[((i * 3 + j) * 3 + l) * 3 + k] = v;
      full[((j * 3 + i) * 3 + l) * 3 + k] = v;
    }
  for (int i = 0; i < 81; ++i) a9[i] = full[i];
}

// dev_a9: 81 doubles of device memory owned by the caller (linear law only)
LawP law_params(const combo_law& L, double* dev_a9) {
  LawP p{};
  p.kind = L.kind;
  p.lambda = L.lambda;
  p.mu = L.mu;
  p.a9 = nullptr;
  if (L.kind == COMBO_LAW_LINEAR) {
    double a9[81];
    mandel_to_mat9(L.c6, a9);
    COMBO_CK(cudaMemcpy(dev_a9, a9, sizeof a9, cudaMemcpyHostToDevice));
    p.a9 = dev_a9;
  }
  return p;
}

// ------------------------------------------------------------------ solver
namespace {
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }
double norm9(const double* m) {
  double s = 0.0;
  for (int i = 0; i < 9; ++i) s += m[i] * m[i];
  return std::sqrt(s);
}
struct LsBudget {};
}  // namespace

// One rank's solver state: the 9N_local field slots (F, F_new/F_trial, x, r,
// pdir, ap, P or tau, spare residual) of a slab.
struct SolverRank {
  combo_ctx* c;
  int64_t N;
  DBuf<double>* f;  // c->solver_fields
};

// The solver runs every rank hosted by the leader context in lockstep: each
// field-sized step is launched per rank, scalars are combined across ranks
// in global block order (group_reduce), the spectrum is transposed inside
// project_group. With one rank it is the plain single-GPU solver.
class Solver {
 public:
  Solver(combo_ctx* c, const combo_solver_cfg& cfg) : c_(c), cfg_(cfg), Ng_(c->Ng) {
    ensure_scratch(c);
    for (combo_ctx* m : members(c)) {
      rk_.emplace_back();
      SolverRank& r = rk_.back();
      r.c = m;
      r.N = m->N;
      r.f = m->solver_fields;
      for (int q = 0; q < 8; ++q) r.f[q].alloc(size_t(9 * r.N));
    }
    double lo, hi;
    const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    spectrum_bounds(c, I, lo, hi);
    stress_floor_ = 1e-12 * std::max(hi, 1e-12);
    shF_ = zero_shift();
  }

  void run(const double* fbar_target, combo_report& rep);
  double* F(size_t k) { return P(F_, k); }
  double* scratch(size_t k) { return P(rb_, k); }
  size_t nranks() const { return rk_.size(); }
  const double* pbar() const { return pbar_; }
  void final_stress(const std::vector<double*>& out);
  void materialize();

 private:
  double* P(int slot, size_t k) { return rk_[k].f[slot].p; }
  // slot `slot` of every rank
  std::vector<double*> field(int slot) {
    std::vector<double*> v;
    for (size_t k = 0; k < rk_.size(); ++k) v.push_back(P(slot, k));
    return v;
  }
  std::vector<const double*> cfield(int slot) {
    std::vector<const double*> v;
    for (size_t k = 0; k < rk_.size(); ++k) v.push_back(P(slot, k));
    return v;
  }
  bool run_step(const double* fbar, combo_host::StepRec& rep);
  bool run_basic(const double* fbar, combo_host::StepRec& rep);
  bool run_newton(const double* fbar, combo_host::StepRec& rep);
  int cg_solve(double tol_rel, double rr0, bool& breakdown, combo_host::StepRec& rep);
  void count_ls() {
    if (cfg_.max_ls_iterations > 0 && ls_total_ >= cfg_.max_ls_iterations) throw LsBudget{};
    ++ls_total_;
  }
  // eval_stress (solver.cpp:59-63): per-cell sweep or DFMG; P sums -> slot
  void eval_sweep(int fin, const Shift9& sh, double alpha, int out, bool writeback, int slot) {
    if (cfg_.eval == COMBO_EVAL_DFMG) {
      dfmg_sweep(c_, cfield(fin), sh, alpha, field(out), slot);
      return;
    }
    for (size_t k = 0; k < rk_.size(); ++k) sweep_launch(rk_[k].c, P(fin, k), sh, alpha, P(out, k), writeback);
    group_reduce(c_, chunk_blocks(c_), 9, slot);
  }
  combo_sweep_stats stats() const {
    const Stats* s = reinterpret_cast<const Stats*>(c_->hres + 64);
    combo_sweep_stats o;
    o.inadmissible_cells = int64_t(s->inadmissible);
    o.laminate_failures = int64_t(s->failures);
    o.back_projections = int64_t(s->backproj);
    o.laminate_iter_max = int64_t(s->iter_max);
    return o;
  }
  // F + shift materialized in place; per-component sums -> slot
  void materialize_sum(int slot) {
    const int64_t nb = chunk_blocks(c_);
    for (auto& r : rk_) {
      double* part = part_ptr(r.c, nb, 9);
      ProfScope ps(r.c, kTagMaterialize, 144.0 * double(r.N));
      k_materialize<<<unsigned(nb), kEwThreads, 0, r.c->stream>>>(r.f[F_].p, shF_, r.N, chunks_of(r.c), part);
      ++r.c->launches;
      COMBO_CK(cudaGetLastError());
    }
    group_reduce(c_, nb, 9, slot);
  }
  // pin_mean on F (field.cpp:28-38): materialize pending shift, sum, new shift
  void pin_mean(const double* target) {
    materialize_sum(0);
    fetch_results(c_, false);
    for (int q = 0; q < 9; ++q) shF_.v[q] = target[q] - c_->hres[q] / double(Ng_);
  }
  void copy_all(int dst, int src) {
    for (auto& r : rk_)
      COMBO_CK(cudaMemcpyAsync(r.f[dst].p, r.f[src].p, size_t(9 * r.N) * sizeof(double), cudaMemcpyDeviceToDevice,
                               r.c->stream));
  }

  combo_ctx* c_;
  combo_solver_cfg cfg_;
  int64_t Ng_;
  std::vector<SolverRank> rk_;
  // field slots (indices into SolverRank::f); swaps exchange the indices
  int F_ = 0, Fo_ = 1, x_ = 2, r_ = 3, pd_ = 4, ap_ = 5, rb_ = 6, bn_ = 7;
  Shift9 shF_;
  double alpha_ = 1.0;
  double stress_floor_;
  double pbar_[9] = {0};
  int64_t ls_total_ = 0;
  int last_eval_ = -1;
  Shift9 last_eval_shift_;
};

void Solver::materialize() {
  materialize_sum(0);
  shF_ = zero_shift();
}

// run_basic (solver.cpp:124-164)
bool Solver::run_basic(const double* fbar, combo_host::StepRec& rep) {
  double lo, hi;
  spectrum_bounds(c_, fbar, lo, hi);  // pick_alpha (:99-104)
  alpha_ = 0.5 * (std::max(lo, 0.0) + hi);
  if (!(alpha_ > 0.0)) alpha_ = std::max(hi, 1.0);
  for (int it = 1; it <= cfg_.max_outer; ++it) {
    reset_stats(c_);
    eval_sweep(F_, shF_, alpha_, rb_, true, 0);  // tau = P - alpha F ; P sums -> slot 0
    last_eval_ = F_;
    last_eval_shift_ = shF_;
    project_group(
        c_, cfg_.green, [&](size_t k) { return ProdLoad9{P(rb_, k), rk_[k].N}; },
        [&](size_t k) {
          ConsBasic cons;
          cons.fold = P(F_, k);
          cons.fold_shift = shF_;
          cons.fnew = P(Fo_, k);
          for (int q = 0; q < 9; ++q) cons.fbar.v[q] = fbar[q];
          cons.alpha = alpha_;
          cons.N = rk_[k].N;
          return cons;
        },
        9);  // diff^2 -> 9, F_new sums -> 10..18
    fetch_results(c_);
    rep.sweep = stats();
    if (rep.sweep.inadmissible_cells > 0) return false;
    count_ls();
    ++rep.ls_basic;
    for (int q = 0; q < 9; ++q) pbar_[q] = c_->hres[q] / double(Ng_);
    rep.pbar_history.push_back({});
    std::memcpy(rep.pbar_history.back().data(), pbar_, sizeof pbar_);
    const double resid = alpha_ * std::sqrt(c_->hres[9] / double(Ng_)) / std::max(norm9(pbar_), stress_floor_);
    rep.residuals.push_back(resid);
    rep.cg_iters.push_back(0);
    rep.outer_iters = it;
    if (cfg_.verbose) std::printf("  basic it %3d resid %.3e\n", it, resid);
    std::swap(F_, Fo_);
    for (int q = 0; q < 9; ++q) shF_.v[q] = fbar[q] - c_->hres[10 + q] / double(Ng_);
    if (rep.sweep.laminate_failures > 0 && resid <= cfg_.tol_equilibrium) return false;
    if (resid <= cfg_.tol_equilibrium) {
      rep.converged = true;
      return true;
    }
  }
  return false;
}

// cg_solve (solver.cpp:166-200); r holds b on entry, x is zeroed here
int Solver::cg_solve(double tol_rel, double rr0, bool& breakdown, combo_host::StepRec& rep) {
  breakdown = false;
  for (auto& r : rk_) COMBO_CK(cudaMemsetAsync(r.f[x_].p, 0, size_t(9 * r.N) * sizeof(double), r.c->stream));
  double rr = rr0;
  const double bnorm = std::sqrt(rr);
  if (bnorm == 0.0) return 0;
  // tangents of this Newton iteration (stress_sweep(&tangents45) /
  // dfmg_tangent_pass, solver.cpp:72-82)
  const bool dfmg = cfg_.eval == COMBO_EVAL_DFMG;
  if (dfmg)
    dfmg_tangent_prepare(c_, cfield(F_), shF_);
  else
    for (auto& r : rk_) comp_tangents(r.c, r.f[F_].p, shF_);
  int it = 0;
  double beta = 0.0, step_prev = 0.0;
  const int64_t nbc = chunk_blocks(c_);
  // x += step * pdir is deferred into the next matvec (which reads pdir
  // anyway); the last pending update is flushed on exit (solver.cpp:186)
  auto axpy_x = [&](double s) {
    for (auto& r : rk_) {
      ProfScope ps(r.c, kTagCgUpdate, 216.0 * double(r.N));
      k_axpy<<<ew_grid(9 * r.N), kEwThreads, 0, r.c->stream>>>(r.f[x_].p, r.f[pd_].p, s, 9 * r.N);
      ++r.c->launches;
      COMBO_CK(cudaGetLastError());
    }
  };
  auto flush_x = [&]() {
    if (dfmg || it == 0) return;
    axpy_x(step_prev);
  };
  auto cons = [&](size_t k) { return ConsCg{P(ap_, k), P(pd_, k), rk_[k].N}; };
  // pdir^T A pdir taken in the matvec as pdir . q (see MatvecArgs::pq_part):
  // the step is known before the projection, whose z-inverse applies
  // r -= s Pi(q) and sums r^T r (ConsCgUpdate). Needs the bulk matvec and
  // tiles that do not straddle planes (decomposition invariance).
  bool pq = !dfmg && c_->plan->pq_dot && (c_->dims[1] * c_->dims[2]) % combo_dev::kMvT == 0;
  const int64_t ntiles = (c_->N / combo_dev::kMvT) * (combo_dev::kMvT / 32);  // per-warp sums
  while (it < cfg_.cg_max) {
    count_ls();
    ++rep.ls_cg;
    if (dfmg) {
      dfmg_matvec(c_, cfield(F_), shF_, cfield(r_), field(pd_), beta, it == 0, field(rb_));
      COMBO_CK(cudaGetLastError());
      project_group(
          c_, cfg_.green, [&](size_t k) { return ProdLoad9{P(rb_, k), rk_[k].N}; }, cons, 20);
    } else {
      // r, F, cid, pdir (r/w), x (r/w, deferred update); composite packed tangents
      auto mv = [&](size_t k) {
        combo_ctx* m = rk_[k].c;
        return MatvecArgs{m->mp, m->cell_data(), P(F_, k), shF_, P(r_, k), P(pd_, k), beta, it == 0 ? 1 : 0,
                          rk_[k].N, P(x_, k), step_prev, nullptr};
      };
      if (pq)
        for (size_t k = 0; k < rk_.size(); ++k) pq = pq && mv_bulk_ok(rk_[k].c, mv(k));
      const double mvb = (it == 0 ? 220.0 : 436.0) * double(c_->N) + 360.0 * double(c_->ncomp);
      {
        for (size_t k = 0; k < rk_.size(); ++k) {
          combo_ctx* m = rk_[k].c;
          ProfScope ps(m, kTagMatvec, mvb + 72.0 * double(rk_[k].N));
          MatvecArgs a = mv(k);
          if (pq) a.pq_part = part_ptr(m, ntiles, 1);
          launch_matvec(m, a, P(rb_, k));
          ++m->launches;
          COMBO_CK(cudaGetLastError());
        }
        if (pq) {
          // pap -> dres[20]; the host forms s = rr / pap (one scalar round
          // trip), the z-inverse writes r' = r - s Pi(q) into the free ap
          // slot and sums r'^T r' -> dres[21]
          group_reduce(c_, ntiles, 1, 20);
          fetch_results(c_, false);
          const double pap = c_->hres[20];
          if (!(pap > 0.0)) {
            breakdown = true;  // solver.cpp:182-185 (see below)
            return it;
          }
          const double s = rr / pap;
          project_group(
              c_, cfg_.green, [&](size_t k) { return ProdLoad9{P(rb_, k), rk_[k].N}; },
              [&](size_t k) { return ConsCgUpdate{P(r_, k), P(ap_, k), s, rk_[k].N}; }, 21);
          std::swap(r_, ap_);
        } else {
          project_group(
              c_, cfg_.green, [&](size_t k) { return ProdLoad9{P(rb_, k), rk_[k].N}; }, cons, 20);
        }
      }
    }
    fetch_results(c_, false);
    const double pap = c_->hres[20];
    if (!(pap > 0.0)) {
      breakdown = true;
      // the previous iteration's x update was applied by this iteration's
      // matvec; this iteration's is not applied (solver.cpp:182-185)
      return it;
    }
    const double step = rr / pap;
    if (dfmg) axpy_x(step);
    if (!pq) {
      for (auto& r : rk_) {
        double* part = part_ptr(r.c, nbc, 1);
        ProfScope ps(r.c, kTagCgUpdate, 216.0 * double(r.N));
        k_cg_update<<<unsigned(nbc), kEwThreads, 0, r.c->stream>>>(r.f[r_].p, r.f[ap_].p, step, r.N, chunks_of(r.c),
                                                                     part);
        ++r.c->launches;
        COMBO_CK(cudaGetLastError());
      }
      group_reduce(c_, nbc, 1, 21);
      fetch_results(c_, false);
    }
    ++it;
    step_prev = step;
    const double rr_new = c_->hres[21];
    if (std::sqrt(rr_new) <= tol_rel * bnorm) {
      flush_x();
      return it;
    }
    beta = rr_new / rr;
    rr = rr_new;
  }
  flush_x();
  return it;
}

// run_newton (solver.cpp:202-259) with the accepted trial's residual reused
// as the next Newton residual (bitwise identical when the trial sweep had no
// laminate failures; still counted as an LS iteration).
bool Solver::run_newton(const double* fbar, combo_host::StepRec& rep) {
  bool reuse = false;
  double reuse_ss = 0.0, reuse_pbar[9];
  for (int it = 1; it <= cfg_.max_outer; ++it) {
    double ss;
    if (!reuse) {
      reset_stats(c_);
      eval_sweep(F_, shF_, 0.0, rb_, true, 0);
      last_eval_ = F_;
      last_eval_shift_ = shF_;
      fetch_results(c_);
      rep.sweep = stats();
      if (rep.sweep.inadmissible_cells > 0) return false;
      for (int q = 0; q < 9; ++q) pbar_[q] = c_->hres[q] / double(Ng_);
      count_ls();
      ++rep.ls_residual;
      project_group(
          c_, cfg_.green, [&](size_t k) { return ProdLoad9{P(rb_, k), rk_[k].N}; },
          [&](size_t k) { return ConsResid{P(r_, k), rk_[k].N}; }, 9);
      fetch_results(c_, false);
      ss = c_->hres[9];
    } else {
      rep.sweep = combo_sweep_stats{0, 0, 0, 0};
      std::memcpy(pbar_, reuse_pbar, sizeof pbar_);
      count_ls();
      ++rep.ls_residual;
      std::swap(r_, bn_);
      ss = reuse_ss;
    }
    rep.pbar_history.push_back({});
    std::memcpy(rep.pbar_history.back().data(), pbar_, sizeof pbar_);
    const double den = std::max(norm9(pbar_), stress_floor_);
    const double resid = std::sqrt(ss / double(Ng_)) / den;
    rep.residuals.push_back(resid);
    rep.outer_iters = it;
    if (cfg_.verbose) std::printf("  newton it %3d resid %.3e\n", it, resid);
    if (resid <= cfg_.tol_equilibrium) {
      rep.cg_iters.push_back(0);
      rep.converged = rep.sweep.laminate_failures == 0;
      return rep.converged;
    }
    const double eta = std::max(std::min(cfg_.cg_tol, std::sqrt(resid)), 1e-8);
    bool breakdown = false;
    const int cg_its = cg_solve(eta, ss, breakdown, rep);
    rep.cg_iters.push_back(cg_its);
    if (breakdown) {
      ++rep.cg_breakdowns;
      if (cg_its == 0) return false;
    }
    // backtracking line search (:238-255)
    double s = 1.0;
    bool accepted = false;
    combo_sweep_stats st_acc{};
    double ss_acc = 0.0;
    Shift9 sh_t{};
    const int64_t nbc = chunk_blocks(c_);
    for (int ls = 0; ls < 10; ++ls) {
      for (size_t k = 0; k < rk_.size(); ++k) {
        combo_ctx* m = rk_[k].c;
        double* part = part_ptr(m, nbc, 9);
        ProfScope ps(m, kTagTrial, 216.0 * double(rk_[k].N));
        k_trial<<<unsigned(nbc), kEwThreads, 0, m->stream>>>(P(F_, k), shF_, P(x_, k), s, P(Fo_, k), rk_[k].N,
                                                               chunks_of(m), part);
        ++m->launches;
        COMBO_CK(cudaGetLastError());
      }
      group_reduce(c_, nbc, 9, 30);
      fetch_results(c_, false);
      for (int q = 0; q < 9; ++q) sh_t.v[q] = fbar[q] - c_->hres[30 + q] / double(Ng_);
      reset_stats(c_);
      eval_sweep(Fo_, sh_t, 0.0, rb_, true, 0);
      last_eval_ = Fo_;
      last_eval_shift_ = sh_t;
      fetch_results(c_);
      const combo_sweep_stats st = stats();
      if (st.inadmissible_cells == 0) {
        double pb[9];
        for (int q = 0; q < 9; ++q) pb[q] = c_->hres[q] / double(Ng_);
        count_ls();
        ++rep.ls_trial;
        project_group(
            c_, cfg_.green, [&](size_t k) { return ProdLoad9{P(rb_, k), rk_[k].N}; },
            [&](size_t k) { return ConsResid{P(bn_, k), rk_[k].N}; }, 9);
        fetch_results(c_, false);
        const double ss_t = c_->hres[9];
        std::memcpy(pbar_, pb, sizeof pb);  // residual_from_stress sets pbar_ (:95)
        const double rtrial = std::sqrt(ss_t / double(Ng_)) / std::max(norm9(pb), stress_floor_);
        if (rtrial <= resid * (1.0 + 1e-12)) {
          accepted = true;
          st_acc = st;
          ss_acc = ss_t;
          std::memcpy(reuse_pbar, pb, sizeof pb);
          break;
        }
      }
      s *= 0.5;
      ++rep.line_search_cuts;
    }
    if (!accepted) return false;
    std::swap(F_, Fo_);
    shF_ = sh_t;
    if (last_eval_ == Fo_) last_eval_ = F_;
    reuse = st_acc.laminate_failures == 0;
    reuse_ss = ss_acc;
  }
  return false;
}

bool Solver::run_step(const double* fbar, combo_host::StepRec& rep) {
  return cfg_.scheme == COMBO_SCHEME_BASIC ? run_basic(fbar, rep) : run_newton(fbar, rep);
}

// solve (solver.cpp:286-346)
void Solver::run(const double* fbar_target, combo_report& report) {
  const auto tic = Clock::now();
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double h[9];
  for (int q = 0; q < 9; ++q) h[q] = fbar_target[q] - I[q];
  double t = 0.0;
  double dt = 1.0 / cfg_.load_steps;
  double fbar_prev[9];
  std::memcpy(fbar_prev, I, sizeof I);
  {
    Shift9 one;
    for (int q = 0; q < 9; ++q) one.v[q] = I[q];
    for (auto& r : rk_) {
      k_fill9<<<ew_grid(r.N), kEwThreads, 0, r.c->stream>>>(r.f[F_].p, one, r.N);
      ++r.c->launches;
    }
  }
  shF_ = zero_shift();
  report.success = true;
  // per-rank backups of F and the warm starts (solver.cpp:313-315)
  std::vector<DBuf<double>> backup_f(rk_.size()), backup_warm(rk_.size());
  for (size_t k = 0; k < rk_.size(); ++k) {
    backup_f[k].alloc(size_t(9 * rk_[k].N));
    if (rk_[k].c->ncomp) backup_warm[k].alloc(size_t(3 * rk_[k].c->ncomp));
  }
  std::vector<DBuf<double>> dfmg_backup(rk_.size());  // DfmgState warm starts (solver.cpp:315,330)
  if (cfg_.eval == COMBO_EVAL_DFMG) {
    // fresh DfmgState per solve (CellSolver ctor, solver.cpp:55)
    for (size_t k = 0; k < rk_.size(); ++k) {
      combo_ctx* m = rk_[k].c;
      m->dfmg_warm.alloc(size_t(3 * 8 * std::max<int64_t>(m->ncomp, 1)));
      COMBO_CK(cudaMemsetAsync(m->dfmg_warm.p, 0, m->dfmg_warm.n * 8, m->stream));
      dfmg_backup[k].alloc(m->dfmg_warm.n);
    }
  }
  auto save_or_restore = [&](bool save) {
    for (size_t k = 0; k < rk_.size(); ++k) {
      combo_ctx* m = rk_[k].c;
      double* f = P(F_, k);
      COMBO_CK(cudaMemcpyAsync(save ? backup_f[k].p : f, save ? f : backup_f[k].p,
                               size_t(9 * rk_[k].N) * sizeof(double), cudaMemcpyDeviceToDevice, m->stream));
      if (m->ncomp)
        COMBO_CK(cudaMemcpyAsync(save ? backup_warm[k].p : m->warm.p, save ? m->warm.p : backup_warm[k].p,
                                 size_t(3 * m->ncomp) * sizeof(double), cudaMemcpyDeviceToDevice, m->stream));
      if (dfmg_backup[k].p)
        COMBO_CK(cudaMemcpyAsync(save ? dfmg_backup[k].p : m->dfmg_warm.p, save ? m->dfmg_warm.p : dfmg_backup[k].p,
                                 dfmg_backup[k].n * sizeof(double), cudaMemcpyDeviceToDevice, m->stream));
    }
  };
  try {
    while (t < 1.0 - 1e-12) {
      const double dt_try = std::min(dt, 1.0 - t);
      double fbar[9];
      for (int q = 0; q < 9; ++q) fbar[q] = I[q] + (t + dt_try) * h[q];
      // backup F (materialized) and warm starts
      materialize();
      save_or_restore(true);
      pin_mean(fbar);
      combo_host::StepRec rep;
      rep.t_start = t;
      rep.t_end = t + dt_try;
      std::memcpy(rep.fbar, fbar, sizeof fbar);
      const auto st0 = Clock::now();
      bool ok = false;
      try {
        ok = run_step(fbar, rep);
      } catch (const LsBudget&) {
        // the step cut short by the LS budget is reported (oracle/solver.cpp)
        rep.seconds = since(st0);
        report.steps.push_back(std::move(rep));
        throw;
      }
      rep.converged = ok;
      rep.seconds = since(st0);
      if (ok) {
        report.steps.push_back(std::move(rep));
        t += dt_try;
        std::memcpy(fbar_prev, fbar, sizeof fbar);
        continue;
      }
      // P of the solve is the stress of the last evaluated F (solver.cpp:343,
      // p_): keep that F out of the slot the backup is restored into
      if (last_eval_ == F_) {
        copy_all(Fo_, F_);
        last_eval_ = Fo_;
      }
      save_or_restore(false);
      shF_ = zero_shift();
      pin_mean(fbar_prev);
      ++report.bisections;
      if (report.bisections > cfg_.max_bisections) {
        report.steps.push_back(std::move(rep));
        report.success = false;
        report.error = "LoadPathFailed: bisection budget exhausted";
        break;
      }
      dt = 0.5 * dt_try;
    }
  } catch (const LsBudget&) {
    report.success = false;
    report.error = "LsBudgetExhausted";
  }
  COMBO_CK(cudaStreamSynchronize(c_->stream));
  report.alpha = alpha_;
  report.ls_total = ls_total_;
  report.seconds_total = since(tic);
}

// P of the last evaluated state into out[k] (one pointer per rank)
void Solver::final_stress(const std::vector<double*>& out) {
  const int fin = last_eval_ >= 0 ? last_eval_ : F_;
  const Shift9 sh = last_eval_ >= 0 ? last_eval_shift_ : shF_;
  reset_stats(c_);
  if (cfg_.eval == COMBO_EVAL_DFMG) {
    dfmg_sweep(c_, cfield(fin), sh, 0.0, out, 40);
    return;
  }
  for (size_t k = 0; k < rk_.size(); ++k) sweep_launch(rk_[k].c, P(fin, k), sh, 0.0, out[k], false);
  group_reduce(c_, chunk_blocks(c_), 9, 40);
}

std::string report_json(const combo_report& r) {
  auto fmt = [](double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return std::string(b);
  };
  std::ostringstream js;
  js << "{\"success\":" << (r.success ? "true" : "false") << ",\"error\":\"" << r.error
     << "\",\"bisections\":" << r.bisections << ",\"alpha\":" << fmt(r.alpha)
     << ",\"seconds_total\":" << fmt(r.seconds_total) << ",\"ls_total\":" << r.ls_total << ",\"steps\":[";
  for (size_t s = 0; s < r.steps.size(); ++s) {
    const auto& st = r.steps[s];
    if (s) js << ",";
    js << "{\"t_start\":" << fmt(st.t_start) << ",\"t_end\":" << fmt(st.t_end)
       << ",\"converged\":" << (st.converged ? "true" : "false") << ",\"outer_iters\":" << st.outer_iters
       << ",\"cg_breakdowns\":" << st.cg_breakdowns << ",\"line_search_cuts\":" << st.line_search_cuts
       << ",\"seconds\":" << fmt(st.seconds) << ",\"ls_basic\":" << st.ls_basic << ",\"ls_residual\":" << st.ls_residual
       << ",\"ls_cg\":" << st.ls_cg << ",\"ls_trial\":" << st.ls_trial << ",\"fbar\":[";
    for (int i = 0; i < 9; ++i) js << (i ? "," : "") << fmt(st.fbar[i]);
    js << "],\"residuals\":[";
    for (size_t i = 0; i < st.residuals.size(); ++i) js << (i ? "," : "") << fmt(st.residuals[i]);
    js << "],\"cg_iters\":[";
    for (size_t i = 0; i < st.cg_iters.size(); ++i) js << (i ? "," : "") << st.cg_iters[i];
    js << "],\"pbar_history\":[";
    for (size_t i = 0; i < st.pbar_history.size(); ++i) {
      js << (i ? "," : "") << "[";
      for (int q = 0; q < 9; ++q) js << (q ? "," : "") << fmt(st.pbar_history[i][size_t(q)]);
      js << "]";
    }
    js << "],\"sweep\":{\"inadmissible\":" << st.sweep.inadmissible_cells << ",\"failures\":" << st.sweep.laminate_failures
       << ",\"back_projections\":" << st.sweep.back_projections << ",\"iter_max\":" << st.sweep.laminate_iter_max << "}}";
  }
  js << "]}";
  return js.str();
}

}  // namespace combo_host

// ====================================================================== C-ABI
using namespace combo_host;

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
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return COMBO_ERR_OOM;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return COMBO_ERR_BAD_ARGUMENT;
  }
}

// Every rank of a single-process multi-GPU group runs fn on its own host
// thread with its device current (the NCCL clique needs all ranks inside a
// collective at once); a plain context runs fn inline. A failing rank
// aborts the clique so the others leave their collectives, and the first
// error is rethrown.
template <class Fn>
void on_ranks(combo_ctx* c, Fn&& fn) {
  if (!c->multi) {
    fn(c);
    return;
  }
  std::vector<combo_ctx*> rs{c};
  for (auto& p : c->peers) rs.push_back(p.get());
  std::vector<std::exception_ptr> errs(rs.size());
  std::vector<std::thread> th;
  for (size_t k = 0; k < rs.size(); ++k)
    th.emplace_back([&, k] {
      try {
        COMBO_CK(cudaSetDevice(rs[k]->device));
        fn(rs[k]);
      } catch (...) {
        errs[k] = std::current_exception();
        for (auto* r : rs) {
          try {
            nccl_abort(r);
          } catch (...) {
          }
        }
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void require_bound(const combo_ctx* c) {
  if (!c->bound) throw ComboError(COMBO_ERR_STATE, "materials not bound (combo_bind_materials)");
}

// stage a 9N field to the device (returns device pointer)
const double* stage_in(combo_ctx* c, const double* p, int mem, int slot) {
  if (mem == COMBO_MEM_DEVICE) return p;
  c->scratch[slot].alloc(size_t(9 * c->N));
  COMBO_CK(cudaMemcpyAsync(c->scratch[slot].p, p, size_t(9 * c->N) * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return c->scratch[slot].p;
}
double* stage_out(combo_ctx* c, double* p, int mem, int slot) {
  if (mem == COMBO_MEM_DEVICE) return p;
  c->scratch[slot].alloc(size_t(9 * c->N));
  return c->scratch[slot].p;
}
void finish_out(combo_ctx* c, double* host, const double* dev, int mem, size_t count) {
  if (mem == COMBO_MEM_DEVICE) return;
  COMBO_CK(cudaMemcpyAsync(host, dev, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaStreamSynchronize(c->stream));
}
}  // namespace

extern "C" {

const char* combo_version(void) { return "combo-b200 0.1 (sm_100a, fp64)"; }

int combo_ctx_create(int device, combo_ctx** out) {
  if (!out) return COMBO_ERR_BAD_ARGUMENT;
  *out = nullptr;
  auto* c = new combo_ctx();
  c->device = device;
  const int rc = guarded(c, [&] {
    int n = 0;
    COMBO_CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "no such CUDA device");
    COMBO_CK(cudaSetDevice(device));
    COMBO_CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    COMBO_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    ensure_scratch(c);
  });
  if (rc) {
    delete c;
    return rc;
  }
  *out = c;
  return COMBO_OK;
}

// One process, R GPUs (combo_ctx_create(ndev, devices)):
// rank q lives on devices[q], the slab / pencil exchanges and reductions run
// over an ncclCommInitAll clique; bind / solve / project take whole-grid
// arrays as with one GPU.
int combo_ctx_create_multi(int ndev, const int* devices, combo_ctx** out) {
  if (!out || ndev < 1 || !devices) return COMBO_ERR_BAD_ARGUMENT;
  *out = nullptr;
  for (int a = 0; a < ndev; ++a)
    for (int b = a + 1; b < ndev; ++b)
      if (devices[a] == devices[b]) return COMBO_ERR_BAD_ARGUMENT;
  combo_ctx* lead = nullptr;
  int rc = combo_ctx_create(devices[0], &lead);
  if (rc) return rc;
  rc = guarded(lead, [&] {
    std::vector<combo_ctx*> rs{lead};
    for (int q = 1; q < ndev; ++q) {
      combo_ctx* p = nullptr;
      const int r = combo_ctx_create(devices[q], &p);
      if (r) throw ComboError(r, "combo_ctx_create_multi: device " + std::to_string(devices[q]));
      lead->peers.emplace_back(p);
      rs.push_back(p);
    }
    if (ndev > 1) nccl_init_all(rs);  // one device: the same threaded path without a clique
    for (int q = 0; q < ndev; ++q) {
      rs[size_t(q)]->R = ndev;
      rs[size_t(q)]->q = q;
      rs[size_t(q)]->in_multi = true;
    }
    lead->multi = true;
  });
  if (rc) {
    combo_ctx_destroy(lead);
    return rc;
  }
  *out = lead;
  return COMBO_OK;
}

int combo_ctx_destroy(combo_ctx* c) {
  if (!c) return COMBO_OK;
  for (auto& p : c->peers) combo_ctx_destroy(p.release());
  c->peers.clear();
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& m : c->vm)
    if (m->hres) cudaFreeHost(m->hres);
  c->vm.clear();
  try {
    nccl_destroy(c);
  } catch (...) {
  }
  c->plan.reset();
  if (c->hres) cudaFreeHost(c->hres);
  if (c->comm_stream) {
    cudaStreamDestroy(c->comm_stream);
    for (auto e : c->pipe_ev)
      if (e) cudaEventDestroy(e);
  }
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return COMBO_OK;
}

const char* combo_last_error(const combo_ctx* c) { return c ? c->err.c_str() : "null context"; }

int combo_kernel_launches(const combo_ctx* c, int64_t* count) {
  if (!c || !count) return COMBO_ERR_BAD_ARGUMENT;
  *count = c->launches;
  for (const auto& p : c->peers) *count += p->launches;
  return COMBO_OK;
}

int combo_synchronize(combo_ctx* c) {
  return guarded(c, [&] { on_ranks(c, [](combo_ctx* r) { COMBO_CK(cudaStreamSynchronize(r->stream)); }); });
}

int combo_profile_enable(combo_ctx* c, int enable) {
  return guarded(c, [&] {
    COMBO_CK(cudaStreamSynchronize(c->stream));
    for (auto& r : c->prof) {
      c->ev_pool.push_back(r.a);
      c->ev_pool.push_back(r.b);
    }
    c->prof.clear();
    c->prof_on = enable != 0;
  });
}

const char* combo_profile_json(combo_ctx* c) {
  const int rc = guarded(c, [&] {
    COMBO_CK(cudaStreamSynchronize(c->stream));
    double ms[kNumTags] = {0}, bytes[kNumTags] = {0};
    int64_t n[kNumTags] = {0};
    for (const auto& r : c->prof) {
      float t = 0.f;
      COMBO_CK(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.tag] += double(t);
      bytes[r.tag] += r.bytes;
      ++n[r.tag];
    }
    std::ostringstream js;
    js << "{";
    bool first = true;
    for (int t = 0; t < kNumTags; ++t) {
      if (!n[t]) continue;
      char b[256];
      std::snprintf(b, sizeof b, "%s\"%s\":{\"launches\":%lld,\"ms\":%.6f,\"bytes\":%.6e}", first ? "" : ",",
                    kTagNames[t], (long long)n[t], ms[t], bytes[t]);
      js << b;
      first = false;
    }
    js << "}";
    c->prof_json = js.str();
  });
  if (rc) c->prof_json = "{}";
  return c->prof_json.c_str();
}

int combo_set_grid(combo_ctx* c, const int64_t dims[3], const double lengths[3]) {
  return guarded(c, [&] {
    on_ranks(c, [&](combo_ctx* r) {
      for (combo_ctx* m : members(r)) set_grid(m, dims, lengths);
    });
  });
}

// Slab decomposition along axis 0. Emulated: nranks ranks in
// this process on this context's device (member contexts sharing its
// stream; the transpose is a device copy) -- the decomposition-invariance
// test harness. Must precede combo_bind_materials.
int combo_ctx_set_virtual_ranks(combo_ctx* c, int nranks) {
  return guarded(c, [&] {
    if (nranks < 1) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "nranks must be >= 1");
    if (c->nccl || c->in_multi) throw ComboError(COMBO_ERR_STATE, "context already joined an NCCL decomposition");
    COMBO_CK(cudaStreamSynchronize(c->stream));
    c->vm.clear();
    c->R = nranks;
    c->q = 0;
    c->bound = false;
    for (int q = 1; q < nranks; ++q) {
      auto m = std::make_unique<combo_ctx>();
      m->device = c->device;
      m->num_sms = c->num_sms;
      m->stream = c->stream;
      m->own_stream = false;
      m->lead = c;
      m->R = nranks;
      m->q = q;
      ensure_scratch(m.get());
      c->vm.push_back(std::move(m));
    }
    if (c->has_grid) {
      const auto d = c->dims;
      const auto l = c->lengths;
      for (combo_ctx* m : members(c)) set_grid(m, d.data(), l.data());
    }
  });
}

// One rank per process: this context is rank `rank` of `nranks`; nccl_id is
// the 128-byte id from combo_nccl_unique_id on rank 0 (broadcast by the
// caller, e.g. over torch.distributed). Must precede combo_bind_materials.
int combo_ctx_set_ranks(combo_ctx* c, int nranks, int rank, const void* nccl_id) {
  return guarded(c, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "bad rank / nranks");
    if (!c->vm.empty()) throw ComboError(COMBO_ERR_STATE, "context hosts emulated ranks");
    if (c->in_multi) throw ComboError(COMBO_ERR_STATE, "context is a multi-GPU group (combo_ctx_create_multi)");
    if (nranks > 1 && !nccl_id) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "nccl_id required for nranks > 1");
    nccl_destroy(c);
    c->R = nranks;
    c->q = rank;
    c->bound = false;
    if (nranks > 1) nccl_init(c, nranks, rank, nccl_id);
    if (c->has_grid) {
      const auto d = c->dims;
      const auto l = c->lengths;
      set_grid(c, d.data(), l.data());
    }
  });
}

// Host-side layout introspection (no device work): the spectrum row offset
// of (component c, plane i, column j) on the slab side (side 0: i local to
// the rank's slab, j global) or the pencil side (side 1: i global, j local),
// and the cell range of chunk `block` of a slab of `nplanes` planes. Used by
// the multi-process CPU tests to drive the same layout through gloo.
int combo_slab_row(const int64_t dims[3], int nranks, int rank, int side, int64_t c, int64_t i, int64_t j,
                   int64_t* off) {
  if (!dims || !off || nranks < 1 || rank < 0 || rank >= nranks || dims[0] % nranks || dims[1] % nranks)
    return COMBO_ERR_BAD_ARGUMENT;
  SpecView v{};
  v.n1 = dims[0];
  v.n2 = dims[1];
  v.n3 = dims[2];
  v.n3c = dims[2] / 2 + 1;
  v.n3p = (v.n3c + 7) / 8 * 8;
  v.blocked = nranks > 1;
  v.swap = 1;  // the default layout (COMBO_SWAP=1)
  v.ni = dims[0] / nranks;
  v.nj = dims[1] / nranks;
  v.i0 = rank * v.ni;
  v.j0 = rank * v.nj;
  v.blk = 9 * v.ni * v.nj * v.n3p;
  v.cs = nranks > 1 ? v.ni * v.nj * v.n3p : v.n1 * v.n2 * v.n3p;
  v.si = v.n3p;  // j-major rows (COMBO_SWAP=1)
  v.sj = v.n1 * v.n3p;
  *off = c * v.cs + (side == 0 ? v.rowA(i, j) : v.rowB(i, j));
  return COMBO_OK;
}

int combo_chunk_range(const int64_t dims[3], int64_t nplanes, int64_t block, int64_t* beg, int64_t* end,
                      int64_t* nblocks) {
  if (!dims || nplanes < 1) return COMBO_ERR_BAD_ARGUMENT;
  const int64_t plane = dims[1] * dims[2];
  const int64_t cpp = (plane + kChunk - 1) / kChunk;
  if (nblocks) *nblocks = nplanes * cpp;
  if (block < 0 || block >= nplanes * cpp) return COMBO_ERR_BAD_ARGUMENT;
  const int64_t p = block / cpp, k = block - p * cpp;
  if (beg) *beg = p * plane + k * kChunk;
  if (end) *end = std::min(p * plane + (k + 1) * kChunk, (p + 1) * plane);
  return COMBO_OK;
}

int combo_ctx_ranks(const combo_ctx* c, int* nranks, int* rank, int* local_ranks, int64_t* i0, int64_t* ni) {
  if (!c) return COMBO_ERR_BAD_ARGUMENT;
  if (nranks) *nranks = c->R;
  if (rank) *rank = c->q;
  if (local_ranks) *local_ranks = int(1 + c->vm.size() + c->peers.size());
  const int64_t n = c->has_grid ? c->dims[0] / c->R : 0;
  if (i0) *i0 = int64_t(c->q) * n;
  if (ni) *ni = n;
  return COMBO_OK;
}

// CellMaterials::CellMaterials (cell_material.cpp:12-55)
}  // extern "C"

namespace {
// binding of one slab: kind / c_plus / normal3 point at the slab's first cell
static void bind_slab(combo_ctx* c, const int64_t dims[3], const double lengths[3], const uint8_t* kind,
                         const double* c_plus, const double* normal3, const combo_law* matrix,
                         const combo_law* inclusion, int combo, const combo_laminate_opts* lam, int mem) {
    if (!kind || !c_plus || !matrix || !inclusion) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "null argument");
    set_grid(c, dims, lengths);
    const int64_t N = c->N;
    combo_laminate_opts opts{0.0, 1e-10, 0.0, 50, 1, 0.0};
    if (lam) opts = *lam;
    // the grid arrays go to the device once (host callers) and the cell
    // binding runs there (bind.cu)
    DBuf<uint8_t> dk;
    DBuf<double> dc, dn;
    const uint8_t* kd = kind;
    const double* cd = c_plus;
    const double* nd = normal3;
    if (mem != COMBO_MEM_DEVICE) {
      dk.alloc(size_t(N));
      dc.alloc(size_t(N));
      COMBO_CK(cudaMemcpyAsync(dk.p, kind, size_t(N), cudaMemcpyHostToDevice, c->stream));
      COMBO_CK(cudaMemcpyAsync(dc.p, c_plus, size_t(N) * 8, cudaMemcpyHostToDevice, c->stream));
      kd = dk.p;
      cd = dc.p;
      if (normal3) {
        dn.alloc(size_t(3 * N));
        COMBO_CK(cudaMemcpyAsync(dn.p, normal3, size_t(3 * N) * 8, cudaMemcpyHostToDevice, c->stream));
        nd = dn.p;
      }
    }
    bind_cells_device(c, kd, cd, nd, combo, opts.c_min);
    c->t45.release();
    c->law_m = *matrix;
    c->law_i = *inclusion;
    c->lam = opts;
    double lo, hi;
    const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    spectrum_bounds(c, I, lo, hi);
    c->stress_floor = 1e-12 * std::max(hi, 1e-12);
    if (c->lam.stress_floor == 0.0) c->lam.stress_floor = c->stress_floor;
    c->a9.alloc(162);
    c->mp.law[0] = law_params(c->law_m, c->a9.p);
    c->mp.law[1] = law_params(c->law_i, c->a9.p + 81);
    c->mp.lam.tol_abs = c->lam.tol_abs;
    c->mp.lam.tol_rel = c->lam.tol_rel;
    c->mp.lam.stress_floor = c->lam.stress_floor;
    c->mp.lam.max_iter = c->lam.max_iter;
    c->mp.lam.back_projection = c->lam.back_projection;
    c->dfmg_warm.release();
    c->bound = true;
}
}  // namespace

extern "C" {

namespace {
// local: the arrays hold this process's slabs only (its ranks' planes, in
// rank order) instead of the whole grid
int bind_members(combo_ctx* c, const int64_t dims[3], const double lengths[3], const uint8_t* kind,
                 const double* c_plus, const double* normal3, const combo_law* matrix, const combo_law* inclusion,
                 int combo, const combo_laminate_opts* lam, int mem, bool local) {
  return guarded(c, [&] {
    if (!kind || !c_plus || !matrix || !inclusion) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "null argument");
    // a multi-GPU group's local slabs are the whole grid
    const int q0 = local && !c->multi ? c->q : 0;
    on_ranks(c, [&](combo_ctx* r) {
      for (combo_ctx* m : members(r)) {
        m->R = r->R;
        set_grid(m, dims, lengths);
        const int64_t off = int64_t(m->q - q0) * m->N;
        bind_slab(m, dims, lengths, kind + off, c_plus + off, normal3 ? normal3 + 3 * off : nullptr, matrix,
                  inclusion, combo, lam, mem);
      }
    });
    ++c->bind_gen;
  });
}
}  // namespace

// the arrays describe the whole grid; every rank binds its slab of planes
int combo_bind_materials(combo_ctx* c, const int64_t dims[3], const double lengths[3], const uint8_t* kind,
                         const double* c_plus, const double* normal3, const combo_law* matrix,
                         const combo_law* inclusion, int combo, const combo_laminate_opts* lam, int mem) {
  return bind_members(c, dims, lengths, kind, c_plus, normal3, matrix, inclusion, combo, lam, mem, false);
}

// the arrays hold this process's slabs (one rank per process: its own
// n1/R planes), e.g. from combo_generate_planes / combo_normals_slab
int combo_bind_materials_slab(combo_ctx* c, const int64_t dims[3], const double lengths[3], const uint8_t* kind,
                              const double* c_plus, const double* normal3, const combo_law* matrix,
                              const combo_law* inclusion, int combo, const combo_laminate_opts* lam, int mem) {
  return bind_members(c, dims, lengths, kind, c_plus, normal3, matrix, inclusion, combo, lam, mem, true);
}

int combo_bind_generation(const combo_ctx* c, int64_t* gen) {
  if (!c || !gen) return COMBO_ERR_BAD_ARGUMENT;
  *gen = c->bind_gen;
  return COMBO_OK;
}

int combo_composite_cells(const combo_ctx* c, int64_t* count) {
  if (!c || !count) return COMBO_ERR_BAD_ARGUMENT;
  *count = c->ncomp;  // emulated ranks / multi-GPU group: all slabs; one rank per process: this slab
  for (const auto& m : c->vm) *count += m->ncomp;
  for (const auto& m : c->peers) *count += m->ncomp;
  return COMBO_OK;
}

int combo_stress_floor(const combo_ctx* c, double* f) {
  if (!c || !f) return COMBO_ERR_BAD_ARGUMENT;
  *f = c->lam.stress_floor;
  return COMBO_OK;
}

int combo_spectrum_bounds(combo_ctx* c, const double fbar[9], double* lo, double* hi) {
  return guarded(c, [&] {
    require_bound(c);
    spectrum_bounds(c, fbar, *lo, *hi);
  });
}

int combo_get_warm_starts(combo_ctx* c, double* warm3, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    require_single(c);
    const int64_t n = c->ncomp;
    if (!n) return;
    std::vector<double> soa(size_t(3 * n));
    COMBO_CK(cudaMemcpy(soa.data(), c->warm.p, soa.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<double> aos(size_t(3 * n));
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) aos[size_t(3 * i + d)] = soa[size_t(d * n + i)];
    if (mem == COMBO_MEM_DEVICE)
      COMBO_CK(cudaMemcpy(warm3, aos.data(), aos.size() * 8, cudaMemcpyHostToDevice));
    else
      std::memcpy(warm3, aos.data(), aos.size() * 8);
  });
}

int combo_set_warm_starts(combo_ctx* c, const double* warm3, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    require_single(c);
    const int64_t n = c->ncomp;
    if (!n) return;
    std::vector<double> aos(size_t(3 * n));
    if (mem == COMBO_MEM_DEVICE)
      COMBO_CK(cudaMemcpy(aos.data(), warm3, aos.size() * 8, cudaMemcpyDeviceToHost));
    else
      std::memcpy(aos.data(), warm3, aos.size() * 8);
    std::vector<double> soa(size_t(3 * n));
    for (int64_t i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) soa[size_t(d * n + i)] = aos[size_t(3 * i + d)];
    COMBO_CK(cudaMemcpy(c->warm.p, soa.data(), soa.size() * 8, cudaMemcpyHostToDevice));
  });
}

int combo_reset_warm_starts(combo_ctx* c) {
  return guarded(c, [&] {
    require_bound(c);
    on_ranks(c, [](combo_ctx* r) {
      for (combo_ctx* m : members(r)) {
        if (m->ncomp) COMBO_CK(cudaMemsetAsync(m->warm.p, 0, size_t(3 * m->ncomp) * 8, m->stream));
        if (m->dfmg_warm.p) COMBO_CK(cudaMemsetAsync(m->dfmg_warm.p, 0, m->dfmg_warm.n * 8, m->stream));
      }
      COMBO_CK(cudaStreamSynchronize(r->stream));
    });
  });
}

int combo_get_stream(combo_ctx* c, void** stream) {
  if (!c || !stream) return COMBO_ERR_BAD_ARGUMENT;
  *stream = reinterpret_cast<void*>(c->stream);
  return COMBO_OK;
}

int combo_stress_sweep(combo_ctx* c, const double* F, double* P, combo_sweep_stats* st, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    require_single(c);
    ensure_scratch(c);
    const double* f = stage_in(c, F, mem, 0);
    double* p = stage_out(c, P, mem, 1);
    reset_stats(c);
    sweep(c, f, zero_shift(), 0.0, p, true, 0);
    fetch_results(c);
    finish_out(c, P, p, mem, size_t(9 * c->N));
    if (st) {
      const Stats* s = reinterpret_cast<const Stats*>(c->hres + 64);
      st->inadmissible_cells = int64_t(s->inadmissible);
      st->laminate_failures = int64_t(s->failures);
      st->back_projections = int64_t(s->backproj);
      st->laminate_iter_max = int64_t(s->iter_max);
    }
  });
}

// recover_phase_fields + phase_averages (postprocess.cpp:13-106)
int combo_phase_averages(combo_ctx* c, const double* F, combo_phase_avg* out, int mem) {
  return guarded(c, [&] {
    if (!out) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "null argument");
    require_bound(c);
    require_single(c);
    ensure_scratch(c);
    const double* f = stage_in(c, F, mem, 0);
    const size_t nc = size_t(std::max<int64_t>(c->ncomp, 1));
    DBuf<double> pp, pm;
    pp.alloc(9 * nc);
    pm.alloc(9 * nc);
    reset_stats(c);
    if (c->ncomp > 0) {
      const unsigned g = unsigned(std::min<int64_t>((c->ncomp + 127) / 128, int64_t(c->num_sms) * 64));
      k_recover<<<g, 128, 0, c->stream>>>(c->mp, c->cell_data(), f, c->N, pp.p, pm.p, stats_ptr(c));
      ++c->launches;
      COMBO_CK(cudaGetLastError());
    }
    const int64_t nb = chunk_blocks(c);
    double* part = part_ptr(c, nb, 20);
    k_phase_sum<<<unsigned(nb), kEwThreads, 0, c->stream>>>(c->mp, c->cell_data(), f, c->N, pp.p, pm.p,
                                                            chunks_of(c), part);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    group_reduce(c, nb, 20, 0);
    fetch_results(c);
    const Stats* st = reinterpret_cast<const Stats*>(c->hres + 64);
    if (st->inadmissible)
      throw ComboError(COMBO_ERR_INADMISSIBLE_MACRO, "recover_phase_fields: det F_box <= 0 in a composite cell");
    const double* r = c->hres;
    const double n = double(c->Ng);
    out->c_plus = r[9] / n;
    out->has_plus = r[9] > 0.0;
    out->has_minus = r[19] > 0.0;
    for (int q = 0; q < 9; ++q) {
      out->pbar_plus[q] = out->has_plus ? r[q] / r[9] : 0.0;
      out->pbar_minus[q] = out->has_minus ? r[10 + q] / r[19] : 0.0;
      out->pbar[q] = (r[q] + r[10 + q]) / n;
    }
    out->max_resolve_iterations = int32_t(st->iter_max);
  });
}

// recover_phase_fields per composite (postprocess.cpp:13-36) for
// interface_tractions (postprocess.cpp:114-141): component-major outputs by
// composite id, device or host buffers per `mem`
int combo_recover_composites(combo_ctx* c, const double* F, int64_t* cell, double* f_plus, double* f_minus,
                             double* traction, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    require_single(c);
    ensure_scratch(c);
    const double* f = stage_in(c, F, mem, 0);
    const size_t nc = size_t(std::max<int64_t>(c->ncomp, 1));
    if (c->ncomp == 0) return;
    if (!cell || !f_plus || !f_minus || !traction) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "null argument");
    DBuf<int64_t> dcell;
    DBuf<double> dfp, dfm, dtr;
    const bool host = mem == COMBO_MEM_HOST;
    int64_t* oc = cell;
    double *ofp = f_plus, *ofm = f_minus, *otr = traction;
    if (host) {
      dcell.alloc(nc);
      dfp.alloc(9 * nc);
      dfm.alloc(9 * nc);
      dtr.alloc(3 * nc);
      oc = dcell.p;
      ofp = dfp.p;
      ofm = dfm.p;
      otr = dtr.p;
    }
    reset_stats(c);
    const unsigned g = unsigned(std::min<int64_t>((c->ncomp + 127) / 128, int64_t(c->num_sms) * 64));
    k_recover_state<<<g, 128, 0, c->stream>>>(c->mp, c->cell_data(), f, c->N, oc, ofp, ofm, otr, stats_ptr(c));
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    fetch_results(c);
    const Stats* st = reinterpret_cast<const Stats*>(c->hres + 64);
    if (st->inadmissible)
      throw ComboError(COMBO_ERR_INADMISSIBLE_MACRO, "recover_phase_fields: det F_box <= 0 in a composite cell");
    if (host) {
      COMBO_CK(cudaMemcpy(cell, oc, nc * sizeof(int64_t), cudaMemcpyDeviceToHost));
      COMBO_CK(cudaMemcpy(f_plus, ofp, 9 * nc * sizeof(double), cudaMemcpyDeviceToHost));
      COMBO_CK(cudaMemcpy(f_minus, ofm, 9 * nc * sizeof(double), cudaMemcpyDeviceToHost));
      COMBO_CK(cudaMemcpy(traction, otr, 3 * nc * sizeof(double), cudaMemcpyDeviceToHost));
    }
  });
}

int combo_tangent_matvec(combo_ctx* c, const double* F, const double* x, double* y, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    require_single(c);
    const double* f = stage_in(c, F, mem, 0);
    const double* xx = stage_in(c, x, mem, 1);
    double* yy = stage_out(c, y, mem, 2);
    c->scratch[3].alloc(size_t(9 * c->N));
    comp_tangents(c, f, zero_shift());
    MatvecArgs a{c->mp, c->cell_data(), f, zero_shift(), xx, c->scratch[3].p, 0.0, 1, c->N, nullptr, 0.0};
    launch_matvec(c, a, yy);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    finish_out(c, y, yy, mem, size_t(9 * c->N));
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

int combo_tangent45(combo_ctx* c, const double* F, double* t45, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    require_single(c);
    const double* f = stage_in(c, F, mem, 0);
    DBuf<double> t;
    double* dt = t45;
    if (mem != COMBO_MEM_DEVICE) {
      t.alloc(size_t(45 * c->N));
      dt = t.p;
    }
    k_tangent45<<<ew_grid(c->N), kEwThreads, 0, c->stream>>>(c->mp, c->cell_data(), f, dt, c->N);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    finish_out(c, t45, dt, mem, size_t(45 * c->N));
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

int combo_tangent45_matvec(combo_ctx* c, const double* t45, const double* x, double* y, int mem) {
  return guarded(c, [&] {
    if (!c->has_grid) throw ComboError(COMBO_ERR_STATE, "no grid");
    DBuf<double> t;
    const double* dt = t45;
    if (mem != COMBO_MEM_DEVICE) {
      t.alloc(size_t(45 * c->N));
      COMBO_CK(cudaMemcpyAsync(t.p, t45, size_t(45 * c->N) * 8, cudaMemcpyHostToDevice, c->stream));
      dt = t.p;
    }
    const double* xx = stage_in(c, x, mem, 1);
    double* yy = stage_out(c, y, mem, 2);
    k_t45_matvec<<<ew_grid(c->N), kEwThreads, 0, c->stream>>>(dt, xx, yy, c->N);
    ++c->launches;
    COMBO_CK(cudaGetLastError());
    finish_out(c, y, yy, mem, size_t(9 * c->N));
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

// whole-grid [9][N] arrays <-> the slabs: slab k of rank r's members is
// rows [(r0 + k) Nl, ...) of every component, r0 = the multi-GPU rank
// (members of emulated ranks and single contexts: 0)
namespace {
struct SlabRows {
  int64_t Nl, Nt, r0;
};
SlabRows slab_rows(combo_ctx* r) {
  const int64_t nloc = int64_t(members(r).size());
  const int64_t R = r->in_multi ? r->R : nloc;
  return SlabRows{r->N, r->N * R, r->in_multi ? r->q : 0};
}
}  // namespace

int combo_project(combo_ctx* c, int kind, const double* in, double* out, int mem) {
  return guarded(c, [&] {
    if (!c->has_grid) throw ComboError(COMBO_ERR_STATE, "no grid (combo_set_grid)");
    // in / out: [9][N] of the grid (emulated ranks / multi-GPU group: split
    // into / gathered from the slabs; one rank per process: this rank's slab)
    on_ranks(c, [&](combo_ctx* r) {
      ensure_scratch(r);
      const auto ms = members(r);
      const SlabRows sr = slab_rows(r);
      const int64_t Nl = sr.Nl;
      const auto h2d = mem == COMBO_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
      const auto d2h = mem == COMBO_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      for (size_t k = 0; k < ms.size(); ++k) {
        ms[k]->scratch[0].alloc(size_t(9 * Nl));
        ms[k]->scratch[1].alloc(size_t(9 * Nl));
        COMBO_CK(cudaMemcpy2DAsync(ms[k]->scratch[0].p, size_t(Nl) * 8, in + (sr.r0 + int64_t(k)) * Nl,
                                   size_t(sr.Nt) * 8, size_t(Nl) * 8, 9, h2d, r->stream));
      }
      project_group(
          r, kind, [&](size_t k) { return ProdLoad9{ms[k]->scratch[0].p, Nl}; },
          [&](size_t k) { return ConsStore9{ms[k]->scratch[1].p, Nl}; }, 0);
      for (size_t k = 0; k < ms.size(); ++k)
        COMBO_CK(cudaMemcpy2DAsync(out + (sr.r0 + int64_t(k)) * Nl, size_t(sr.Nt) * 8, ms[k]->scratch[1].p,
                                   size_t(Nl) * 8, size_t(Nl) * 8, 9, d2h, r->stream));
      COMBO_CK(cudaStreamSynchronize(r->stream));
    });
  });
}

int combo_fft_forward(combo_ctx* c, const int64_t dims[3], int ncomp, const double* in, double* out, int mem) {
  return guarded(c, [&] {
    require_single(c);
    if (ncomp < 1 || ncomp > 9) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "ncomp must be 1..9");
    double L[3] = {1, 1, 1};
    if (c->has_grid) std::memcpy(L, c->lengths.data(), sizeof L);
    set_grid(c, dims, L);
    ensure_scratch(c);
    const int64_t N = c->N;
    c->scratch[0].alloc(size_t(9 * N));
    COMBO_CK(cudaMemsetAsync(c->scratch[0].p, 0, size_t(9 * N) * 8, c->stream));
    COMBO_CK(cudaMemcpyAsync(c->scratch[0].p, in, size_t(ncomp * N) * 8,
                             mem == COMBO_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    FftPlan& p = *c->plan;
    launch_zfwd(c, ProdLoad9{c->scratch[0].p, N});
    launch_y<false>(c);
    launch_x_plain<false>(c);
    // unpadded [c][i][j][k] copy out, one (c, i) plane of rows at a time
    const SpecView sv = p.sv();
    for (int64_t cc = 0; cc < ncomp; ++cc)
      for (int64_t i = 0; i < p.dims[0]; ++i)
        COMBO_CK(cudaMemcpy2DAsync(reinterpret_cast<char*>(out) + size_t((cc * p.dims[0] + i) * p.dims[1] * p.n3c) * 16,
                                   size_t(p.n3c) * 16, sv.spec + cc * sv.cs + i * sv.si, size_t(sv.sj) * 16,
                                   size_t(p.n3c) * 16, size_t(p.dims[1]),
                                   mem == COMBO_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                   c->stream));
    COMBO_CK(cudaStreamSynchronize(c->stream));
  });
}

int combo_solve(combo_ctx* c, const double fbar[9], const combo_solver_cfg* cfg, double* F_out, double* P_out,
                double pbar[9], combo_report** report, int mem) {
  return guarded(c, [&] {
    require_bound(c);
    if (!cfg || !fbar) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "null argument");
    // SolverConfig::validate (solver.cpp:277-284) + det check (:288-290)
    if (cfg->eval == COMBO_EVAL_DFMG && cfg->green != COMBO_GREEN_STAGGERED)
      throw ComboError(COMBO_ERR_CONFIG_INVALID,
                       "solver: dfmg material evaluation requires the staggered Green operator");
    if (cfg->load_steps < 1) throw ComboError(COMBO_ERR_CONFIG_INVALID, "solver: load_steps must be >= 1");
    if (!(cfg->tol_equilibrium > 0.0))
      throw ComboError(COMBO_ERR_CONFIG_INVALID, "solver: tol_equilibrium must be positive");
    if (!(hdet3(fbar) > 0.0)) throw ComboError(COMBO_ERR_INADMISSIBLE_MACRO, "solve: det(fbar) <= 0");
    auto rep = std::make_unique<combo_report>();
    on_ranks(c, [&](combo_ctx* r) {
      auto rr = std::make_unique<combo_report>();
      Solver s(r, *cfg);
      s.run(fbar, *rr);
      // outputs: [9][N] of the grid (emulated ranks / multi-GPU group
      // gathered in slab order); with one rank per process, its slab
      const SlabRows sr = slab_rows(r);
      auto gather = [&](double* out, std::vector<double*> src) {
        const auto kind = mem == COMBO_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        for (size_t k = 0; k < src.size(); ++k)
          COMBO_CK(cudaMemcpy2DAsync(out + (sr.r0 + int64_t(k)) * sr.Nl, size_t(sr.Nt) * 8, src[k],
                                     size_t(sr.Nl) * 8, size_t(sr.Nl) * 8, 9, kind, r->stream));
      };
      if (P_out) {
        std::vector<double*> p;
        for (size_t k = 0; k < s.nranks(); ++k) p.push_back(s.scratch(k));
        s.final_stress(p);
        gather(P_out, p);
      }
      if (F_out) {
        s.materialize();
        std::vector<double*> f;
        for (size_t k = 0; k < s.nranks(); ++k) f.push_back(s.F(k));
        gather(F_out, f);
      }
      COMBO_CK(cudaStreamSynchronize(r->stream));
      if (r == c) {  // every rank holds the same report and P-bar
        if (pbar) std::memcpy(pbar, s.pbar(), 9 * sizeof(double));
        rep = std::move(rr);
      }
    });
    rep->json = report_json(*rep);
    if (report)
      *report = rep.release();
  });
}

int combo_report_summary(const combo_report* r, int* success, int* bisections, int* nsteps, double* alpha,
                         double* seconds_total, int64_t* ls_total) {
  if (!r) return COMBO_ERR_BAD_ARGUMENT;
  if (success) *success = r->success ? 1 : 0;
  if (bisections) *bisections = r->bisections;
  if (nsteps) *nsteps = int(r->steps.size());
  if (alpha) *alpha = r->alpha;
  if (seconds_total) *seconds_total = r->seconds_total;
  if (ls_total) *ls_total = r->ls_total;
  return COMBO_OK;
}

int combo_report_step(const combo_report* r, int step, combo_step_info* info) {
  if (!r || !info || step < 0 || size_t(step) >= r->steps.size()) return COMBO_ERR_BAD_ARGUMENT;
  const auto& s = r->steps[size_t(step)];
  info->t_start = s.t_start;
  info->t_end = s.t_end;
  std::memcpy(info->fbar, s.fbar, sizeof s.fbar);
  info->converged = s.converged ? 1 : 0;
  info->outer_iters = s.outer_iters;
  info->cg_breakdowns = s.cg_breakdowns;
  info->line_search_cuts = s.line_search_cuts;
  info->n_residuals = int(s.residuals.size());
  info->sweep = s.sweep;
  info->seconds = s.seconds;
  info->ls_basic = s.ls_basic;
  info->ls_residual = s.ls_residual;
  info->ls_cg = s.ls_cg;
  info->ls_trial = s.ls_trial;
  return COMBO_OK;
}

int combo_report_step_history(const combo_report* r, int step, double* residuals, double* pbar9, int* cg_iters) {
  if (!r || step < 0 || size_t(step) >= r->steps.size()) return COMBO_ERR_BAD_ARGUMENT;
  const auto& s = r->steps[size_t(step)];
  for (size_t i = 0; i < s.residuals.size(); ++i) {
    if (residuals) residuals[i] = s.residuals[i];
    if (pbar9 && i < s.pbar_history.size()) std::memcpy(pbar9 + 9 * i, s.pbar_history[i].data(), 72);
  }
  if (cg_iters)
    for (size_t i = 0; i < s.cg_iters.size(); ++i) cg_iters[i] = s.cg_iters[i];
  return COMBO_OK;
}

const char* combo_report_json(const combo_report* r) { return r ? r->json.c_str() : "{}"; }

int combo_report_free(combo_report* r) {
  delete r;
  return COMBO_OK;
}

}  // extern "C"
