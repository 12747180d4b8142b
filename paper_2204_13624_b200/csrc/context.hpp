// Host-side context of the B200 ComBo engine (one device, one stream).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/combo_cuda.h"
#include "fft.cuh"
#include "kernels.cuh"
#include "material.cuh"

namespace combo_host {

struct ComboError : std::exception {
  int code;
  std::string msg;
  ComboError(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

#define COMBO_CK(x)                                                                                     \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess)                                                                              \
      throw ::combo_host::ComboError(e_ == cudaErrorMemoryAllocation ? COMBO_ERR_OOM : COMBO_ERR_CUDA, \
                                     std::string(#x) + ": " + cudaGetErrorString(e_));                  \
  } while (0)

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    if (count == 0) return;
    COMBO_CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
};

struct AxisPlan {
  int n = 1;
  std::vector<int> rad;
  DBuf<double2> tw;
  combo_dev::Axis view() const {
    combo_dev::Axis a{};
    a.n = n;
    a.nrad = int(rad.size());
    for (size_t i = 0; i < rad.size(); ++i) a.rad[i] = rad[i];
    a.tw = tw.p;
    return a;
  }
};

struct GreenPlan {
  int kind = -1;
  DBuf<double2> fwd[3], avg[3];
  DBuf<double> xi[3];
};

// FFT + Gamma plan for one grid
struct FftPlan {
  std::array<int64_t, 3> dims{0, 0, 0};
  std::array<double, 3> lengths{1, 1, 1};
  int64_t n3c = 0, n3p = 0;
  AxisPlan ax[3];
  GreenPlan green[3];
  int zL = 1, zls = 1, zT = 32;  // z pass: lines per block, line stride, threads
  int yW = 8, yT = 32;           // y pass tile width, threads
  int xW = 8, xT = 32;           // x pass tile width (3 components per tile)
  size_t zsmem = 0, ysmem = 0, xsmem = 0;
  // register-resident pow2 path (fft_rr.cuh), used when the axis length is
  // a power of two >= 8
  int rzL = 1, rzT = 32, ryW = 8, ryT = 32, rxW = 4, rxT = 32;
  size_t rzsmem = 0, rysmem = 0, rxsmem = 0;
  int xminb = 2;  // xgamma_v4 blocks per SM (launch bound)
  bool split_sweep = true;  // composite Newton pass + pure streaming pass (COMBO_SPLIT_SWEEP=0: one pass)
  bool mv_bulk = true;  // bulk-staged CG matvec (COMBO_MV_BULK=0: one cell per thread, direct loads)
  bool swap = false;  // j-major spectrum rows (see SpecView), COMBO_SWAP=1
  bool pq_dot = true;    // CG: pdir^T A pdir summed in the matvec (COMBO_PQ=0: in the z-inverse consumer)
  // TMA-staged column-strip passes (fft_tma.cuh): tensor maps over `spec`
  // (single slab, power-of-two axes); COMBO_XTMA / COMBO_YTMA = 0 turn them off
  // persistent ring-staged z-inverse at n3 = 512 (two consumer groups; COMBO_ZRING=0: one block per
  // tile), used for consumers whose epilogue reads no field (Cons::LOADS)
  int zring = 2;
  bool tma_x = false, tma_y = false;
  int tma_x_line_first = 1, tma_y_line_first = 0, tma_yw = 8;
  CUtensorMap xmap{}, ymap{};
  // slab decomposition (R ranks, this plan's rank q): planes [i0, i0 + ni)
  // on the slab side, k2 in [j0, j0 + nj) on the pencil side
  int R = 1, q = 0;
  int64_t ni = 0, nj = 0, i0 = 0, j0 = 0;
  DBuf<double2> spec;   // slab side (z, y passes)
  DBuf<double2> specB;  // pencil side (x pass + Gamma), R > 1 only
  combo_dev::SpecView sv() const {
    combo_dev::SpecView s;
    s.spec = spec.p;
    s.n1 = dims[0];
    s.n2 = dims[1];
    s.n3 = dims[2];
    s.n3c = n3c;
    s.n3p = n3p;
    s.blocked = R > 1 ? 1 : 0;
    s.swap = swap ? 1 : 0;
    s.ni = ni;
    s.nj = nj;
    s.i0 = i0;
    s.j0 = j0;
    s.blk = 9 * ni * nj * n3p;
    s.cs = R > 1 ? ni * nj * n3p : dims[0] * dims[1] * n3p;
    s.si = swap ? n3p : dims[1] * n3p;
    s.sj = swap ? dims[0] * n3p : n3p;
    return s;
  }
  combo_dev::SpecView svB() const {
    combo_dev::SpecView s = sv();
    if (R > 1) s.spec = specB.p;
    return s;
  }
};

struct StepRec {
  double t_start = 0, t_end = 0;
  double fbar[9] = {0};
  bool converged = false;
  int outer_iters = 0;
  std::vector<double> residuals;
  std::vector<int> cg_iters;
  std::vector<std::array<double, 9>> pbar_history;
  int cg_breakdowns = 0;
  int line_search_cuts = 0;
  combo_sweep_stats sweep{0, 0, 0, 0};
  double seconds = 0;
  int64_t ls_basic = 0, ls_residual = 0, ls_cg = 0, ls_trial = 0;
};

}  // namespace combo_host

struct combo_report {
  std::vector<combo_host::StepRec> steps;
  bool success = false;
  std::string error;
  int bisections = 0;
  double alpha = 0;
  double seconds_total = 0;
  int64_t ls_total = 0;
  std::string json;
};

struct combo_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;

  // grid (set by combo_set_grid / combo_bind_materials)
  bool has_grid = false;
  std::array<int64_t, 3> dims{0, 0, 0};
  std::array<double, 3> lengths{1, 1, 1};
  int64_t N = 0;   // cells of this context's slab
  int64_t Ng = 0;  // cells of the whole grid

  // slab decomposition (combo_ctx_set_ranks / combo_ctx_set_virtual_ranks):
  // R ranks along axis 0, this context is rank q. Emulated ranks live in one
  // process on one device as member contexts of the leader (vm) and share
  // its stream; with one rank per process the exchange runs over NCCL.
  int R = 1, q = 0;
  combo_ctx* lead = nullptr;                   // group leader (nullptr: self)
  std::vector<std::unique_ptr<combo_ctx>> vm;  // emulated ranks 1..R-1
  void* nccl = nullptr;                        // ncclComm_t (one rank per process / per peer)
  // single-process multi-GPU (combo_ctx_create_multi): rank 0 owns the
  // contexts of ranks 1..R-1 on the other devices; every API call runs
  // each rank's part on a host thread of its own over the peers' NCCL clique
  std::vector<std::unique_ptr<combo_ctx>> peers;
  bool multi = false;     // this context owns peers
  bool in_multi = false;  // rank of a single-process multi-GPU group (outputs are whole-grid arrays)
  bool own_stream = true;
  // pipelined projection (R > 1): transposes of one Gamma row group run on
  // comm_stream while the passes of the next group run on stream
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t pipe_ev[12] = {nullptr};
  combo_host::DBuf<double> gpart;              // leader: block partials of all ranks
  combo_host::DBuf<double> gpart2;             // leader: chunk sums of long partial vectors
  combo_host::DBuf<combo_dev::Stats> gstats;   // NCCL: laminate stats of all ranks
  std::unique_ptr<combo_host::FftPlan> plan;

  // materials (combo_bind_materials)
  bool bound = false;
  int64_t bind_gen = 0;  // bumped by every binding (stale CellMaterials handles)
  combo_law law_m{}, law_i{};
  combo_laminate_opts lam{};
  double stress_floor = 1e-300;
  combo_host::DBuf<int32_t> cid;
  combo_host::DBuf<double> nrm, cp, cm, warm;
  combo_host::DBuf<int64_t> ccell;  // composite id -> cell
  combo_host::DBuf<double> t45;     // [45][ncomp] packed composite tangents
  int64_t ncomp = 0;
  combo_dev::MatParams mp{};
  combo_host::DBuf<double> a9;  // linear-law 9x9 tangents (device)
  combo_host::DBuf<double> dfmg_warm;  // [3][8 ncomp] per doubly-fine cell of a composite host
  combo_host::DBuf<double> dfmg_pd;    // [9][8][N] per-dfc stress / tangent products
  combo_host::DBuf<double> dfmg_t8;    // [45][8 ncomp] per-dfc packed tangents
  combo_host::DBuf<double> halo[3];    // axis-0 neighbour planes (DFMG: F above, pd below, pdir above)
  combo_host::DBuf<double> halo_send;  // NCCL: packed boundary plane

  // scratch
  combo_host::DBuf<double> partials;   // per-block partial sums
  combo_host::DBuf<double> dres;       // reduced scalars (64 slots)
  combo_host::DBuf<combo_dev::Stats> dstats;
  double* hres = nullptr;              // pinned mirror of dres + stats
  combo_host::DBuf<double> scratch[4];  // operator-level staging (9N each)
  // solver field slots (9N each), kept resident across solve() calls so a
  // solve does not pay cudaMalloc/cudaFree of ~8 fields (77 GB at 512^3)
  combo_host::DBuf<double> solver_fields[8];

  // CUDA-event profiling of every kernel launch (combo_profile_*)
  struct ProfRec {
    int tag;
    cudaEvent_t a, b;
    double bytes;
  };
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  std::string prof_json;

  combo_dev::CellData cell_data() const {
    combo_dev::CellData c;
    c.cid = cid.p;
    c.nrm = nrm.p;
    c.cp = cp.p;
    c.cm = cm.p;
    c.warm = warm.p;
    c.ncomp = ncomp;
    c.ccell = ccell.p;
    c.t45 = t45.p;
    return c;
  }
};

namespace combo_host {
// operator-level entry points act on one slab
inline void require_single(const combo_ctx* c) {
  if (c->R > 1)
    throw ComboError(COMBO_ERR_STATE, "operator-level entry points need a single-slab context (R = 1)");
}
// comm.cu: NCCL (loaded at run time) for one-rank-per-process decompositions
void nccl_init(combo_ctx* c, int nranks, int rank, const void* uid);
void nccl_init_all(const std::vector<combo_ctx*>& ranks);  // ncclCommInitAll over the ranks' devices
void nccl_abort(combo_ctx* c);
void nccl_destroy(combo_ctx* c);
void nccl_allgather_inplace(combo_ctx* c, double* buf, size_t count_per_rank);
void nccl_allreduce_u64(combo_ctx* c, const unsigned long long* in, unsigned long long* out, size_t n, bool max);
void nccl_alltoall_blocks(combo_ctx* c, const double2* src, double2* dst, size_t blk, size_t off, size_t cnt,
                          cudaStream_t stream);
void nccl_allreduce_sum(combo_ctx* c, double* buf, size_t n);
// engine.cu
void set_grid(combo_ctx* c, const int64_t* dims, const double* lengths);
int ew_grid(int64_t n);
void ensure_scratch(combo_ctx* c);
void reduce_partials(combo_ctx* c, int64_t nblocks, int nred, int slot);
// dres (+ laminate stats, combined over NCCL ranks when with_stats) -> hres (sync)
void fetch_results(combo_ctx* c, bool with_stats = true);
combo_dev::LawP law_params(const combo_law& L, double* dev_a9);
void ensure_partials(combo_ctx* c, int64_t count);
// dfmg.cu
// (over every rank hosted by the leader c; vectors: one field per rank)
void dfmg_sweep(combo_ctx* c, const std::vector<const double*>& fin, const combo_dev::Shift9& sh, double alpha,
                const std::vector<double*>& out, int slot);
void dfmg_tangent_prepare(combo_ctx* c, const std::vector<const double*>& fin, const combo_dev::Shift9& sh);
void dfmg_matvec(combo_ctx* c, const std::vector<const double*>& fin, const combo_dev::Shift9& sh,
                 const std::vector<const double*>& r, const std::vector<double*>& pdir, double beta, bool first,
                 const std::vector<double*>& q);
// engine.cu: slab-decomposition helpers
combo_ctx* leader(combo_ctx* c);
std::vector<combo_ctx*> members(combo_ctx* c);
double* part_ptr(combo_ctx* c, int64_t nb, int nred);
combo_dev::Stats* stats_ptr(combo_ctx* c);
void group_reduce(combo_ctx* c, int64_t nb, int nred, int slot);
combo_dev::Chunks chunks_of(const combo_ctx* c);
int64_t chunk_blocks(const combo_ctx* c);
// comm.cu: send count doubles to rank `to` and receive as many from `from`
void nccl_sendrecv(combo_ctx* c, const double* send, int to, double* recv, int from, size_t count);

// kernel tags for the profiler
enum ProfTag {
  kTagSweep, kTagMatvec, kTagZfwd, kTagYfwd, kTagXGamma, kTagYinv, kTagZinv, kTagCgUpdate, kTagTrial,
  kTagMaterialize, kTagReduce, kTagOther, kTagMvZfwd, kTagExchange, kNumTags
};
// RAII: records CUDA events around the launches in its scope when enabled
struct ProfScope {
  combo_ctx* c;
  int idx = -1;
  cudaStream_t st = nullptr;
  ProfScope(combo_ctx* ctx, int tag, double bytes, cudaStream_t stream = nullptr);
  ~ProfScope();
};
// device-side CellMaterials binding of one slab (bind.cu)
void bind_cells_device(combo_ctx* c, const uint8_t* kind, const double* cp, const double* n3, int combo,
                       double c_min);
}  // namespace combo_host
