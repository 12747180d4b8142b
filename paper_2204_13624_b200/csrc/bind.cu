// Device-side CellMaterials binding (cell_material.cpp:12-55,
// laminate.cpp:28-34): kind / c_plus / normal per boxel -> cid (-1 matrix,
// -2 inclusion, >= 0 composite id in cell order), compact composite arrays
// (normal SoA, c+, c-, cell index). Composite ids come from an exclusive
// scan of the composite flags, so they are the same ids, in the same order,
// as a sequential host pass. Compiled with --fmad=false: the normalisation
// a / sqrt(a a + b b + d d) rounds exactly like the host expression.
#include <cub/device/device_scan.cuh>

#include "context.hpp"

namespace {

constexpr int kThreads = 256;

struct BindIn {
  const uint8_t* kind;
  const double* cp;
  const double* n3;  // AoS (3 per cell) or null
  int64_t N;
  int combo;
  double c_min;
};

__device__ __forceinline__ bool composite_cell(const BindIn& b, int64_t i) {
  if (b.kind[i] != 2) return false;
  const double cpl = b.cp[i];
  return b.combo && cpl >= b.c_min && 1.0 - cpl >= b.c_min;
}

// flags[i] = composite; first offending cell per error kind (ComboMeta::make)
__global__ void k_bind_flags(BindIn b, int32_t* flags, unsigned long long* err) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < b.N; i += int64_t(gridDim.x) * blockDim.x) {
    const bool f = composite_cell(b, i);
    flags[i] = f ? 1 : 0;
    if (!f) continue;
    const double cpl = b.cp[i];
    if (!(cpl > 0.0) || !(cpl < 1.0)) {
      atomicMin(&err[0], (unsigned long long)i);
      continue;
    }
    if (!b.n3) {
      atomicMin(&err[1], (unsigned long long)i);
      continue;
    }
    const double x = b.n3[3 * i], y = b.n3[3 * i + 1], z = b.n3[3 * i + 2];
    const double len = sqrt(x * x + y * y + z * z);
    if (!(len > 0.0)) atomicMin(&err[1], (unsigned long long)i);
  }
}

__global__ void k_bind_write(BindIn b, const int32_t* flags, const int32_t* ids, int64_t nc, int32_t* cid,
                             int64_t* ccell, double* nrm, double* cp, double* cm) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < b.N; i += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t k = b.kind[i];
    if (k == 0) {
      cid[i] = -1;
    } else if (k == 1) {
      cid[i] = -2;
    } else if (!flags[i]) {
      cid[i] = b.cp[i] >= 0.5 ? -2 : -1;  // composite below c_min (or combo off): majority phase
    } else {
      const int32_t id = ids[i];
      cid[i] = id;
      ccell[id] = i;
      const double x = b.n3[3 * i], y = b.n3[3 * i + 1], z = b.n3[3 * i + 2];
      const double len = sqrt(x * x + y * y + z * z);
      nrm[id] = x / len;
      nrm[nc + id] = y / len;
      nrm[2 * nc + id] = z / len;
      cp[id] = b.cp[i];
      cm[id] = 1.0 - b.cp[i];
    }
  }
}

int grid_for(const combo_ctx* c, int64_t n) {
  const int64_t b = (n + kThreads - 1) / kThreads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(c->num_sms) * 16)));
}

}  // namespace

namespace combo_host {

// kind / cp / n3 are device pointers to this slab's N boxels
void bind_cells_device(combo_ctx* c, const uint8_t* kind, const double* cp, const double* n3, int combo,
                       double c_min) {
  const int64_t N = c->N;
  if (N >= (int64_t(1) << 31)) throw ComboError(COMBO_ERR_BAD_ARGUMENT, "bind: more than 2^31 boxels per slab");
  const BindIn b{kind, cp, n3, N, combo, c_min};
  DBuf<int32_t> flags, ids;
  DBuf<unsigned long long> err;
  flags.alloc(size_t(N));
  ids.alloc(size_t(N));
  err.alloc(2);
  COMBO_CK(cudaMemsetAsync(err.p, 0xff, 2 * sizeof(unsigned long long), c->stream));
  k_bind_flags<<<grid_for(c, N), kThreads, 0, c->stream>>>(b, flags.p, err.p);
  ++c->launches;
  COMBO_CK(cudaGetLastError());
  size_t tmp = 0;
  COMBO_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flags.p, ids.p, int(N), c->stream));
  DBuf<unsigned char> tbuf;
  tbuf.alloc(std::max<size_t>(tmp, 1));
  COMBO_CK(cub::DeviceScan::ExclusiveSum(tbuf.p, tmp, flags.p, ids.p, int(N), c->stream));
  unsigned long long herr[2];
  int32_t last[2];
  COMBO_CK(cudaMemcpyAsync(herr, err.p, sizeof(herr), cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaMemcpyAsync(&last[0], ids.p + (N - 1), 4, cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaMemcpyAsync(&last[1], flags.p + (N - 1), 4, cudaMemcpyDeviceToHost, c->stream));
  COMBO_CK(cudaStreamSynchronize(c->stream));
  // the host pass throws at the first offending cell in cell order
  if (herr[0] != ~0ull || herr[1] != ~0ull) {
    if (herr[0] < herr[1])
      throw ComboError(COMBO_ERR_BAD_ARGUMENT, "ComboMeta: volume fraction must lie in (0,1)");
    throw ComboError(COMBO_ERR_BAD_ARGUMENT, "ComboMeta: zero normal");
  }
  const int64_t nc = int64_t(last[0]) + int64_t(last[1]);
  c->ncomp = nc;
  c->cid.alloc(size_t(N));
  const size_t ncap = size_t(std::max<int64_t>(nc, 1));
  c->nrm.alloc(3 * ncap);
  c->cp.alloc(ncap);
  c->cm.alloc(ncap);
  c->warm.alloc(3 * ncap);
  c->ccell.alloc(ncap);
  k_bind_write<<<grid_for(c, N), kThreads, 0, c->stream>>>(b, flags.p, ids.p, nc, c->cid.p, c->ccell.p, c->nrm.p,
                                                          c->cp.p, c->cm.p);
  ++c->launches;
  COMBO_CK(cudaGetLastError());
  COMBO_CK(cudaMemsetAsync(c->warm.p, 0, 3 * ncap * 8, c->stream));
  COMBO_CK(cudaStreamSynchronize(c->stream));
}

}  // namespace combo_host
