// TMA-staged column-strip passes (x + Gamma, y) for power-of-two lines.
//
// The register-resident passes of fft_rr.cuh fetch their tile with 8-24
// 16-byte loads per thread; every warp load touches eight 64-byte row
// segments, so the LSU / L1 miss path, not HBM, bounds the load phase
// (x + Gamma: 0.53-0.57 of the copy bandwidth, top stall long_scoreboard).
// Here one thread moves the whole [components][N rows][W columns] tile with
// cp.async.bulk.tensor (a 4-D tensor map over the spectrum: column, the two
// row indices, component) into shared memory, completing on an mbarrier;
// the transform's first stage reads its operands from shared memory, the
// stage exchanges reuse the same buffer in place, and the outputs go back
// through the buffer with one bulk tensor store. Two blocks per SM alternate
// their load / compute / store phases.
//
// The arithmetic (stage order, twiddles, Gamma projection) is the one of
// xgamma_v4 / ypass_rr, so results are bitwise identical to them.
#pragma once

#include <cuda.h>

#include "fft_rr.cuh"
#include "stage.cuh"

namespace combo_dev {

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// generic-proxy shared-memory writes -> visible to the async proxy (TMA store)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Tile geometry shared by host and device: tensor coordinates are (column in
// doubles, row a, row b, component) with the transformed row index first
// when `lineFirst` (its stride is the smaller one) -- see make_strip_map.
constexpr int kTmaW = 4;  // columns (complex) per tile: 64-byte rows

// rows of one bulk tensor copy (box dims are limited to 256)
template <int N>
struct TmaRows {
  static constexpr int RB = N < 256 ? N : 256;
  static constexpr int NB = N / RB;
};

// ------------------------------------------------------------ X + Gamma
// Tile: 3 components (Gamma row group rg) x N rows (k1) x W columns of one
// k2 = j. Shared buffer: [box b][component][RB rows][W] double2 for the
// input and output, 2 x (N + N/8) x W for the in-place stage exchanges.
template <int L, int KIND>
static __global__ void __launch_bounds__((1 << L) / 8 * kTmaW, (1 << L) <= 512 ? 2 : 1)
    xgamma_tma(const __grid_constant__ CUtensorMap map, SpecView sv, const double2* __restrict__ tw, GreenTables G,
               int lineFirst) {
  constexpr int N = 1 << L, W = kTmaW, RB = TmaRows<N>::RB, NB = TmaRows<N>::NB;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar;
  const int rg = blockIdx.z, j = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  const bool active = line < w;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map);
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, uint32_t(3 * N * W * sizeof(double2)));
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (lineFirst)
        tma_load_4d(sm + b * 3 * RB * W, &map, &bar, 2 * kc0, b * RB, j, 3 * rg);
      else
        tma_load_4d(sm + b * 3 * RB * W, &map, &bar, 2 * kc0, j, b * RB, 3 * rg);
    }
  }
  const RankCol<KIND> col = rank_col<KIND>(G, rg, sv.j0 + j, kc0 + line, sv.n2, sv.n3);
  __syncthreads();  // barrier initialised before anyone polls it
  mbar_wait(&bar, 0);
  auto tile = [&](int comp, int pos) { return ((pos / RB * 3 + comp) * RB + pos % RB) * W + line; };
  double2 v[2][8];
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int pos = rr_first_pos<L, false>(u, q);
      v[0][q] = sm[tile(0, pos)];
      const double2 a = cmulc(col.o1, sm[tile(1, pos)]), b = cmulc(col.o2, sm[tile(2, pos)]);
      v[1][q] = make_double2(a.x + b.x, a.y + b.y);
    }
  }
  __syncthreads();  // the exchanges below overwrite the input tile
  constexpr int chs = (N + N / 8) * W;
  auto addr = [&](int ch, int pos) { return ch * chs + pad8(pos) * W + line; };
  rr_stages<L, false, false, 0, 2>(v, u, active, sm, tw, addr);
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) rank_gamma<KIND>(G, col, rg, rr_final_pos<L, false>(u, q), sv.n1, v[0][q], v[1][q]);
  }
  rr_stages<L, true, true, 0, 2>(v, u, active, sm, tw, addr);
  // every thread is past the last exchange barrier: the buffer is free
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int pos = rr_final_pos<L, true>(u, q);
      sm[tile(0, pos)] = v[0][q];
      sm[tile(1, pos)] = cmul(col.o1, v[1][q]);
      sm[tile(2, pos)] = cmul(col.o2, v[1][q]);
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (lineFirst)
        tma_store_4d(&map, sm + b * 3 * RB * W, 2 * kc0, b * RB, j, 3 * rg);
      else
        tma_store_4d(&map, sm + b * 3 * RB * W, 2 * kc0, j, b * RB, 3 * rg);
    }
    tma_store_commit_wait();
  }
}

// ------------------------------------------------------------------ Y pass
// Tile: N rows (k2) x W columns of component c on local plane i (box
// component extent 1). Same buffer discipline as above with one channel.
template <int L, bool INV, int W>
static __global__ void __launch_bounds__((1 << L) / 8 * W, ((1 << L) / 8 * W) <= 256 ? 4 : 2)
    ypass_tma(const __grid_constant__ CUtensorMap map, SpecView sv, const double2* __restrict__ tw, int lineFirst) {
  constexpr int N = 1 << L, RB = TmaRows<N>::RB, NB = TmaRows<N>::NB;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ uint64_t bar;
  const int c = blockIdx.z, i = blockIdx.y, kc0 = blockIdx.x * W;
  const int w = min(W, int(sv.n3c) - kc0);
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  const bool active = line < w;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&map);
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, uint32_t(N * W * sizeof(double2)));
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (lineFirst)
        tma_load_4d(sm + b * RB * W, &map, &bar, 2 * kc0, b * RB, i, c);
      else
        tma_load_4d(sm + b * RB * W, &map, &bar, 2 * kc0, i, b * RB, c);
    }
  }
  __syncthreads();  // barrier initialised before anyone polls it
  mbar_wait(&bar, 0);
  double2 v[1][8];
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) v[0][q] = sm[rr_first_pos<L, false>(u, q) * W + line];
  }
  __syncthreads();  // the exchanges below overwrite the input tile
  auto addr = [&](int, int pos) { return pad8(pos) * W + line; };
  rr_stages<L, INV, false, 0, 1>(v, u, active, sm, tw, addr);
  if (active) {
#pragma unroll
    for (int q = 0; q < 8; ++q) sm[rr_final_pos<L, false>(u, q) * W + line] = v[0][q];
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (lineFirst)
        tma_store_4d(&map, sm + b * RB * W, 2 * kc0, b * RB, i, c);
      else
        tma_store_4d(&map, sm + b * RB * W, 2 * kc0, i, b * RB, c);
    }
    tma_store_commit_wait();
  }
}

}  // namespace combo_dev
