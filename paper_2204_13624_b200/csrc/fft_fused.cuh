// Plane-pipelined Z/Y passes: the z and y transforms of one x-plane run back
// to back inside one persistent kernel, so the spectrum rows the first pass
// writes are still in L2 when the second pass reads them.
//
// z and y lines both lie inside x-planes (storage axis 0), so the two passes
// of a plane are independent of every other plane. Work items are claimed in
// a fixed global order from a ticket counter:
//   forward  Z(0) | Z(1) Y(0) | Z(2) Y(1) | ... | Y(n-1)
//   inverse  Y(0) | Y(1) Z(0) | Y(2) Z(1) | ... | Z(n-1)
// A tile of the second pass of plane i waits until every tile of the first
// pass of plane i has completed (per-plane counters; all of them were
// claimed earlier by running blocks, so the wait cannot deadlock). At most
// about two planes of spectrum (2 x 19.5 MB at 512^3) are live in L2.
//
// Forward: the z pass writes the half spectrum of plane i, the y pass
// transforms it in place from L2; one write-back reaches HBM. Inverse: the y
// pass transforms the plane in place, the z pass reads it back from L2 and
// then discards the rows (dead after the c2r), so neither the y output nor
// the z input touches HBM. Per LS iteration this removes 4 of the 10
// spectrum-sized HBM transfers of the five separate passes.
//
// Results are bitwise those of the separate passes (same tile functions,
// same partial-sum slots).
#pragma once

#include "fft_rr.cuh"

namespace combo_dev {

#ifndef COMBO_FUSED_MINB
#define COMBO_FUSED_MINB 2
#endif
#ifndef COMBO_FUSED_T
#define COMBO_FUSED_T 320
#endif
constexpr int kFusedThreads = COMBO_FUSED_T, kFusedMinBlocks = COMBO_FUSED_MINB;

struct PlaneSched {
  unsigned* ticket;  // work-item counter (zeroed before the launch)
  unsigned* done;    // per local plane: completed first-pass tiles (zeroed)
  int64_t nplanes;   // local planes
  int nz;            // z tiles per plane (rzL lines each)
  int nyk;           // y column groups per plane
  int zl;            // z-lines per z tile
  int wy;            // y columns per tile
  int discard;       // inverse: drop the consumed spectrum rows from L2
};

// item t -> (second pass?, plane, tile within the plane's pass)
__device__ __forceinline__ void sched_item(const PlaneSched& s, int64_t t, int n_first, int n_second, bool& second,
                                           int64_t& plane, int64_t& tile) {
  if (t < n_first) {
    second = false;
    plane = 0;
    tile = t;
    return;
  }
  const int64_t tt = t - n_first, pair = n_first + n_second;
  const int64_t i = tt / pair, r = tt - i * pair;
  if (i + 1 < s.nplanes && r < n_first) {
    second = false;
    plane = i + 1;
    tile = r;
  } else {
    second = true;
    plane = i;
    tile = i + 1 < s.nplanes ? r - n_first : r;
  }
}

__device__ __forceinline__ int64_t claim(unsigned* ticket) {
  __shared__ int64_t item;
  __syncthreads();  // the previous item is finished with shared memory
  if (threadIdx.x == 0) item = int64_t(atomicAdd(ticket, 1u));
  __syncthreads();
  return item;
}

__device__ __forceinline__ void wait_plane(const unsigned* done, int64_t plane, unsigned need) {
  if (threadIdx.x == 0) {
    const volatile unsigned* d = done + plane;
    while (*d < need) __nanosleep(128);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void finish_tile(unsigned* done, int64_t plane) {
  __threadfence();  // this thread's stores of the tile are visible device-wide
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(done + plane, 1u);
}

// the tiles are separate (non-inlined) functions: each keeps the register
// allocation of its stand-alone kernel instead of the union of both
template <class Prod, int L>
__device__ __noinline__ void zfwd_tile_nc(SpecView sv, const double2* __restrict__ tw, int64_t line0, int nl,
                                          Prod prod) {
  zfwd_tile<Prod, L>(sv, tw, line0, nl, prod);
}
template <int L, bool INV, bool CG>
__device__ __noinline__ void ypass_tile_nc(SpecView sv, const double2* __restrict__ tw, int W, int c, int64_t i,
                                           int kc0) {
  ypass_tile<L, INV, CG>(sv, tw, W, c, i, kc0);
}
template <class Cons, int L>
__device__ __noinline__ void zinv_tile_nc(SpecView sv, const double2* __restrict__ tw, int64_t line0, int nl,
                                          double scale, Cons cons, double* partials, int64_t slot, bool discard) {
  zinv_tile<Cons, L, true, true>(sv, tw, line0, nl, scale, cons, partials, slot, discard);
}

template <class Prod, int LZ, int LY>
static __global__ void __launch_bounds__(kFusedThreads, kFusedMinBlocks)
    zy_fwd_fused(SpecView sv, const double2* __restrict__ twz, const double2* __restrict__ twy, Prod prod,
                 PlaneSched s) {
  const int ny = 9 * s.nyk;
  const int64_t total = s.nplanes * (s.nz + ny);
  for (;;) {
    const int64_t t = claim(s.ticket);
    if (t >= total) return;
    bool second;
    int64_t plane, tile;
    sched_item(s, t, s.nz, ny, second, plane, tile);
    if (!second) {
      zfwd_tile<Prod, LZ>(sv, twz, plane * sv.n2 + tile * s.zl, s.zl, prod);
      finish_tile(s.done, plane);
    } else {
      wait_plane(s.done, plane, unsigned(s.nz));
      const int c = int(tile / s.nyk), kt = int(tile - int64_t(c) * s.nyk);
      ypass_tile<LY, false, true>(sv, twy, s.wy, c, plane, kt * s.wy);
    }
  }
}

template <class Cons, int LZ, int LY>
static __global__ void __launch_bounds__(kFusedThreads, kFusedMinBlocks)
    yz_inv_fused(SpecView sv, const double2* __restrict__ twz, const double2* __restrict__ twy, double scale,
                 Cons cons, double* partials, PlaneSched s) {
  const int ny = 9 * s.nyk;
  const int64_t total = s.nplanes * (s.nz + ny);
  for (;;) {
    const int64_t t = claim(s.ticket);
    if (t >= total) return;
    bool second;
    int64_t plane, tile;
    sched_item(s, t, ny, s.nz, second, plane, tile);
    if (!second) {
      const int c = int(tile / s.nyk), kt = int(tile - int64_t(c) * s.nyk);
      ypass_tile<LY, true, false>(sv, twy, s.wy, c, plane, kt * s.wy);
      finish_tile(s.done, plane);
    } else {
      wait_plane(s.done, plane, unsigned(ny));
      zinv_tile<Cons, LZ, true, true>(sv, twz, plane * sv.n2 + tile * s.zl, s.zl, scale, cons, partials,
                                      plane * s.nz + tile, s.discard != 0);
    }
  }
}

}  // namespace combo_dev
