// Memory-pattern probe for the FFT passes: in-place read+write of the
// half-spectrum layout [9][n1][n2][n3p] (complex) with the same tiles the
// y / x passes use, without any arithmetic. Separates access-pattern limits
// from compute/latency limits. Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/memprobe.cu -o gpurun_out/memprobe
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                           \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

constexpr int N = 512, N3P = 264, N3C = 257;

// tile of W columns x N rows; rows `stride` complex apart; thread (line, u)
// touches rows u + q N/8
template <int W, bool TOUCH>
__global__ void __launch_bounds__(W * 64) tile_rw(double2* spec, long stride, long plane, int ncomp_per_block) {
  const int kc0 = blockIdx.x * W;
  const int line = threadIdx.x % W, u = threadIdx.x / W;
  if (kc0 + line >= N3C) return;
  const int j = blockIdx.y;
  for (int cc = 0; cc < ncomp_per_block; ++cc) {
    const int c = blockIdx.z * ncomp_per_block + cc;
    double2* base = spec + long(c) * plane + long(j) * (stride == N3P ? long(N) * N3P : N3P) + kc0 + line;
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = base[long(u + q * (N / 8)) * stride];
    if (TOUCH) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q].x += 1.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) base[long(u + q * (N / 8)) * stride] = v[q];
  }
}

__global__ void copy_lin(const double2* a, double2* b, long n) {
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) b[i] = a[i];
}
__global__ void rw_lin(double2* a, long n) {
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    double2 v = a[i];
    v.x += 1.0;
    a[i] = v;
  }
}

int main() {
  const long plane = long(N) * N * N3P;
  const long total = 9 * plane;
  double2 *a, *b;
  CK(cudaMalloc(&a, total * sizeof(double2)));
  CK(cudaMalloc(&b, total * sizeof(double2)));
  CK(cudaMemset(a, 0, total * sizeof(double2)));
  CK(cudaMemset(b, 0, total * sizeof(double2)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double bytes = 2.0 * total * sizeof(double2);
    std::printf("%-40s %8.3f ms  %7.1f GB/s  (%s)\n", name, ms, bytes / ms / 1e6,
                cudaGetErrorString(cudaGetLastError()));
  };
  timeit("copy linear (a->b)", [&] { copy_lin<<<148 * 8, 512>>>(a, b, total); });
  timeit("rw linear in place", [&] { rw_lin<<<148 * 8, 512>>>(a, total); });
  // y pattern: rows N3P apart, grid (cols/W, n1, 9)
  timeit("y W=2", [&] { tile_rw<2, true><<<dim3((N3C + 1) / 2, N, 9), 128>>>(a, N3P, plane, 1); });
  timeit("y W=4", [&] { tile_rw<4, true><<<dim3((N3C + 3) / 4, N, 9), 256>>>(a, N3P, plane, 1); });
  timeit("y W=8", [&] { tile_rw<8, true><<<dim3((N3C + 7) / 8, N, 9), 512>>>(a, N3P, plane, 1); });
  // x pattern: rows N*N3P apart, grid (cols/W, n2, 9)
  timeit("x W=2", [&] { tile_rw<2, true><<<dim3((N3C + 1) / 2, N, 9), 128>>>(a, long(N) * N3P, plane, 1); });
  timeit("x W=4", [&] { tile_rw<4, true><<<dim3((N3C + 3) / 4, N, 9), 256>>>(a, long(N) * N3P, plane, 1); });
  timeit("x W=8", [&] { tile_rw<8, true><<<dim3((N3C + 7) / 8, N, 9), 512>>>(a, long(N) * N3P, plane, 1); });
  timeit("x W=4, 3 comps/block", [&] {
    tile_rw<4, true><<<dim3((N3C + 3) / 4, N, 3), 256>>>(a, long(N) * N3P, plane, 3);
  });
  // x pattern W=4 with 2-CTA clusters along the column tiles (adjacent
  // 64-byte segments of a row requested by co-scheduled CTAs)
  for (int cl : {2, 4}) {
    char name[64];
    std::snprintf(name, sizeof name, "x W=4 cluster %d", cl);
    timeit(name, [&] {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(((N3C + 3) / 4 + cl - 1) / cl * cl, N, 9);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, tile_rw<4, true>, a, long(N) * N3P, plane, 1);
    });
  }
  return 0;
}
