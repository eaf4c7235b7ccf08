// Micro-benchmark: copy bandwidth of strided tiles (2^a contiguous complex128 x 2^g rows at
// stride 2^p elements), the access pattern of the hi bit-group passes. Build + run on the box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sb tools/stride_bench.cu && /tmp/sb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void tile_copy(const double2* __restrict__ x, double2* __restrict__ y, int n, int a, int p, int g,
                          uint64_t ntiles) {
  const int tile = 1 << (a + g);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int m = p - a;
    const uint64_t tmid = t & ((1ull << m) - 1), thi = t >> m;
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
      const uint64_t lo = e & ((1 << a) - 1), h = e >> a;
      const uint64_t gi = lo | (tmid << a) | (h << p) | (thi << (p + g));
      y[gi] = __ldcs(x + gi);
    }
  }
}

int main() {
  const int n = 29;
  const size_t N = size_t(1) << n;
  double2 *x, *y;
  cudaMalloc(&x, N * sizeof(double2));
  cudaMalloc(&y, N * sizeof(double2));
  cudaMemset(x, 0, N * sizeof(double2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int configs[][3] = {{11, 11, 0}, {1, 20, 9}, {2, 20, 9}, {3, 20, 9}, {4, 20, 9}, {5, 20, 9},
                      {2, 11, 9}, {3, 11, 9}, {4, 11, 9}, {2, 14, 9}, {2, 17, 9}, {3, 17, 9},
                      {3, 21, 8}, {4, 22, 7}, {2, 20, 6}, {5, 20, 6}};
  for (auto& c : configs) {
    const int a = c[0], p = c[1], g = c[2];
    const uint64_t ntiles = N >> (a + g);
    for (int threads : {256, 512}) {
      for (int bps : {2, 4, 8}) {
        const int grid = 148 * bps;
        tile_copy<<<grid, threads>>>(x, y, n, a, p, g, ntiles);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) tile_copy<<<grid, threads>>>(x, y, n, a, p, g, ntiles);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("a=%d p=%2d g=%d threads=%d ctas/sm=%d : %.0f GB/s\n", a, p, g, threads, bps,
               3.0 * 2 * N * sizeof(double2) / (ms * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
