// Does SHFL share the shared-memory data port with LDS.128? Throughput of 16-byte partner reads by
// LDS.128, by 4 x SHFL.32 (xor), and both interleaved, per SM (148 CTAs x 256 threads).
// usage: ./shfl_lds_bench   (prints ns and bytes/clk/SM per variant)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>   // 0: LDS.128, 1: 4 x SHFL.32, 2: both
__global__ void __launch_bounds__(256, 1) k(double* out, int iters) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += 256) s[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  double2 v = make_double2(threadIdx.x, 1.0);
  const int tid = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (MODE == 0 || MODE == 2) {
        const double2 p = s[((tid + 256 * r) ^ (1 << (it & 7))) & 2047];
        acc.x += p.x;
        acc.y += p.y;
      }
      if (MODE == 1 || MODE == 2) {
        const int m = 1 << (r & 4 ? 4 : (r & 3));
        double2 q;
        q.x = __shfl_xor_sync(0xffffffffu, v.x, m);
        q.y = __shfl_xor_sync(0xffffffffu, v.y, m);
        acc.x += q.x;
        acc.y += q.y;
        v.x += 1.0;
      }
    }
  }
  if (acc.x == 12345.0) out[0] = acc.y;
}

template <int MODE>
float run(int iters) {
  double* d;
  cudaMalloc(&d, 8);
  k<MODE><<<148, 256>>>(d, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<148, 256>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(d);
  return ms;
}

int main() {
  const int iters = 20000;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double reads = 148.0 * 256 * 8 * iters;   // 16-byte partner reads
  const char* names[3] = {"LDS.128", "4xSHFL.32", "both"};
  float t[3] = {run<0>(iters), run<1>(iters), run<2>(iters)};
  for (int m = 0; m < 3; ++m) {
    const double bytes = reads * 16 * (m == 2 ? 2 : 1);
    printf("%-10s %8.3f ms  %.1f B/clk/SM at %d MHz (max clock; check nvidia-smi for the real one)\n", names[m], t[m],
           bytes / 148 / (t[m] * 1e-3 * clk * 1e3), clk / 1000);
  }
  return 0;
}
