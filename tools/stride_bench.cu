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

// Same tile walk, staged through shared memory like the pass kernels: persistent CTAs, cp.async
// ring of STAGES tiles of 2^TB amplitudes, NT threads, then a shared read + global store.
template <int TB, int NT, int STAGES>
__global__ void __launch_bounds__(NT, 1) staged_copy(const double2* __restrict__ x, double2* __restrict__ y, int a,
                                                     int p, int g, uint64_t ntiles, int work) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sb = reinterpret_cast<double2*>(smem_raw);
  constexpr int EPT = (1 << TB) / NT;
  const int tid = threadIdx.x;
  auto gidx = [&](uint64_t t, uint32_t e) {
    const int m = p - a;
    const uint64_t tmid = t & ((1ull << m) - 1), thi = t >> m;
    const uint64_t lo = e & ((1u << a) - 1), h = e >> a;
    return lo | (tmid << a) | (h << p) | (thi << (p + g));
  };
  const uint64_t G = gridDim.x;
  for (int s0 = 0; s0 < STAGES - 1; ++s0) {
    const uint64_t tp = blockIdx.x + s0 * G;
    if (tp < ntiles)
      for (int i = 0; i < EPT; ++i) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(sb + s0 * (1 << TB) + tid + i * NT);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(x + gidx(tp, tid + i * NT)));
      }
    asm volatile("cp.async.commit_group;");
  }
  int stage = 0;
  double acc = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += G, stage = (stage + 1) % STAGES) {
    const uint64_t tn = t + (STAGES - 1) * G;
    if (tn < ntiles)
      for (int i = 0; i < EPT; ++i) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(sb + ((stage + STAGES - 1) % STAGES) * (1 << TB) + tid + i * NT);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(x + gidx(tn, tid + i * NT)));
      }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1));
    __syncthreads();
    const double2* s = sb + stage * (1 << TB);
    for (int i = 0; i < EPT; ++i) {
      double2 v = s[tid + i * NT];
      for (int w = 0; w < work; ++w) {   // synthetic flip work: shared partner loads
        const double2 q = s[(tid ^ (1 << w)) + i * NT];
        v.x = fma(1.0001, q.x, v.x);
        v.y = fma(1.0001, q.y, v.y);
      }
      y[gidx(t, tid + i * NT)] = v;
    }
    __syncthreads();
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
  int configs[][3] = {{11, 11, 0}, {3, 20, 9}, {4, 20, 8}};
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
  // staged variants
  for (int work : {0, 4, 9}) {
    for (int sel = 0; sel < 4; ++sel) {
      const int a = sel < 2 ? 12 : 4, p = sel < 2 ? 12 : 20, g = sel < 2 ? 0 : 8;
      const uint64_t ntiles = N >> 12;
      float ms = 0;
      const char* name = "";
      auto run = [&](auto kern, int nt, size_t smem, const char* nm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
        kern<<<148 * occ, nt, smem>>>(x, y, a, p, g, ntiles, work);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) kern<<<148 * occ, nt, smem>>>(x, y, a, p, g, ntiles, work);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("staged %-22s a=%2d work=%d occ=%d : %.0f GB/s\n", nm, a, work, occ,
               3.0 * 2 * N * sizeof(double2) / (ms * 1e-3) / 1e9);
      };
      if (sel == 0 || sel == 2) run(staged_copy<12, 512, 2>, 512, 2 * 65536, "TB12 NT512 S2");
      else run(staged_copy<12, 512, 3>, 512, 3 * 65536, "TB12 NT512 S3");
      (void)name;
    }
    const uint64_t nt11 = N >> 11;
    float ms = 0;
    auto run11 = [&](auto kern, int nt, size_t smem, const char* nm) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
      kern<<<148 * occ, nt, smem>>>(x, y, 11, 11, 0, nt11, work);
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) kern<<<148 * occ, nt, smem>>>(x, y, 11, 11, 0, nt11, work);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("staged %-22s a=11 work=%d occ=%d : %.0f GB/s\n", nm, work, occ,
             3.0 * 2 * N * sizeof(double2) / (ms * 1e-3) / 1e9);
    };
    run11(staged_copy<11, 256, 2>, 256, 2 * 32768, "TB11 NT256 S2");
    run11(staged_copy<11, 256, 3>, 256, 3 * 32768, "TB11 NT256 S3");
  }
  return 0;
}
