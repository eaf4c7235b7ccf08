// Micro-benchmark: can the TMA engine de-interleave complex128 tiles into re/im planes in shared
// memory (tensor map with elementStrides[0] = 2) at full HBM bandwidth?
// A tile = 2^a contiguous complex x 2^g strided rows (the hi-pass shape) or 2^13 contiguous complex
// (lo shape). Modes (per tile, persistent CTAs, 2-stage mbarrier ring, copy x -> y):
//   0 interleaved: one 5-D TMA load of the tile (current pass kernels), LDS.128 + STG.128
//   1 planar     : two TMA loads with elementStrides = 2 (re plane, im plane), LDS.64 x2 + STG.128
// Build + run on the box:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pb tools/plane_tma_bench.cu -lcuda && /tmp/pb
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(su32(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(bar)) : "memory");
}

struct Geo { int n, a, p, g; uint64_t ntiles; };

template <int MODE>
__global__ void __launch_bounds__(256, 1) kcopy(const __grid_constant__ CUtensorMap tm, const double2* x, double2* y, Geo G) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* al = sm + ((128u - (su32(sm) & 127u)) & 127u);
  const int TILE = 1 << (G.a + G.g);
  double* buf = reinterpret_cast<double*>(al);      // 2 stages x 2 x TILE doubles
  uint64_t* bars = reinterpret_cast<uint64_t*>(buf + 4 * TILE);
  if (threadIdx.x == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int m = G.p - G.a;
  auto issue = [&](uint64_t t, int st) {
    if (threadIdx.x != 0) return;
    mbar_expect(&bars[st], TILE * 16);
    const int c1 = (int)(t & ((1ull << m) - 1)), c4 = (int)(t >> m);
    double* d = buf + st * 2 * TILE;
    if (MODE == 0) {
      tma5(d, &tm, 0, c1, 0, 0, c4, &bars[st]);
    } else {
      tma5(d, &tm, 0, c1, 0, 0, c4, &bars[st]);          // re plane (even doubles)
      tma5(d + TILE, &tm, 1, c1, 0, 0, c4, &bars[st]);   // im plane (odd doubles)
    }
  };
  unsigned ph = 0;
  const uint64_t T0 = blockIdx.x, GS = gridDim.x;
  if (T0 < G.ntiles) issue(T0, 0);
  int st = 0;
  for (uint64_t t = T0; t < G.ntiles; t += GS, st ^= 1) {
    mbar_wait(&bars[st], (ph >> st) & 1u);
    ph ^= 1u << st;
    __syncthreads();
    if (t + GS < G.ntiles) issue(t + GS, st ^ 1);
    const double* d = buf + st * 2 * TILE;
    const int c1 = (int)(t & ((1ull << m) - 1)), c4 = (int)(t >> m);
    for (int e = threadIdx.x; e < TILE; e += 256) {
      double2 v;
      if (MODE == 0) v = reinterpret_cast<const double2*>(d)[e];
      else v = make_double2(d[e], d[TILE + e]);
      const uint64_t lo = e & ((1 << G.a) - 1), h = e >> G.a;
      const uint64_t gi = lo | ((uint64_t)c1 << G.a) | (h << G.p) | ((uint64_t)c4 << (G.p + G.g));
      __stcs(y + gi, v);
    }
  }
}

__global__ void fill(double2* x, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    x[i] = make_double2((double)i, -(double)i - 0.5);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 29;
  const uint64_t N = 1ull << n;
  double2 *x, *y;
  CK(cudaMalloc(&x, N * 16));
  CK(cudaMalloc(&y, N * 16));
  fill<<<1024, 256>>>(x, N);
  CK(cudaDeviceSynchronize());
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fp;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Case { int a, p, g; } cases[] = {{4, 21, 8}, {3, 12, 9}, {5, 21, 7}, {6, 6, 6}, {2, 21, 10}};
  for (auto cs : cases) {
    Geo G{n, cs.a, cs.p, cs.g, 1ull << (n - cs.a - cs.g)};
    for (int mode = 0; mode < 2; ++mode) {
      CUtensorMap tm;
      const int g1 = cs.g;
      cuuint64_t dim[5] = {2ull << cs.a, 1ull << (cs.p - cs.a), 1ull << g1, 1, 1ull << (n - cs.p - cs.g)};
      cuuint64_t stride[4] = {16ull << cs.a, 16ull << cs.p, 16ull << (cs.p + g1), 16ull << (cs.p + cs.g)};
      cuuint32_t box[5] = {2u << cs.a, 1u, 1u << g1, 1u, 1u};
      cuuint32_t es[5] = {mode == 0 ? 1u : 2u, 1, 1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, x, dim, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("a=%d g=%d mode %d: encode failed %d\n", cs.a, cs.g, mode, (int)r); continue; }
      const int TILE = 1 << (cs.a + cs.g);
      const size_t smem = 4 * TILE * 8 + 64 + 128;
      auto kern = mode == 0 ? kcopy<0> : kcopy<1>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      kern<<<sms, 256, smem>>>(tm, x, y, G);
      CK(cudaDeviceSynchronize());
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<sms, 256, smem>>>(tm, x, y, G);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      // correctness spot check: y == x at scattered indices
      bool ok = true;
      for (uint64_t i : {(uint64_t)0, (uint64_t)1, N / 3, N / 2 + 17, N - 1, (uint64_t)12345677}) {
        double2 h;
        CK(cudaMemcpy(&h, y + i, sizeof(h), cudaMemcpyDeviceToHost));
        ok = ok && h.x == (double)i && h.y == -(double)i - 0.5;
      }
      printf("a=%d p=%d g=%d %-11s %.3f ms  %.0f GB/s  %s\n", cs.a, cs.p, cs.g, mode == 0 ? "interleaved" : "planar",
             best, 32.0 * N / best / 1e6, ok ? "ok" : "MISMATCH");
      CK(cudaMemset(y, 0, N * 16));
    }
  }
  return 0;
}
