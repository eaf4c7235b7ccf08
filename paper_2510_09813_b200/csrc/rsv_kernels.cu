// rsv_kernels.cu -- see rsv_kernels.cuh for the design notes.
#include "rsv_kernels.cuh"

namespace rsv {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

__device__ __forceinline__ cplx ld_stream(const cplx* p) {
  // streaming 128-bit load (evict-first). Coherent path on purpose: the
  // accumulator operand may alias the output (in-place H.psi).
  return __ldcs(p);
}
__device__ __forceinline__ void st_stream(cplx* p, cplx v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
}

// Global index of tile-local element e in tile t.
__device__ __forceinline__ uint64_t tile_index(const Shape& sh, uint64_t t, uint32_t e) {
  const uint32_t lo = e & ((1u << sh.a) - 1u);
  const uint64_t h = e >> sh.a;
  const int m = sh.p - sh.a;
  const uint64_t tmid = t & ((1ull << m) - 1ull);
  const uint64_t thi = t >> m;
  return (uint64_t)lo | (tmid << sh.a) | (h << sh.p) | (thi << (sh.p + sh.g));
}

// Sum over the lanes of a (possibly partial, NT < 32) warp.
template <int NT>
__device__ __forceinline__ double warp_sum(double v) {
  constexpr unsigned mask = NT >= 32 ? 0xffffffffu : ((1u << NT) - 1u);
  constexpr int top = NT >= 32 ? 16 : NT / 2;
  #pragma unroll
  for (int o = top; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// Block-wide sum for a CTA of exactly NT threads; every thread gets the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  constexpr int NW = (NT + 31) / 32;
  v = warp_sum<NT>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  #pragma unroll
  for (int i = 0; i < NW; ++i) s += red[i];   // fixed order: deterministic
  return s;
}

// Deterministic grid reduction: every CTA writes its row, the last CTA to
// arrive sums the rows in index order. Returns true in the last CTA, where
// `tot` then holds the column sums.
template <int NCOL, int NT>
__device__ bool grid_finalize(const double (&mine)[NCOL], double* part, unsigned* counter,
                              double (&tot)[NCOL], double* red) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    #pragma unroll
    for (int c = 0; c < NCOL; ++c) part[(size_t)blockIdx.x * NCOL + c] = mine[c];
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  #pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    double v = 0.0;
    for (unsigned r = threadIdx.x; r < gridDim.x; r += NT) v += __ldcg(part + (size_t)r * NCOL + c);
    tot[c] = block_sum<NT>(v, red);
  }
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

// Per-tile diagonal helpers for the lo tile (bits [0, a) contiguous, g == 0).
// d[b] = dl[lo] + dh(tile) + sum_{i<a} bit_i(lo) * gcross_i(tile)
// gcross_i = sum_{j>=a} U_ij bit_j ; t1/t2 tabulate the cross sum on 6-bit halves.
struct DiagTile {
  double dh;
  double t1[64];
  double t2[64];
  double gc[kLoBits];
};

template <int NT>
__device__ void diag_tile_setup(const DiagArgs& dg, const Shape& sh, uint64_t tile, DiagTile* dt) {
  const int n = sh.n, a = sh.a;
  const uint64_t hb = tile;   // bits a..n-1 of the global index (n - a <= 32 hi qubits, NT >= 32 whenever n > a)
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
    // hi part: detuning and hi-hi interactions, one hi qubit per lane (n - a <= 32)
    double v = 0.0;
    const int j = a + l;
    if (j < n && ((hb >> l) & 1ull)) {
      v = -dg.delta[j];
      if (dg.mode == DIAG_FLY) {
        for (int i = a; i < j; ++i)
          if ((hb >> (i - a)) & 1ull) v += __ldg(dg.umat + (size_t)i * n + j);
      }
    }
    v = warp_sum<NT>(v);
    if (l == 0) dt->dh = v;
    if (l < kLoBits) {
      double gsum = 0.0;
      if (dg.mode == DIAG_FLY && l < a) {
        for (int jj = a; jj < n; ++jj)
          if ((hb >> (jj - a)) & 1ull) gsum += __ldg(dg.umat + (size_t)l * n + jj);
      }
      dt->gc[l] = gsum;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 128; idx += NT) {
    const int m = idx & 63;
    const int half = idx >> 6;
    double s = 0.0;
    #pragma unroll
    for (int b = 0; b < 6; ++b)
      if ((m >> b) & 1) s += dt->gc[half * 6 + b];
    if (half == 0) dt->t1[m] = s; else dt->t2[m] = s;
  }
  // caller syncs
}

__device__ __forceinline__ double diag_value(const DiagArgs& dg, const DiagTile* dt, uint32_t e,
                                             uint64_t gi) {
  double d = __ldg(dg.dl + e) + dt->dh;
  if (dg.mode == DIAG_FLY) d += dt->t1[e & 63] + dt->t2[(e >> 6) & 63];
  else d += __ldg(dg.dvec + gi);
  return d;
}

template <int TB, int KIND>
__global__ void __launch_bounds__((1 << TB) < kThreads ? (1 << TB) : kThreads, 2)
pass_kernel(const __grid_constant__ PassArgs A) {
  constexpr int TILE = 1 << TB;
  constexpr int NT = TILE < kThreads ? TILE : kThreads;
  constexpr int EPT = TILE / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* s = reinterpret_cast<cplx*>(smem_raw);
  __shared__ DiagTile dtile;
  __shared__ double red[32];

  const int tid = threadIdx.x;
  const double* sc = A.sc;
  const double xs = sc[A.x_scale_slot];
  const bool has_diag = A.dg.mode != DIAG_NONE;
  double alpha = 0.0, bprev = 0.0;
  if (KIND == PASS_LAST_LANCZOS) {
    alpha = sc[SC_AP + A.j] + sc[SC_Q + A.j];
    if (A.prev != nullptr && A.j > 0) bprev = sc[SC_BE + A.j - 1] * sc[SC_SG + A.j - 1];
  }
  double acc_a = 0.0, acc_n = 0.0, acc_q = 0.0;

  for (uint64_t t = blockIdx.x; t < A.sh.n_tiles; t += gridDim.x) {
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const uint32_t e = tid + i * NT;
      cp_async16(&s[e], A.x + tile_index(A.sh, t, e));
    }
    if (has_diag) diag_tile_setup<NT>(A.dg, A.sh, t, &dtile);
    cp_async_wait_all();
    __syncthreads();

    cplx wv[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const uint32_t e = tid + i * NT;
      const uint64_t gi = tile_index(A.sh, t, e);
      const cplx xv = s[e];
      double cr = 0.0, ci = 0.0;
      for (int f = 0; f < A.fl.count; ++f) {
        const cplx pv = s[e ^ A.fl.mask[f]];
        cr = fma(A.fl.coef[f], pv.x, cr);
        ci = fma(A.fl.coef[f], pv.y, ci);
      }
      if (has_diag) {
        const double d = diag_value(A.dg, &dtile, e, gi);
        cr = fma(d, xv.x, cr);
        ci = fma(d, xv.y, ci);
      }
      cr *= xs; ci *= xs;   // contribution of this pass's operator applied to v = xs * x
      // <v | contribution>, real part
      acc_a = fma(xs * xv.x, cr, fma(xs * xv.y, ci, acc_a));
      double orr = cr, oi = ci;
      if (A.uin != nullptr) {
        const cplx u = ld_stream(A.uin + gi);
        orr += u.x; oi += u.y;
      }
      if (KIND == PASS_LAST_LANCZOS) {
        orr = fma(-alpha * xs, xv.x, orr);
        oi = fma(-alpha * xs, xv.y, oi);
        if (bprev != 0.0) {
          const cplx pv = ld_stream(A.prev + gi);
          orr = fma(-bprev, pv.x, orr);
          oi = fma(-bprev, pv.y, oi);
        }
        acc_n = fma(orr, orr, fma(oi, oi, acc_n));
      }
      if (KIND == PASS_LAST_LANCZOS) wv[i] = make_double2(orr, oi);
      st_stream(A.out + gi, make_double2(orr, oi));
    }

    if (KIND == PASS_LAST_LANCZOS && A.qsweep) {
      // q-sweep: <w | A_this w> with w still on chip (this pass's share of alpha_{j+1})
      __syncthreads();
      #pragma unroll
      for (int i = 0; i < EPT; ++i) s[tid + i * NT] = wv[i];
      __syncthreads();
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const uint32_t e = tid + i * NT;
        double cr = 0.0, ci = 0.0;
        for (int f = 0; f < A.fl.count; ++f) {
          const cplx pv = s[e ^ A.fl.mask[f]];
          cr = fma(A.fl.coef[f], pv.x, cr);
          ci = fma(A.fl.coef[f], pv.y, ci);
        }
        if (has_diag) {
          const double d = diag_value(A.dg, &dtile, e, tile_index(A.sh, t, e));
          cr = fma(d, wv[i].x, cr);
          ci = fma(d, wv[i].y, ci);
        }
        acc_q = fma(wv[i].x, cr, fma(wv[i].y, ci, acc_q));
      }
    }
    __syncthreads();
  }

  if (KIND == PASS_LAST_APPLY) return;
  double mine[3];
  mine[0] = block_sum<NT>(acc_a, red);
  mine[1] = block_sum<NT>(acc_n, red);
  mine[2] = block_sum<NT>(acc_q, red);
  double tot[3];
  if (!grid_finalize<3, NT>(mine, A.part, A.counter, tot, red)) return;
  if (threadIdx.x != 0) return;
  double* scw = A.sc;
  if (KIND == PASS_FIRST) {
    scw[SC_AP + A.j] = tot[0];
  } else if (KIND == PASS_MID) {
    scw[SC_AP + A.j] += tot[0];
  } else {  // LAST_LANCZOS
    const double nrm2 = tot[1];
    const double beta = sqrt(nrm2);
    scw[SC_AL + A.j] = alpha;
    scw[SC_BE + A.j] = beta;
    scw[SC_SG + A.j + 1] = beta > 0.0 ? 1.0 / beta : 0.0;
    scw[SC_Q + A.j + 1] = nrm2 > 0.0 ? tot[2] / nrm2 : 0.0;
  }
}

// Krylov combination psi_new = sum_i coef_i v_i, fused with the next step's
// ||psi||^2, q_0 and the observable masks.
template <int TB>
__global__ void __launch_bounds__((1 << TB) < kThreads ? (1 << TB) : kThreads, 2)
combine_kernel(const __grid_constant__ CombineArgs A) {
  constexpr int TILE = 1 << TB;
  constexpr int NT = TILE < kThreads ? TILE : kThreads;
  constexpr int EPT = TILE / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* s = reinterpret_cast<cplx*>(smem_raw);
  __shared__ DiagTile dtile;
  __shared__ double red[32];
  __shared__ double s_obs[kMaxMasks];
  const int tid = threadIdx.x;
  const bool has_diag = A.qsweep && A.dg.mode != DIAG_NONE;
  for (int m = tid; m < A.nmask; m += NT) s_obs[m] = 0.0;
  double acc_n = 0.0, acc_q = 0.0;

  for (uint64_t t = blockIdx.x; t < A.sh.n_tiles; t += gridDim.x) {
    if (has_diag) diag_tile_setup<NT>(A.dg, A.sh, t, &dtile);
    cplx wv[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) wv[i] = make_double2(0.0, 0.0);
    for (int k = 0; k < A.k; ++k) {
      const cplx* vk = A.v[k];
      const double2 c = A.coef[k];
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const cplx x = ld_stream(vk + tile_index(A.sh, t, tid + i * NT));
        wv[i].x = fma(c.x, x.x, fma(-c.y, x.y, wv[i].x));
        wv[i].y = fma(c.x, x.y, fma(c.y, x.x, wv[i].y));
      }
    }
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const uint64_t gi = tile_index(A.sh, t, tid + i * NT);
      if (A.out != nullptr) st_stream(A.out + gi, wv[i]);
      acc_n = fma(wv[i].x, wv[i].x, fma(wv[i].y, wv[i].y, acc_n));
    }
    if (A.qsweep) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) s[tid + i * NT] = wv[i];
      __syncthreads();
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const uint32_t e = tid + i * NT;
        double cr = 0.0, ci = 0.0;
        for (int f = 0; f < A.fl.count; ++f) {
          const cplx pv = s[e ^ A.fl.mask[f]];
          cr = fma(A.fl.coef[f], pv.x, cr);
          ci = fma(A.fl.coef[f], pv.y, ci);
        }
        if (has_diag) {
          const double d = diag_value(A.dg, &dtile, e, tile_index(A.sh, t, e));
          cr = fma(d, wv[i].x, cr);
          ci = fma(d, wv[i].y, ci);
        }
        acc_q = fma(wv[i].x, cr, fma(wv[i].y, ci, acc_q));
      }
    }
    if (A.nmask > 0) {
      double p[EPT];
      #pragma unroll
      for (int i = 0; i < EPT; ++i) p[i] = wv[i].x * wv[i].x + wv[i].y * wv[i].y;
      for (int m0 = 0; m0 < A.nmask; m0 += 8) {
        double acc[8];
        #pragma unroll
        for (int mm = 0; mm < 8; ++mm) acc[mm] = 0.0;
        #pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const uint64_t gi = tile_index(A.sh, t, tid + i * NT);
          #pragma unroll
          for (int mm = 0; mm < 8; ++mm) {
            const int m = m0 + mm;
            const uint64_t M = m < A.nmask ? A.mask[m] : ~0ull;
            acc[mm] += ((gi & M) == M) ? p[i] : 0.0;
          }
        }
        #pragma unroll
        for (int mm = 0; mm < 8; ++mm) {
          const double v = block_sum<NT>(acc[mm], red);
          if (tid == 0 && m0 + mm < A.nmask) s_obs[m0 + mm] += v;
        }
      }
    }
    __syncthreads();
  }

  double mine[2];
  mine[0] = block_sum<NT>(acc_n, red);
  mine[1] = block_sum<NT>(acc_q, red);
  __syncthreads();
  // write observables as extra rows: reuse the generic finalize with a fixed column count
  __shared__ bool s_last;
  const int ncol = 2 + A.nmask;
  if (tid == 0) {
    A.part[(size_t)blockIdx.x * (2 + kMaxMasks) + 0] = mine[0];
    A.part[(size_t)blockIdx.x * (2 + kMaxMasks) + 1] = mine[1];
  }
  for (int m = tid; m < A.nmask; m += NT) A.part[(size_t)blockIdx.x * (2 + kMaxMasks) + 2 + m] = s_obs[m];
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned tk = atomicAdd(A.counter, 1u);
    s_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double tot[2];
  for (int c = 0; c < ncol; ++c) {
    double v = 0.0;
    for (unsigned r = tid; r < gridDim.x; r += NT) v += __ldcg(A.part + (size_t)r * (2 + kMaxMasks) + c);
    const double sum = block_sum<NT>(v, red);
    if (c < 2) tot[c] = sum;
    else if (tid == 0) A.sc[SC_OBS + c - 2] = sum;   // raw sums; host divides by ||psi||^2
  }
  if (tid == 0) {
    *A.counter = 0u;
    A.sc[SC_N0SQ] = tot[0];
    A.sc[SC_SG + 0] = tot[0] > 0.0 ? 1.0 / sqrt(tot[0]) : 0.0;
    A.sc[SC_Q + 0] = tot[0] > 0.0 ? tot[1] / tot[0] : 0.0;
  }
}

__global__ void build_dl_kernel(int a, int n, const double* __restrict__ umat, const double* __restrict__ delta_dev,
                                DiagArgs dg, int with_interaction, double* __restrict__ dl) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (1 << a)) return;
  double v = 0.0;
  for (int i = 0; i < a; ++i) {
    if (!((e >> i) & 1)) continue;
    v -= delta_dev ? delta_dev[i] : dg.delta[i];
    if (with_interaction)
      for (int j = i + 1; j < a; ++j)
        if ((e >> j) & 1) v += umat[(size_t)i * n + j];
  }
  dl[e] = v;
}

// Diagonal -sum_i delta_i bit_i + sum_{i<j} U_ij bit_i bit_j for every index
// (precomputed-vector variant, sv.py:116; rydsim/hamiltonian.py:114 build_diagonal).
__global__ void interaction_diag_kernel(int n, const double* __restrict__ umat, DiagArgs dg, int with_delta,
                                        double* __restrict__ dvec) {
  __shared__ double su[kMaxQubits * kMaxQubits];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) su[i] = umat[i];
  __syncthreads();
  const uint64_t total = 1ull << n;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < total;
       b += (uint64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int i = 0; i < n; ++i) {
      if (!((b >> i) & 1ull)) continue;
      if (with_delta) v -= dg.delta[i];
      for (int j = i + 1; j < n; ++j)
        if ((b >> j) & 1ull) v += su[i * n + j];
    }
    dvec[b] = v;
  }
}

__global__ void zdotc_kernel(const cplx* __restrict__ x, const cplx* __restrict__ y, uint64_t n,
                             double* part, unsigned* counter, double* result2) {
  __shared__ double red[32];
  double re = 0.0, im = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const cplx a = x[i], b = y[i];
    re = fma(a.x, b.x, fma(a.y, b.y, re));   // conj(a) * b
    im = fma(a.x, b.y, fma(-a.y, b.x, im));
  }
  double mine[2] = {block_sum<kThreads>(re, red), block_sum<kThreads>(im, red)};
  double tot[2];
  if (!grid_finalize<2, kThreads>(mine, part, counter, tot, red)) return;
  if (threadIdx.x == 0) { result2[0] = tot[0]; result2[1] = tot[1]; }
}

// sum |x - y|^2 (norm_difference, observables.py:137, without cancellation)
__global__ void diff_norm_kernel(const cplx* __restrict__ x, const cplx* __restrict__ y, uint64_t n,
                                 double* part, unsigned* counter, double* result) {
  __shared__ double red[32];
  double s = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const cplx a = x[i], b = y[i];
    const double dr = a.x - b.x, di = a.y - b.y;
    s = fma(dr, dr, fma(di, di, s));
  }
  double mine[1] = {block_sum<kThreads>(s, red)};
  double tot[1];
  if (!grid_finalize<1, kThreads>(mine, part, counter, tot, red)) return;
  if (threadIdx.x == 0) result[0] = tot[0];
}

// w -= alpha v + beta vprev ; result = ||w||^2 (generic-matvec Lanczos, krylov.py:100-105)
__global__ void lanczos_update_kernel(cplx* __restrict__ w, const cplx* __restrict__ v,
                                      const cplx* __restrict__ vprev, double alpha, double beta, uint64_t n,
                                      double* part, unsigned* counter, double* result) {
  __shared__ double red[32];
  double nn = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    cplx a = w[i];
    const cplx b = v[i];
    a.x -= alpha * b.x; a.y -= alpha * b.y;
    if (vprev != nullptr) { const cplx c = vprev[i]; a.x -= beta * c.x; a.y -= beta * c.y; }
    w[i] = a;
    nn = fma(a.x, a.x, fma(a.y, a.y, nn));
  }
  double mine[1] = {block_sum<kThreads>(nn, red)};
  double tot[1];
  if (!grid_finalize<1, kThreads>(mine, part, counter, tot, red)) return;
  if (threadIdx.x == 0) result[0] = tot[0];
}

__global__ void axpy_kernel(cplx* __restrict__ y, const cplx* __restrict__ x, double2 a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const cplx b = x[i];
    cplx c = y[i];
    c.x = fma(a.x, b.x, fma(-a.y, b.y, c.x));
    c.y = fma(a.x, b.y, fma(a.y, b.x, c.y));
    y[i] = c;
  }
}

__global__ void scale_kernel(cplx* __restrict__ y, const cplx* __restrict__ x, double2 a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const cplx b = x[i];
    y[i] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
}

int g_num_sms = 0;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int TB, int KIND>
cudaError_t launch_pass_tbk(const PassArgs& args, int grid, cudaStream_t st) {
  constexpr int TILE = 1 << TB;
  constexpr int NT = TILE < kThreads ? TILE : kThreads;
  const size_t smem = TILE * sizeof(cplx);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(pass_kernel<TB, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  pass_kernel<TB, KIND><<<grid, NT, smem, st>>>(args);
  return cudaGetLastError();
}

template <int TB>
cudaError_t launch_pass_tb(const PassArgs& args, int grid, cudaStream_t st) {
  switch (args.kind) {
    case PASS_FIRST: return launch_pass_tbk<TB, PASS_FIRST>(args, grid, st);
    case PASS_MID: return launch_pass_tbk<TB, PASS_MID>(args, grid, st);
    case PASS_LAST_APPLY: return launch_pass_tbk<TB, PASS_LAST_APPLY>(args, grid, st);
    case PASS_LAST_LANCZOS: return launch_pass_tbk<TB, PASS_LAST_LANCZOS>(args, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int TB>
cudaError_t launch_combine_tb(const CombineArgs& args, int grid, cudaStream_t st) {
  constexpr int TILE = 1 << TB;
  constexpr int NT = TILE < kThreads ? TILE : kThreads;
  const size_t smem = TILE * sizeof(cplx);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(combine_kernel<TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  combine_kernel<TB><<<grid, NT, smem, st>>>(args);
  return cudaGetLastError();
}

}  // namespace

int max_pass_grid(int tile_bits) {
  // 64 KB tiles: 3 resident CTAs per SM
  const int per_sm = tile_bits >= 12 ? 3 : 4;
  return num_sms() * per_sm;
}

int pass_grid(const Shape& sh) {
  const uint64_t cap = (uint64_t)max_pass_grid(sh.a + sh.g);
  return (int)(sh.n_tiles < cap ? sh.n_tiles : cap);
}

cudaError_t launch_pass(const PassArgs& args, int grid, cudaStream_t st) {
  const int tb = args.sh.a + args.sh.g;
  switch (tb) {
    case 1: return launch_pass_tb<1>(args, grid, st);
    case 2: return launch_pass_tb<2>(args, grid, st);
    case 3: return launch_pass_tb<3>(args, grid, st);
    case 4: return launch_pass_tb<4>(args, grid, st);
    case 5: return launch_pass_tb<5>(args, grid, st);
    case 6: return launch_pass_tb<6>(args, grid, st);
    case 7: return launch_pass_tb<7>(args, grid, st);
    case 8: return launch_pass_tb<8>(args, grid, st);
    case 9: return launch_pass_tb<9>(args, grid, st);
    case 10: return launch_pass_tb<10>(args, grid, st);
    case 11: return launch_pass_tb<11>(args, grid, st);
    case 12: return launch_pass_tb<12>(args, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_combine(const CombineArgs& args, int grid, cudaStream_t st) {
  const int tb = args.sh.a + args.sh.g;
  switch (tb) {
    case 1: return launch_combine_tb<1>(args, grid, st);
    case 2: return launch_combine_tb<2>(args, grid, st);
    case 3: return launch_combine_tb<3>(args, grid, st);
    case 4: return launch_combine_tb<4>(args, grid, st);
    case 5: return launch_combine_tb<5>(args, grid, st);
    case 6: return launch_combine_tb<6>(args, grid, st);
    case 7: return launch_combine_tb<7>(args, grid, st);
    case 8: return launch_combine_tb<8>(args, grid, st);
    case 9: return launch_combine_tb<9>(args, grid, st);
    case 10: return launch_combine_tb<10>(args, grid, st);
    case 11: return launch_combine_tb<11>(args, grid, st);
    case 12: return launch_combine_tb<12>(args, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_build_dl(int a, int n, const double* umat, const double* delta_dev_or_null,
                            const double* delta_host, int with_interaction, double* dl, cudaStream_t st) {
  DiagArgs dg{};
  if (delta_host != nullptr)
    for (int i = 0; i < n && i < kMaxQubits; ++i) dg.delta[i] = delta_host[i];
  const int total = 1 << a;
  const int nt = total < 256 ? total : 256;
  build_dl_kernel<<<(total + nt - 1) / nt, nt, 0, st>>>(a, n, umat, delta_dev_or_null, dg, with_interaction, dl);
  return cudaGetLastError();
}

cudaError_t launch_interaction_diag(int n, const double* umat, const double* delta_host, double* dvec,
                                    cudaStream_t st) {
  const uint64_t total = 1ull << n;
  uint64_t blocks = (total + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  DiagArgs dg{};
  if (delta_host != nullptr)
    for (int i = 0; i < n && i < kMaxQubits; ++i) dg.delta[i] = delta_host[i];
  interaction_diag_kernel<<<(unsigned)blocks, 256, 0, st>>>(n, umat, dg, delta_host != nullptr, dvec);
  return cudaGetLastError();
}

static unsigned flat_grid(uint64_t n, int grid) {
  if (grid > 0) return (unsigned)grid;
  uint64_t blocks = (n + kThreads - 1) / kThreads;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

cudaError_t launch_zdotc(const cplx* x, const cplx* y, uint64_t n, double* part, unsigned* counter,
                         double* result2, int grid, cudaStream_t st) {
  zdotc_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(x, y, n, part, counter, result2);
  return cudaGetLastError();
}

cudaError_t launch_diff_norm(const cplx* x, const cplx* y, uint64_t n, double* part, unsigned* counter,
                             double* result, int grid, cudaStream_t st) {
  diff_norm_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(x, y, n, part, counter, result);
  return cudaGetLastError();
}

cudaError_t launch_lanczos_update(cplx* w, const cplx* v, const cplx* vprev, double alpha, double beta,
                                  uint64_t n, double* part, unsigned* counter, double* result, int grid,
                                  cudaStream_t st) {
  lanczos_update_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(w, v, vprev, alpha, beta, n, part, counter,
                                                                  result);
  return cudaGetLastError();
}

cudaError_t launch_axpy(cplx* y, const cplx* x, double2 a, uint64_t n, int grid, cudaStream_t st) {
  axpy_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(y, x, a, n);
  return cudaGetLastError();
}

cudaError_t launch_scale(cplx* y, const cplx* x, double2 a, uint64_t n, int grid, cudaStream_t st) {
  scale_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(y, x, a, n);
  return cudaGetLastError();
}

}  // namespace rsv
