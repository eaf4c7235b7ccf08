// rsv_kernels.cu -- sm_100a kernels; see rsv_kernels.cuh for the design notes.
#include "rsv_kernels.cuh"

#include <algorithm>
#include <type_traits>

#ifndef RSV_STAGES
#define RSV_STAGES 2
#endif
#ifndef RSV_L2_PREFETCH
#define RSV_L2_PREFETCH 1
#endif
// elementwise operand staged through shared memory (cp.async) or prefetched into registers
// issue the next x tile before (1, needs an end-of-tile barrier) or after (0) the tile wait
#ifndef RSV_EARLY_ISSUE
#define RSV_EARLY_ISSUE 0
#endif
// bulk-async (TMA) data movement in the pass kernels (0: per-thread cp.async)
#ifndef RSV_TMA
#define RSV_TMA 1
#endif
// timing experiments only: skip the last pass's q-sweep (wrong Lanczos coefficients)
#ifndef RSV_QSWEEP_OFF
#define RSV_QSWEEP_OFF 0
#endif
// Krylov combination ring filled by per-warp bulk copies (TMA) instead of per-thread cp.async
#ifndef RSV_COMBINE_TMA
#define RSV_COMBINE_TMA 0
#endif
#ifndef RSV_ROT_MID
#define RSV_ROT_MID 0
#endif
// rotating tile buffers: the elementwise operand is prefetched one tile ahead too (pass_kernel_rot)
#ifndef RSV_ROT
#define RSV_ROT 1
#endif
#ifndef RSV_EIN_REGS
#define RSV_EIN_REGS 0
#endif
// output tiles leave through shared memory by TMA stores (PassArgs::tstore) instead of STG: in the
// last pass (rotating buffers, w is staged in shared memory for the q-sweep anyway) and, opt-in, in
// the lo/mid passes (measured slower there: the store delays the operand refill of the e buffer)
#ifndef RSV_TSTORE
#define RSV_TSTORE 1
#endif
#ifndef RSV_TSTORE_TMA
#define RSV_TSTORE_TMA 0
#endif
// last pass: the q-sweep's shared-memory bits 4..7 as register pairs of a transposed layout
#ifndef RSV_QT
#define RSV_QT 1
#endif
// tile barrier before the wait for x(t): the next tile's load is issued one wait earlier (measured
// at N=29: no difference, lo/mid/last within 0.5 %; off)
#ifndef RSV_DVEC_SMEM
#define RSV_DVEC_SMEM 1   // diag="vec": stage the diagonal tile in shared memory by a bulk copy
#endif
#ifndef RSV_EARLY_X
#define RSV_EARLY_X 0
#endif

namespace rsv {

namespace {

constexpr int kThreads = 256;     // generic / combine kernels

#ifndef RSV_CP_L2PF
#define RSV_CP_L2PF 0   // cp.async L2 prefetch-size hint (0: none, 128, 256 bytes)
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
#if RSV_CP_L2PF == 256
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
#elif RSV_CP_L2PF == 128
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- mbarrier + bulk (TMA) copies
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// ---- TMA stores (shared -> global, bulk-group completion)
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2,
                                             int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                 "r"(c4) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the source buffers of every committed store have been read (the buffer may be refilled)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed store is complete
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Output tile tt of a pass leaves shared memory (src, tile order e) by one TMA store; issued by one
// thread after a CTA barrier that follows every writer's fence.proxy.async.
__device__ __forceinline__ void store_tile(const PassArgs& A, uint64_t tt, const void* src) {
  if (A.load == LOAD_CONTIG) {
    bulk_s2g(A.out + ((uint64_t)tt << (A.sh.a + A.sh.g)), src, (unsigned)(sizeof(cplx) << (A.sh.a + A.sh.g)));
  } else {
    const int m = A.sh.p - A.sh.a;
    tma_store_5d(&A.tm_o, src, 0, (int)(tt & ((1ull << m) - 1ull)), 0, 0, (int)(tt >> m));
  }
  bulk_commit();
}

__device__ __forceinline__ cplx ld_stream(const cplx* p) {
  // streaming 128-bit load (evict-first). Coherent path on purpose: the
  // accumulator operand may alias the output (in-place H.psi).
  return __ldcs(p);
}
__device__ __forceinline__ void st_stream(cplx* p, cplx v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
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
// Offset of tile element e relative to element 0 of the same tile (the fields are disjoint,
// so index(t, tid + i*NT) = index(t, tid) + offset(i*NT)).
__device__ __forceinline__ uint64_t elem_offset(const Shape& sh, uint32_t e) {
  const uint32_t lo = e & ((1u << sh.a) - 1u);
  const uint64_t h = e >> sh.a;
  return (uint64_t)lo | (h << sh.p);
}

// Flips on a tile bit that is a lane bit of the thread layout (mask < 32) take the partner from the
// neighbouring lane's registers by warp shuffles instead of a shared-memory load: 4 x SHFL.32 per
// complex128 cost half the MIO/shared-memory-port time of one LDS.128 (tools/shfl_lds_bench.cu:
// 243 vs 126 B/clk/SM; the two share the pipe), and the x tile is already in registers.
// Measured at N=29 (profiles/r2_shfl_flips.md): slower in the mid pass (five of its eight shared-
// memory flips are lane bits: the shuffles' issue slots and dependent latency outweigh the port time
// they save) and the lo pass; in the last pass (one lane bit among four) 1.7 % faster on a
// 1687 MHz box, 2 % slower on a 1537 MHz one. Off; RSV_SHFL_FLIPS=1 shuffles every lane bit in the
// last pass (rotating-buffer body) and lane bits >= RSV_SHFL_TMA_MIN in the lo/mid passes.
#ifndef RSV_SHFL_FLIPS
#define RSV_SHFL_FLIPS 0
#endif
#ifndef RSV_SHFL_TMA_MIN
#define RSV_SHFL_TMA_MIN 32
#endif
__device__ __forceinline__ cplx shfl_xor_c(cplx v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
// ac[i] += c * (partner of xv[i] across tile bit m), partners of lane bits by shuffles, the others
// from the tile in shared memory (s: this thread's element 0)
template <int NT, int EPT, int MMIN>
__device__ __forceinline__ void flip_into(cplx (&ac)[EPT], const cplx (&xv)[EPT], const cplx* s, int tid, int m,
                                          double c) {
  if (RSV_SHFL_FLIPS && NT >= 32 && m >= MMIN && m < 32) {
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const cplx p = shfl_xor_c(xv[i], m);
      ac[i].x = fma(c, p.x, ac[i].x);
      ac[i].y = fma(c, p.y, ac[i].y);
    }
    return;
  }
  const cplx* ps = s + (tid ^ m);
  #pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const cplx p = ps[i * NT];
    ac[i].x = fma(c, p.x, ac[i].x);
    ac[i].y = fma(c, p.y, ac[i].y);
  }
}

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

// Deterministic grid reduction: every CTA writes its row, the last CTA to arrive sums the
// rows in index order. Returns true in the last CTA, where `tot` holds the column sums.
template <int NCOL, int NT>
__device__ bool grid_finalize(const double (&mine)[NCOL], double* part, unsigned* counter, double (&tot)[NCOL],
                              double* red) {
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

template <int EPT>
struct RegBits {
  static constexpr int value = EPT >= 32 ? 5 : (EPT >= 16 ? 4 : (EPT >= 8 ? 3 : (EPT >= 4 ? 2 : (EPT >= 2 ? 1 : 0))));
};
template <int N>
struct Log2 {
  static constexpr int value = N <= 1 ? 0 : 1 + Log2<N / 2>::value;
};

// Last pass of Lanczos iteration j: alpha_j, beta_j, sigma_{j+1}, q_{j+1} from the grid sums
// ||w||^2 and <w|A_last|w>. Sharded runs (raw) store the local sums (beta slot = ||w||^2, q slot =
// <w|A|w>); the host all-reduces them and writes the scalars back (rsv_capi.cu, shard_finish_iteration).
__device__ __forceinline__ void lanczos_scalars(double* scw, int j, int raw, double alpha, double nrm2, double qraw,
                                                double* mail) {
  scw[SC_AL + j] = alpha;
  if (raw) {
    scw[SC_BE + j] = nrm2;
    scw[SC_Q + j + 1] = qraw;
    return;
  }
  const double beta = sqrt(nrm2);
  scw[SC_BE + j] = beta;
  scw[SC_SG + j + 1] = beta > 0.0 ? 1.0 / beta : 0.0;
  scw[SC_Q + j + 1] = nrm2 > 0.0 ? qraw / nrm2 : 0.0;
  if (mail != nullptr) {   // host mailbox (mapped pinned memory): read after the iteration's event
    if (j == 0) mail[0] = scw[SC_N0SQ];
    mail[1 + 2 * j] = alpha;
    mail[2 + 2 * j] = beta;
    __threadfence_system();
  }
}

// ---------------------------------------------------------------- on-the-fly diagonal
// For the lo tile (bits [0, a) contiguous, tile t = bits a..n-1):
//   d(b) = dl[e] + hh[t] - sum_{j>=a} delta_j bit_j(t) + sum_{i<a} bit_i(e) gc[t][i]
// dl (2^a, per step): lo detuning (+ lo-lo interactions for DIAG_FLY);
// hh, gc (per run, DIAG_FLY): hi-hi interactions and the lo-hi couplings of tile t.
// Thread tid owns e_i = tid + i*NT, so the cross term splits into a per-thread part
// (bits of tid) and a per-element part (bits of i): no shared tables, no barriers.
template <int NT, int EPT>
struct DiagRow {
  double d[EPT];

  // row: shared copy of [gc[t][0..11], hh[t], tb[t]] (see pass_kernel), or nullptr to read global
  __device__ __forceinline__ void setup(const DiagArgs& dg, const Shape& sh, uint64_t t, int tid,
                                        const double* row) {
    constexpr int LT = Log2<NT>::value;
    constexpr int RB = RegBits<EPT>::value;
    const int a = sh.a;
    const double base = row ? row[13] : __ldg(dg.gc + t * kGcStride + 13);   // tb[t] = hh[t] - sum_{j>=a} delta_j bit_j(t)
    double cross_t = 0.0;
    double gy[RB > 0 ? RB : 1];
    if (dg.mode == DIAG_FLY) {
      const double* g = row ? row : dg.gc + t * kGcStride;
      #pragma unroll
      for (int b = 0; b < LT; ++b)
        if (b < a && ((tid >> b) & 1)) cross_t += g[b];
      #pragma unroll
      for (int b = 0; b < RB; ++b) gy[b] = (LT + b < a) ? g[LT + b] : 0.0;
    } else {
      #pragma unroll
      for (int b = 0; b < RB; ++b) gy[b] = 0.0;
    }
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      double v = base + cross_t + __ldg(dg.dl + tid + i * NT);
      #pragma unroll
      for (int b = 0; b < RB; ++b)
        if ((i >> b) & 1) v += gy[b];
      d[i] = v;
    }
  }
};

// ---------------------------------------------------------------- bit-group pass
// Persistent CTAs walk tiles t = blockIdx.x + k*gridDim.x. The x tile goes through a ring
// of STAGES shared-memory buffers filled by cp.async one ring ahead; the elementwise
// operands (uin, prev) are prefetched into registers at the top of each iteration. Thread
// tid owns tile elements e_i = tid + i*NT: flips on tile bits >= log2(NT) are register
// permutations, the others one conflict-free 16-byte shared load per element.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

template <int TB, int KIND, int NT, bool DIAG>
__global__ void __launch_bounds__(NT, NT >= RSV_PASS_THREADS ? 1 : 2) pass_kernel(const __grid_constant__ PassArgs A) {
  constexpr int TILE = 1 << TB;
  constexpr int EPT = TILE / NT;
  constexpr int RB = RegBits<EPT>::value;
  constexpr int STAGES = TB >= 8 ? RSV_STAGES : 2;
  constexpr bool LANCZOS = KIND == PASS_LAST_LANCZOS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cplx* sbuf = reinterpret_cast<cplx*>(smem_raw);   // STAGES x TILE
  __shared__ double red[32];

  const int tid = threadIdx.x;
  const double* sc = A.sc;
  const double xs = sc[A.x_scale_slot];
  double alpha = 0.0;
  if (LANCZOS) alpha = sc[SC_AP + A.j] + sc[SC_Q + A.j];
  const bool has_e = A.ein != nullptr;
  const double ecoef = A.ein_is_prev ? -(sc[SC_BE + A.j - 1] * sc[SC_SG + A.j - 1]) : 1.0;
  // coefficients pre-scaled by the operand scale (v = xs * x)
  double rc[RB > 0 ? RB : 1];
  #pragma unroll
  for (int b = 0; b < RB; ++b) rc[b] = A.fl.rcoef[b] * xs;
  const double axs = alpha * xs;
  double acc_a = 0.0, acc_n = 0.0, acc_q = 0.0;
  // element i of a thread sits at index(t, tid) + i*S: the plan keeps the i*NT bits either all
  // contiguous (lo tile) or all in the strided group (hi tiles, a <= log2 NT)
  const uint64_t S = elem_offset(A.sh, NT);

  const uint64_t ntiles = A.sh.n_tiles;
  const uint64_t G = gridDim.x;
  // shared layout: x ring [STAGES][TILE] | elementwise-operand buffer [TILE] | tile-table rows [STAGES][16]
  cplx* ubuf = sbuf + STAGES * TILE;
  double* rows = reinterpret_cast<double*>(sbuf + (STAGES + 1) * TILE);
  auto issue_x = [&](uint64_t tt, int st_idx) {
    const cplx* src = A.x + tile_index(A.sh, tt, tid);
    cplx* dst = sbuf + st_idx * TILE + tid;
    #pragma unroll
    for (int i = 0; i < EPT; ++i) cp_async16(dst + i * NT, src + i * S);
    if (DIAG)
      for (int k = tid; k < kGcStride / 2; k += NT) cp_async16(rows + st_idx * 16 + 2 * k, A.dg.gc + tt * kGcStride + 2 * k);
  };
  #pragma unroll
  for (int s0 = 0; s0 < STAGES - 1; ++s0) {
    const uint64_t tp = blockIdx.x + (uint64_t)s0 * G;
    if (tp < ntiles) issue_x(tp, s0);
    cp_async_commit();
  }
  int stage = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += G, stage = (stage + 1 == STAGES ? 0 : stage + 1)) {
    const uint64_t g0 = tile_index(A.sh, t, tid);
    // group A_t: this tile's elementwise operand u (each thread copies and later reads only its own
    // amplitudes, so no barrier is needed around ubuf)
    cplx ev[EPT];
    if (has_e) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        if (RSV_EIN_REGS && KIND == PASS_MID) ev[i] = ld_stream(A.ein + g0 + i * S);
        else cp_async16(ubuf + tid + i * NT, A.ein + g0 + i * S);
      }
    }
    cp_async_commit();
#if RSV_EARLY_ISSUE
    // group B_t: the x tile (and tile-table row) one ring ahead
    const uint64_t tn = t + (uint64_t)(STAGES - 1) * G;
    if (tn < ntiles) issue_x(tn, stage == 0 ? STAGES - 1 : stage - 1);
    cp_async_commit();
#endif
#if RSV_L2_PREFETCH
    // only for the contiguous lo tile: on strided tiles the extra LSU traffic costs more than it saves
    if (DIAG && (tid & 7) == 0) {
      const uint64_t t1 = t + G, t2 = t + (uint64_t)STAGES * G;
      if (t1 < ntiles && has_e) {
        const uint64_t g1 = tile_index(A.sh, t1, tid);
        #pragma unroll
        for (int i = 0; i < EPT; ++i) prefetch_l2(A.ein + g1 + i * S);
      }
      if (t2 < ntiles) {
        const uint64_t g2 = tile_index(A.sh, t2, tid);
        #pragma unroll
        for (int i = 0; i < EPT; ++i) prefetch_l2(A.x + g2 + i * S);
      }
    }
#endif
#if RSV_EARLY_ISSUE
    // x(t) was group B_{t-1}: at most A_t and B_t may still be in flight
    cp_async_wait<STAGES>();
    __syncthreads();
#else
    // x(t) was group B_{t-1}: only A_t may still be in flight
    cp_async_wait<1>();
    __syncthreads();
    {
      // group B_t: every thread is past its reads of the buffer tile t+G overwrites (it belonged to
      // tile t-G, processed before this barrier), so no end-of-tile barrier is needed
      const uint64_t tn = t + (uint64_t)(STAGES - 1) * G;
      if (tn < ntiles) issue_x(tn, stage == 0 ? STAGES - 1 : stage - 1);
      cp_async_commit();
    }
#endif
    const cplx* s = sbuf + stage * TILE;
    DiagRow<NT, EPT> dr;
    if (DIAG) dr.setup(A.dg, A.sh, t, tid, rows + stage * 16);

    cplx xv[EPT], ac[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      xv[i] = s[tid + i * NT];
      ac[i] = make_double2(0.0, 0.0);
    }
    #pragma unroll
    for (int b = 0; b < RB; ++b) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        ac[i].x = fma(rc[b], xv[i ^ (1 << b)].x, ac[i].x);
        ac[i].y = fma(rc[b], xv[i ^ (1 << b)].y, ac[i].y);
      }
    }
    for (int f = 0; f < A.fl.count; ++f) {
      const cplx* ps = s + (tid ^ A.fl.mask[f]);   // partner of element i is ps[i*NT]
      const double c = A.fl.coef[f] * xs;
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const cplx p = ps[i * NT];
        ac[i].x = fma(c, p.x, ac[i].x);
        ac[i].y = fma(c, p.y, ac[i].y);
      }
    }
    if (DIAG) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double d = dr.d[i];
        if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
        d *= xs;
        ac[i].x = fma(d, xv[i].x, ac[i].x);
        ac[i].y = fma(d, xv[i].y, ac[i].y);
      }
    }
    if (!(RSV_EIN_REGS && KIND == PASS_MID) && has_e) cp_async_wait<1>();   // A_t (this tile's operand) done; B_t may be in flight
    cplx* po = A.out + g0;
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      double cr = ac[i].x, ci = ac[i].y;   // this pass's operator applied to v = xs * x
      acc_a = fma(xv[i].x, cr, fma(xv[i].y, ci, acc_a));
      if (has_e) {
        const cplx u = (RSV_EIN_REGS && KIND == PASS_MID) ? ev[i] : ubuf[tid + i * NT];
        cr = fma(ecoef, u.x, cr);
        ci = fma(ecoef, u.y, ci);
      }
      if (LANCZOS) {
        cr = fma(-axs, xv[i].x, cr);
        ci = fma(-axs, xv[i].y, ci);
        acc_n = fma(cr, cr, fma(ci, ci, acc_n));
      }
      ac[i] = make_double2(cr, ci);
      st_stream(po + i * S, ac[i]);
    }

    if (LANCZOS && A.qsweep) {
      // q-sweep: <w | A_this w> while w is on chip (this pass's share of alpha_{j+1})
      __syncthreads();
      cplx* sw = sbuf + stage * TILE;
      #pragma unroll
      for (int i = 0; i < EPT; ++i) sw[tid + i * NT] = ac[i];
      __syncthreads();
      // <w|X_k|w> = 2 Re sum_{bit k of b = 0} conj(w_b) w_{b^k}: each pair is visited once
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double hr = 0.0, hi = 0.0;
        #pragma unroll
        for (int b = 0; b < RB; ++b) {
          if ((i >> b) & 1) continue;
          hr = fma(2.0 * A.fl.rcoef[b], ac[i ^ (1 << b)].x, hr);
          hi = fma(2.0 * A.fl.rcoef[b], ac[i ^ (1 << b)].y, hi);
        }
        if (DIAG) {
          double d = dr.d[i];
          if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
          hr = fma(d, ac[i].x, hr);
          hi = fma(d, ac[i].y, hi);
        }
        acc_q = fma(ac[i].x, hr, fma(ac[i].y, hi, acc_q));
      }
      for (int f = 0; f < A.fl.count; ++f) {
        const int m = A.fl.mask[f];
        if (tid & m) continue;   // partner visits the pair (whole warps skip for mask >= 32)
        const cplx* ps = sw + (tid ^ m);
        const double c2 = 2.0 * A.fl.coef[f];
        #pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const cplx p = ps[i * NT];
          acc_q = fma(c2, fma(ac[i].x, p.x, ac[i].y * p.y), acc_q);
        }
      }
    }
#if RSV_EARLY_ISSUE
    __syncthreads();
#endif
  }
  cp_async_wait<0>();
  acc_a *= xs;

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
  } else {
    lanczos_scalars(scw, A.j, A.raw, alpha, tot[1], tot[2], A.mail);
  }
}

// ---------------------------------------------------------------- bit-group pass, TMA version
// Same arithmetic as pass_kernel; the data movement is bulk-async (TMA engine) instead of
// per-thread cp.async: each warp copies its own amplitudes' contiguous runs (min(2^a, 32)
// amplitudes) with cp.async.bulk, completion is tracked by mbarriers (expected-transaction
// bytes), so the LSU/MIO queues only carry the shared-memory partner loads and the stores.
//   x ring : 2 stages, tile t+G is requested right after the tile-t barrier
//   e buf  : this tile's elementwise operand, requested after the same barrier, awaited
//            just before the epilogue
// Peer-memory mode with NPEER > 0 partners: their tiles come by TMA over NVLink into a ring of
// kPeerSlots shared-memory slots of one eighth of a tile (8 KB) each -- chunk c of the CTA's
// sequence (tile it, eighth k, partner p) = it * 8 * NPEER + k * NPEER + p -- completed by mbarriers
// (full: expected bytes; empty: every thread has read the slot). The ring holds half a partner tile
// (a quarter with two partners), so a tile's chunks are consumed at 2 * NPEER points spread over the
// flip phase (before the flips, between them, in the epilogue), kPeerSlots chunks at each; once every
// thread has read a point's last chunk, thread 0 refills all its slots, so the chunks of the next
// point land while the flips in between run. The partner reads take no LSU instructions.
constexpr int kPeerSlots = 4;
constexpr int kPeerChunk = (1 << kLoBits) / 8;   // amplitudes per slot
constexpr size_t kPeerRingBytes = kPeerSlots * kPeerChunk * sizeof(cplx) + 2 * kPeerSlots * sizeof(uint64_t) + 128;

template <int TB, int KIND, int NT, bool DIAG, int NPEER = 0>
__device__ __forceinline__ void pass_tma_body(const PassArgs& A) {
  constexpr bool PEER = NPEER > 0;
  static_assert(NPEER <= 2 && (!PEER || (TB == kLoBits && (1 << TB) / NT >= 8)),
                "peer ring: 1 or 2 partners, full tiles, >= 8 amplitudes a thread");
  // 32 amplitudes a thread (the 128-thread mid pass): outputs in two halves
  constexpr bool SPLIT = (1 << TB) / NT == 32 && KIND == PASS_MID && !DIAG && !PEER;
  static_assert(!SPLIT || !RSV_TSTORE_TMA, "the split mid pass stores by thread");
  constexpr int TILE = 1 << TB;
  constexpr int EPT = TILE / NT;
  constexpr int RB = RegBits<EPT>::value;
  constexpr bool LANCZOS = KIND == PASS_LAST_LANCZOS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // TMA tensor destinations need 128-byte alignment; the dynamic window starts after the
  // static shared variables, so align by hand (the launch adds 128 bytes of slack)
  unsigned char* smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  cplx* xbuf = reinterpret_cast<cplx*>(smem_al);             // [2][TILE]
  cplx* ebuf = xbuf + 2 * TILE;                               // [TILE]
  double* rows = reinterpret_cast<double*>(ebuf + TILE);     // [2][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rows + 32);   // xbar[0], xbar[1], ebar
  // peer ring (PEER): slots 128-byte aligned after the barriers, then full[4], empty[4]
  cplx* pring = reinterpret_cast<cplx*>(smem_al + ((3 * TILE * sizeof(cplx) + 32 * sizeof(double) +
                                                    4 * sizeof(uint64_t) + 127) & ~size_t(127)));
  uint64_t* pfull = reinterpret_cast<uint64_t*>(pring + kPeerSlots * kPeerChunk);
  uint64_t* pempty = pfull + kPeerSlots;
  // diag="vec": the tile's float64 diagonal entries arrive by one bulk copy at the tile barrier (bars[3]),
  // where the peer ring would sit (never both); per-thread loads had exposed a DRAM latency per tile
  const bool dvt = DIAG && !PEER && A.dvec_smem != 0;
  const double* dbuf = reinterpret_cast<const double*>(pring);
  __shared__ double red[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // scalars through L2 (__ldcg): in the fused iteration kernel another CTA wrote them this launch
  const double* sc = A.sc;
  const double xs = __ldcg(sc + A.x_scale_slot);
  double alpha = 0.0;
  if (LANCZOS) alpha = __ldcg(sc + SC_AP + A.j) + __ldcg(sc + SC_Q + A.j);
  const bool has_e = A.ein != nullptr;
  const double ecoef = A.ein_is_prev ? -(__ldcg(sc + SC_BE + A.j - 1) * __ldcg(sc + SC_SG + A.j - 1)) : 1.0;
  double rc[RB > 0 ? RB : 1];
  #pragma unroll
  for (int b = 0; b < RB; ++b) rc[b] = A.fl.rcoef[b] * xs;
  const double axs = alpha * xs;
  double acc_a = 0.0, acc_n = 0.0, acc_q = 0.0;
  const uint64_t S = elem_offset(A.sh, NT);
  const uint64_t ntiles = A.sh.n_tiles;
  const uint64_t G = gridDim.x;

  // copy geometry: a warp owns tile elements [32 w + NT i, +32) for i < EPT, made of
  // runs of R amplitudes contiguous in global memory (R = 2^a, capped at the warp's 32)
  const int R = (1 << A.sh.a) < 32 ? (1 << A.sh.a) : (NT < 32 ? NT : 32);
  const int RUNS = (NT < 32 ? NT : 32) / R;   // runs per warp per i
  const unsigned tile_bytes = TILE * sizeof(cplx) + (DIAG ? 112u : 0u);
  auto issue = [&](const cplx* base, const CUtensorMap* map, uint64_t tt, cplx* dst, uint64_t* bar) {
    if (A.load == LOAD_CONTIG) {
      if (tid == 0) bulk_g2s(dst, base + tile_index(A.sh, tt, 0), TILE * sizeof(cplx), bar);
      return;
    }
    if (A.load == LOAD_TENSOR) {
      if (tid == 0) {
        const int m = A.sh.p - A.sh.a;
        tma_load_5d(dst, map, 0, (int)(tt & ((1ull << m) - 1ull)), 0, 0, (int)(tt >> m), bar);
      }
      return;
    }
    // lane k < RUNS copies run k of every i-chunk of this warp
    if (lane < RUNS) {
      const uint32_t e0 = (uint32_t)(warp * 32 + lane * R);
      const cplx* src = base + tile_index(A.sh, tt, e0);
      #pragma unroll
      for (int i = 0; i < EPT; ++i) bulk_g2s(dst + e0 + i * NT, src + i * S, R * sizeof(cplx), bar);
    }
  };

  // peer chunks of this CTA: (tiles it owns) x 8 eighths x npeer partners
  constexpr int npeer = PEER ? NPEER : 1;
  const uint32_t pchunks = PEER ? (uint32_t)((ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0) * 8 *
                                             (uint64_t)npeer) : 0u;
  auto issue_peer = [&](uint32_t c) {   // thread 0: chunk c into slot c % kPeerSlots
    const uint32_t per_tile = 8u * (uint32_t)npeer;
    const uint64_t tt = blockIdx.x + (uint64_t)(c / per_tile) * G;
    const uint32_t rem = c % per_tile;
    const int k = (int)(rem / (uint32_t)npeer), pp = (int)(rem % (uint32_t)npeer);
    const int slot = (int)(c % kPeerSlots);
    mbar_arrive_expect_tx(&pfull[slot], kPeerChunk * sizeof(cplx));
    if (A.load == LOAD_CONTIG) {
      bulk_g2s(pring + slot * kPeerChunk, A.peer[pp] + tile_index(A.sh, tt, 0) + (uint64_t)k * kPeerChunk,
               kPeerChunk * sizeof(cplx), &pfull[slot]);
    } else {
      const int m = A.sh.p - A.sh.a;
      tma_load_5d(pring + slot * kPeerChunk, &A.tm_peer[pp], 0, (int)(tt & ((1ull << m) - 1ull)), 0, k,
                  (int)(tt >> m), &pfull[slot]);
    }
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    if (dvt) mbar_init(&bars[3], 1);
    if (PEER) {
      for (int s2 = 0; s2 < kPeerSlots; ++s2) {
        mbar_init(&pfull[s2], 1);
        mbar_init(&pempty[s2], NT);
      }
    }
    mbar_init_fence();
  }
  __syncthreads();
  if constexpr (PEER) {
    if (tid == 0)
      for (uint32_t c = 0; c < pchunks && c < (uint32_t)kPeerSlots; ++c) issue_peer(c);
  }
  uint32_t pc = 0;                     // next peer chunk to consume
  unsigned xphase = 0u, ephase = 0u;   // bit s = parity of x stage s (a register, not a local array)
  unsigned dphase = 0u;
  // output tiles through the e buffer (in place over the operand) and a TMA store issued at the
  // next tile barrier (no per-thread global stores, no 64-bit address arithmetic per amplitude)
  const bool tstore = RSV_TSTORE_TMA && A.tstore != 0;
  // prologue: tile blockIdx.x into stage 0
  if (blockIdx.x < ntiles) {
    if (tid == 0) mbar_arrive_expect_tx(&bars[0], tile_bytes);
    __syncthreads();
    issue(A.x, &A.tm_x, blockIdx.x, xbuf, &bars[0]);
    if (DIAG && tid == 0) bulk_g2s(rows, A.dg.gc + blockIdx.x * kGcStride, 112, &bars[0]);
  }
  int stage = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += G, stage ^= 1) {
    const uint64_t g0 = tile_index(A.sh, t, tid);
    const uint64_t tn = t + G;
    // arm the barriers before the tile barrier so every copy is issued after its expect_tx
    if (tid == 0) {
      if (tn < ntiles) mbar_arrive_expect_tx(&bars[stage ^ 1], tile_bytes);
      if (has_e) mbar_arrive_expect_tx(&bars[2], TILE * sizeof(cplx));
    }
#if !RSV_EARLY_X
    mbar_wait(&bars[stage], (xphase >> stage) & 1u);
    xphase ^= 1u << stage;
#endif
    __syncthreads();   // everyone is done with tile t-G: its x buffer and the e buffer are free
    if (tn < ntiles) {
      issue(A.x, &A.tm_x, tn, xbuf + (stage ^ 1) * TILE, &bars[stage ^ 1]);
      if (DIAG && tid == 0) bulk_g2s(rows + (stage ^ 1) * 16, A.dg.gc + tn * kGcStride, 112, &bars[stage ^ 1]);
    }
    if (tstore && t != blockIdx.x) {
      // tile t-G's output sits in the e buffer: store it and let it be read before the refill
      if (tid == 0) {
        store_tile(A, t - G, ebuf);
        bulk_wait_read0();
      }
      // without an operand nothing else orders this tile's epilogue writes after the store's reads
      if (!has_e) __syncthreads();
    }
    if (has_e) issue(A.ein, &A.tm_e, t, ebuf, &bars[2]);
    if (dvt && tid == 0) {
      mbar_arrive_expect_tx(&bars[3], TILE * sizeof(double));
      bulk_g2s(const_cast<double*>(dbuf), A.dg.dvec + tile_index(A.sh, t, 0), TILE * sizeof(double), &bars[3]);
    }
#if RSV_EARLY_X
    // x(t) is awaited after the refills are issued: tile t+G's load starts one wait earlier
    mbar_wait(&bars[stage], (xphase >> stage) & 1u);
    xphase ^= 1u << stage;
#endif
    const cplx* s = xbuf + stage * TILE;
    DiagRow<NT, EPT> dr;
    if (DIAG) dr.setup(A.dg, A.sh, t, tid, rows + stage * 16);

    if constexpr (SPLIT) {
      // 32 amplitudes a thread (5 register bits): all of x in registers, the outputs in two halves
      // of 16 accumulators (half h = tile bit log2(NT)+4), so the register file holds 128 + 64
      constexpr int H = EPT / 2;
      cplx xv[EPT];
      #pragma unroll
      for (int i = 0; i < EPT; ++i) xv[i] = s[tid + i * NT];
      cplx* po = A.out + g0;
      #pragma unroll
      for (int h = 0; h < 2; ++h) {
        cplx ac[H];
        #pragma unroll
        for (int ii = 0; ii < H; ++ii) ac[ii] = make_double2(0.0, 0.0);
        #pragma unroll
        for (int b = 0; b < RB; ++b) {
          #pragma unroll
          for (int ii = 0; ii < H; ++ii) {
            ac[ii].x = fma(rc[b], xv[(ii + h * H) ^ (1 << b)].x, ac[ii].x);
            ac[ii].y = fma(rc[b], xv[(ii + h * H) ^ (1 << b)].y, ac[ii].y);
          }
        }
        for (int f = 0; f < A.fl.count; ++f) {
          const cplx* ps = s + (tid ^ A.fl.mask[f]) + h * H * NT;
          const double c = A.fl.coef[f] * xs;
          #pragma unroll
          for (int ii = 0; ii < H; ++ii) {
            const cplx p = ps[ii * NT];
            ac[ii].x = fma(c, p.x, ac[ii].x);
            ac[ii].y = fma(c, p.y, ac[ii].y);
          }
        }
        for (int g = 0; g < A.npeer; ++g) {   // sharded, per-thread partner loads
          const cplx* pp = A.peer[g] + g0 + (uint64_t)h * H * S;
          const double c = A.peer_coef[g] * xs;
          #pragma unroll
          for (int ii = 0; ii < H; ++ii) {
            const cplx v = __ldcg(pp + ii * S);
            ac[ii].x = fma(c, v.x, ac[ii].x);
            ac[ii].y = fma(c, v.y, ac[ii].y);
          }
        }
        if (h == 0 && has_e) {
          mbar_wait(&bars[2], ephase);
          ephase ^= 1u;
        }
        #pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          const int i = ii + h * H;
          double cr = ac[ii].x, ci = ac[ii].y;
          acc_a = fma(xv[i].x, cr, fma(xv[i].y, ci, acc_a));
          if (has_e) {
            const cplx u = ebuf[tid + i * NT];
            cr = fma(ecoef, u.x, cr);
            ci = fma(ecoef, u.y, ci);
          }
          st_stream(po + i * S, make_double2(cr, ci));
        }
      }
      continue;
    }
    cplx xv[EPT], ac[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      xv[i] = s[tid + i * NT];
      ac[i] = make_double2(0.0, 0.0);
    }
    // partner chunks of consumption point Q: eighths [Q*E8, (Q+1)*E8) of every partner
    constexpr int NPTS = 2 * npeer, E8 = 8 / NPTS, EPK = EPT / 8;
    auto consume = [&](auto qc) {
      constexpr int Q = decltype(qc)::value;
      #pragma unroll
      for (int k = Q * E8; k < (Q + 1) * E8; ++k) {
        #pragma unroll
        for (int pp = 0; pp < npeer; ++pp, ++pc) {
          const int slot = (int)(pc % kPeerSlots);
          mbar_wait(&pfull[slot], (pc / kPeerSlots) & 1u);
          const cplx* src = pring + slot * kPeerChunk + tid;   // e = tid + NT (k EPK + ii)
          const double c = A.peer_coef[pp] * xs;
          #pragma unroll
          for (int ii = 0; ii < EPK; ++ii) {
            const cplx v = src[ii * NT];
            ac[k * EPK + ii].x = fma(c, v.x, ac[k * EPK + ii].x);
            ac[k * EPK + ii].y = fma(c, v.y, ac[k * EPK + ii].y);
          }
          mbar_arrive(&pempty[slot]);
        }
      }
      // once every thread has read the point's last chunk it has read all kPeerSlots of them (in
      // order): one wait, then each slot takes the chunk kPeerSlots ahead
      if (tid == 0) {
        const uint32_t last = pc - 1;
        mbar_wait(&pempty[last % kPeerSlots], (last / kPeerSlots) & 1u);
        for (uint32_t c = pc - kPeerSlots; c < pc; ++c)
          if ((int64_t)pchunks - (int64_t)c > kPeerSlots) issue_peer(c + kPeerSlots);
      }
    };
    if constexpr (PEER) consume(std::integral_constant<int, 0>{});
    #pragma unroll
    for (int b = 0; b < RB; ++b) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        ac[i].x = fma(rc[b], xv[i ^ (1 << b)].x, ac[i].x);
        ac[i].y = fma(rc[b], xv[i ^ (1 << b)].y, ac[i].y);
      }
    }
    if constexpr (NPEER == 2) {   // points 1 and 2 after a third and two thirds of the shared-memory flips
      if (A.fl.count < 3) {
        consume(std::integral_constant<int, 1>{});
        consume(std::integral_constant<int, 2>{});
      }
    }
    for (int f = 0; f < A.fl.count; ++f) {
      if constexpr (NPEER == 2) {
        if (A.fl.count >= 3 && f == A.fl.count / 3) consume(std::integral_constant<int, 1>{});
        if (A.fl.count >= 3 && f == (2 * A.fl.count) / 3) consume(std::integral_constant<int, 2>{});
      }
      flip_into<NT, EPT, RSV_SHFL_TMA_MIN>(ac, xv, s, tid, A.fl.mask[f], A.fl.coef[f] * xs);
    }
    if constexpr (PEER) consume(std::integral_constant<int, NPTS - 1>{});
    if (DIAG) {
      if (dvt) {
        mbar_wait(&bars[3], dphase);
        dphase ^= 1u;
      }
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double d = dr.d[i];
        if (dvt) d += dbuf[tid + i * NT];
        else if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
        d *= xs;
        ac[i].x = fma(d, xv[i].x, ac[i].x);
        ac[i].y = fma(d, xv[i].y, ac[i].y);
      }
    }
    // sharded runs in peer-memory mode: the flips on the global qubits read the partner shards'
    // x (same local index) straight from their HBM over NVLink; they are part of this pass's
    // operator, so they also enter <x|A x> (alpha's partial share)
    for (int g = 0; g < (PEER ? 0 : A.npeer); ++g) {
      const cplx* pp = A.peer[g] + g0;
      const double c = A.peer_coef[g] * xs;
      cplx pv[EPT];
      #pragma unroll
      for (int i = 0; i < EPT; ++i) pv[i] = __ldcg(pp + i * S);
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        ac[i].x = fma(c, pv[i].x, ac[i].x);
        ac[i].y = fma(c, pv[i].y, ac[i].y);
      }
    }
    if (has_e) {
      mbar_wait(&bars[2], ephase);
      ephase ^= 1u;
    }
    cplx* po = A.out + g0;
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      double cr = ac[i].x, ci = ac[i].y;
      acc_a = fma(xv[i].x, cr, fma(xv[i].y, ci, acc_a));
      if (has_e) {
        const cplx u = ebuf[tid + i * NT];
        cr = fma(ecoef, u.x, cr);
        ci = fma(ecoef, u.y, ci);
      }
      if (LANCZOS) {
        cr = fma(-axs, xv[i].x, cr);
        ci = fma(-axs, xv[i].y, ci);
        acc_n = fma(cr, cr, fma(ci, ci, acc_n));
      }
      ac[i] = make_double2(cr, ci);
      if (tstore) ebuf[tid + i * NT] = ac[i];   // over this thread's own operand entry
      else st_stream(po + i * S, ac[i]);
    }
    if (tstore) fence_proxy_async_smem();   // generic writes -> the TMA store's reads

    if (LANCZOS && A.qsweep) {
      // w goes to the e buffer: each thread overwrites only the entries it alone has read,
      // so a single barrier (w complete) suffices; the next refill of the buffer is issued
      // after the next tile barrier
      cplx* sw = ebuf;
      if (!tstore) {
        #pragma unroll
        for (int i = 0; i < EPT; ++i) sw[tid + i * NT] = ac[i];
      }
      __syncthreads();
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double hr = 0.0, hi = 0.0;
        #pragma unroll
        for (int b = 0; b < RB; ++b) {
          if ((i >> b) & 1) continue;
          hr = fma(2.0 * A.fl.rcoef[b], ac[i ^ (1 << b)].x, hr);
          hi = fma(2.0 * A.fl.rcoef[b], ac[i ^ (1 << b)].y, hi);
        }
        if (DIAG) {
          double d = dr.d[i];
          if (dvt) d += dbuf[tid + i * NT];
          else if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
          hr = fma(d, ac[i].x, hr);
          hi = fma(d, ac[i].y, hi);
        }
        acc_q = fma(ac[i].x, hr, fma(ac[i].y, hi, acc_q));
      }
      for (int f = 0; f < A.fl.count; ++f) {
        const int m = A.fl.mask[f];
        if (tid & m) continue;
        const cplx* ps = sw + (tid ^ m);
        const double c2 = 2.0 * A.fl.coef[f];
        #pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const cplx p = ps[i * NT];
          acc_q = fma(c2, fma(ac[i].x, p.x, ac[i].y * p.y), acc_q);
        }
      }
      fence_proxy_async_smem();   // generic writes to a buffer the TMA engine refills later
    }
  }
  if (tstore && blockIdx.x < ntiles) {
    __syncthreads();   // the CTA's last output tile is complete in the e buffer
    if (tid == 0) {
      const uint64_t tl = blockIdx.x + ((ntiles - 1 - blockIdx.x) / G) * G;
      store_tile(A, tl, ebuf);
      bulk_wait0();
    }
  }
  acc_a *= xs;

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
  } else {
    lanczos_scalars(scw, A.j, A.raw, alpha, tot[1], tot[2], A.mail);
  }
}

// ---------------------------------------------------------------- bit-group pass, rotating buffers
// Same arithmetic as pass_kernel_tma, but both operands are prefetched: three tile buffers rotate
// through the roles "x of tile it", "operand of tile it" and "x of tile it+1". Buffer it%3 holds
// x(it); once every thread is past the flips (barrier B) it receives the operand of tile it+1, so
// that load has a whole epilogue plus the next tile's flips to land; the operand buffer of tile it
// receives x(it+2) after the next tile barrier (A). Cost: one more CTA barrier per tile.
// X0: x of the CTA's first tile was already requested into buffer 0 (and the barriers initialised) by
// rot_issue_x0 -- the fused iteration kernel does that before its grid barrier.
template <int TB, int KIND, int NT, bool DIAG, bool X0 = false>
__device__ __forceinline__ void pass_rot_body(const PassArgs& A) {
  constexpr int TILE = 1 << TB;
  constexpr int EPT = TILE / NT;
  constexpr int RB = RegBits<EPT>::value;
  constexpr bool LANCZOS = KIND == PASS_LAST_LANCZOS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  cplx* buf = reinterpret_cast<cplx*>(smem_al);              // [3][TILE]
  double* rows = reinterpret_cast<double*>(buf + 3 * TILE);  // [3][16] tile-table rows (ride with x)
  uint64_t* bars = reinterpret_cast<uint64_t*>(rows + 48);   // one mbarrier per buffer
  __shared__ double red[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* sc = A.sc;   // through L2: see pass_tma_body
  const double xs = __ldcg(sc + A.x_scale_slot);
  double alpha = 0.0;
  if (LANCZOS) alpha = __ldcg(sc + SC_AP + A.j) + __ldcg(sc + SC_Q + A.j);
  const bool has_e = A.ein != nullptr;
  const double ecoef = A.ein_is_prev ? -(__ldcg(sc + SC_BE + A.j - 1) * __ldcg(sc + SC_SG + A.j - 1)) : 1.0;
  double rc[RB > 0 ? RB : 1];
  #pragma unroll
  for (int b = 0; b < RB; ++b) rc[b] = A.fl.rcoef[b] * xs;
  double r2[RB > 0 ? RB : 1];   // q-sweep: 2 Omega_b / 2 of the register bits
  #pragma unroll
  for (int b = 0; b < RB; ++b) r2[b] = 2.0 * A.fl.rcoef[b];
  const double axs = alpha * xs;
  double acc_a = 0.0, acc_n = 0.0, acc_q = 0.0;
  const uint64_t S = elem_offset(A.sh, NT);
  const uint64_t ntiles = A.sh.n_tiles;
  const uint64_t G = gridDim.x;
  const bool tstore = RSV_TSTORE && A.tstore != 0;
  // q-sweep flips on tile bits 4..7 in a transposed layout (4096-amplitude tile, 16 per thread)
  constexpr bool kQT = RSV_QT && TB == 12 && NT == 256;
  unsigned qt_mask = 0u;
  double qc[4] = {0.0, 0.0, 0.0, 0.0};
  if (kQT) {
    for (int f = 0; f < A.fl.count; ++f) {
      const int m = A.fl.mask[f];
      #pragma unroll
      for (int b = 0; b < 4; ++b)
        if (m == (16 << b)) {
          qt_mask |= (unsigned)m;
          qc[b] = 2.0 * A.fl.coef[f];
        }
    }
  }

  const int R = (1 << A.sh.a) < 32 ? (1 << A.sh.a) : (NT < 32 ? NT : 32);
  const int RUNS = (NT < 32 ? NT : 32) / R;
  const unsigned x_bytes = TILE * sizeof(cplx) + (DIAG ? 112u : 0u);
  auto issue = [&](const cplx* base, const CUtensorMap* map, uint64_t tt, cplx* dst, uint64_t* bar) {
    if (A.load == LOAD_CONTIG) {
      if (tid == 0) bulk_g2s(dst, base + tile_index(A.sh, tt, 0), TILE * sizeof(cplx), bar);
      return;
    }
    if (A.load == LOAD_TENSOR) {
      if (tid == 0) {
        const int m = A.sh.p - A.sh.a;
        tma_load_5d(dst, map, 0, (int)(tt & ((1ull << m) - 1ull)), 0, 0, (int)(tt >> m), bar);
      }
      return;
    }
    if (lane < RUNS) {
      const uint32_t e0 = (uint32_t)(warp * 32 + lane * R);
      const cplx* src = base + tile_index(A.sh, tt, e0);
      #pragma unroll
      for (int i = 0; i < EPT; ++i) bulk_g2s(dst + e0 + i * NT, src + i * S, R * sizeof(cplx), bar);
    }
  };
  auto issue_x = [&](uint64_t tt, int b) {
    issue(A.x, &A.tm_x, tt, buf + b * TILE, &bars[b]);
    if (DIAG && tid == 0) bulk_g2s(rows + b * 16, A.dg.gc + tt * kGcStride, 112, &bars[b]);
  };

  if (!X0 && tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    mbar_init_fence();
  }
  __syncthreads();
  unsigned phase = 0u;   // bit b: parity of buffer b's next completion
  const uint64_t t0 = blockIdx.x;
  if (t0 < ntiles) {   // prologue: x(0) -> buffer 0, operand(0) -> buffer 2
    if (tid == 0) {
      if (!X0) mbar_arrive_expect_tx(&bars[0], x_bytes);
      if (has_e) mbar_arrive_expect_tx(&bars[2], TILE * sizeof(cplx));
    }
    __syncthreads();
    if (!X0) issue_x(t0, 0);
    if (has_e) issue(A.ein, &A.tm_e, t0, buf + 2 * TILE, &bars[2]);
  }
  int bx = 0;   // buffer of x(it); the operand of tile it sits in (bx + 2) % 3
  for (uint64_t t = t0; t < ntiles; t += G) {
    const int be = bx == 0 ? 2 : bx - 1;
    const int bn = bx == 2 ? 0 : bx + 1;
    const uint64_t g0 = tile_index(A.sh, t, tid);
    const uint64_t tn = t + G;
    if (tid == 0 && tn < ntiles) mbar_arrive_expect_tx(&bars[bn], x_bytes);
#if !RSV_EARLY_X
    mbar_wait(&bars[bx], (phase >> bx) & 1u);
    phase ^= 1u << bx;
#endif
    __syncthreads();   // (A) everyone is past tile it-1: its operand buffer (= bn) is free
    if (tn < ntiles) {
      if (tstore && tid == 0) bulk_wait_read0();   // ... once the TMA store of w(it-1) has read it
      issue_x(tn, bn);
    }
#if RSV_EARLY_X
    mbar_wait(&bars[bx], (phase >> bx) & 1u);   // x(it), after x(it+1) is on its way
    phase ^= 1u << bx;
#endif
    const cplx* s = buf + bx * TILE;
    DiagRow<NT, EPT> dr;
    if (DIAG) dr.setup(A.dg, A.sh, t, tid, rows + bx * 16);

    cplx xv[EPT], ac[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      xv[i] = s[tid + i * NT];
      ac[i] = make_double2(0.0, 0.0);
    }
    #pragma unroll
    for (int b = 0; b < RB; ++b) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        ac[i].x = fma(rc[b], xv[i ^ (1 << b)].x, ac[i].x);
        ac[i].y = fma(rc[b], xv[i ^ (1 << b)].y, ac[i].y);
      }
    }
    for (int f = 0; f < A.fl.count; ++f) flip_into<NT, EPT, 1>(ac, xv, s, tid, A.fl.mask[f], A.fl.coef[f] * xs);
    if (DIAG) {
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double d = dr.d[i];
        if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
        d *= xs;
        ac[i].x = fma(d, xv[i].x, ac[i].x);
        ac[i].y = fma(d, xv[i].y, ac[i].y);
      }
    }
    if (has_e && tn < ntiles) {
      if (tid == 0) mbar_arrive_expect_tx(&bars[bx], TILE * sizeof(cplx));
      __syncthreads();   // (B) everyone is past the flips on x(it): its buffer takes operand(it+1)
      issue(A.ein, &A.tm_e, tn, buf + bx * TILE, &bars[bx]);
    }
    const cplx* eb = buf + be * TILE;
    cplx* sw = buf + be * TILE;   // the same buffer receives w(it)
    if (has_e) {
      mbar_wait(&bars[be], (phase >> be) & 1u);
      phase ^= 1u << be;
    }
    cplx* po = A.out + g0;
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      double cr = ac[i].x, ci = ac[i].y;
      acc_a = fma(xv[i].x, cr, fma(xv[i].y, ci, acc_a));
      if (has_e) {
        const cplx u = eb[tid + i * NT];
        cr = fma(ecoef, u.x, cr);
        ci = fma(ecoef, u.y, ci);
      }
      if (LANCZOS) {
        cr = fma(-axs, xv[i].x, cr);
        ci = fma(-axs, xv[i].y, ci);
        acc_n = fma(cr, cr, fma(ci, ci, acc_n));
      }
      ac[i] = make_double2(cr, ci);
      if (tstore) sw[tid + i * NT] = ac[i];   // over this thread's own operand entry
      else st_stream(po + i * S, ac[i]);
    }
    if (tstore) {
      fence_proxy_async_smem();   // generic writes -> the TMA store's reads
      __syncthreads();            // w(it) complete in the operand buffer
      if (tid == 0) store_tile(A, t, sw);
    }

    if (LANCZOS && A.qsweep && !RSV_QSWEEP_OFF) {
      // w goes to the operand buffer of this tile (refilled only after the next barrier A);
      // without an operand that buffer is idle
      if (!tstore) {
        #pragma unroll
        for (int i = 0; i < EPT; ++i) sw[tid + i * NT] = ac[i];
        __syncthreads();
      }
      // <w|A_last|w> = sum over flip pairs (e, e^m) of 2 c Re(conj(w_e) w_{e^m}) (+ <w|D|w>):
      // register bits pair the thread's own amplitudes (per-bit sums, scaled once)
      #pragma unroll
      for (int b = 0; b < RB; ++b) {
        double s0 = 0.0, s1 = 0.0;
        #pragma unroll
        for (int i = 0; i < EPT; ++i) {
          if ((i >> b) & 1) continue;
          const cplx& q = ac[i ^ (1 << b)];
          if (i & 1) s1 = fma(ac[i].x, q.x, fma(ac[i].y, q.y, s1));
          else s0 = fma(ac[i].x, q.x, fma(ac[i].y, q.y, s0));
        }
        acc_q = fma(r2[b], s0 + s1, acc_q);
      }
      if (DIAG) {
        #pragma unroll
        for (int i = 0; i < EPT; ++i) {
          double d = dr.d[i];
          if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
          acc_q = fma(d, fma(ac[i].x, ac[i].x, ac[i].y * ac[i].y), acc_q);
        }
      }
      // shared-memory bits: each pair (e, e^m) once -- the partner with bit m clear takes the even
      // amplitudes, the one with bit m set the odd ones (selects instead of predication, so no issue
      // slot is spent on masked-off lanes), per-flip sums scaled once
      for (int f = 0; f < A.fl.count; ++f) {
        const int m = A.fl.mask[f];
        if (qt_mask & m) continue;   // done below in the transposed layout
        const bool own = (tid & m) != 0;
        const cplx* ps = sw + (tid ^ m) + (own ? NT : 0);
        double s0 = 0.0, s1 = 0.0;
        #pragma unroll
        for (int k = 0; k < EPT / 2; ++k) {
          const cplx p = ps[2 * k * NT];
          const double wx = own ? ac[2 * k + 1].x : ac[2 * k].x;
          const double wy = own ? ac[2 * k + 1].y : ac[2 * k].y;
          if (k & 1) s1 = fma(wx, p.x, fma(wy, p.y, s1));
          else s0 = fma(wx, p.x, fma(wy, p.y, s0));
        }
        acc_q = fma(2.0 * A.fl.coef[f], s0 + s1, acc_q);
      }
      if constexpr (kQT) {
        // tile bits 4..7 become register bits: thread tid reads w at e = (tid & 15) | (tid >> 4) << 8
        // | i << 4 (8 consecutive lanes still cover 128 contiguous bytes: conflict free), so each of
        // these flips costs one 16-byte load per amplitude for all four bits instead of a half load
        // per bit
        if (qt_mask != 0u) {
          const cplx* w2p = sw + (tid & 15) + ((tid >> 4) << 8);
          cplx w2[16];
          #pragma unroll
          for (int i = 0; i < 16; ++i) w2[i] = w2p[i << 4];
          #pragma unroll
          for (int b = 0; b < 4; ++b) {
            double s0 = 0.0, s1 = 0.0;
            #pragma unroll
            for (int i = 0; i < 16; ++i) {
              if ((i >> b) & 1) continue;
              const cplx& q = w2[i ^ (1 << b)];
              if (i & 1) s1 = fma(w2[i].x, q.x, fma(w2[i].y, q.y, s1));
              else s0 = fma(w2[i].x, q.x, fma(w2[i].y, q.y, s0));
            }
            acc_q = fma(qc[b], s0 + s1, acc_q);
          }
        }
      }
      fence_proxy_async_smem();   // generic writes to a buffer the TMA engine refills later
    }
    bx = bn;
  }
  if (tstore && tid == 0) bulk_wait0();   // the last output tile is written before the CTA exits
  acc_a *= xs;

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
  } else {
    lanczos_scalars(scw, A.j, A.raw, alpha, tot[1], tot[2], A.mail);
  }
}

template <int TB, int KIND, int NT, bool DIAG, int NPEER = 0>
__global__ void __launch_bounds__(NT, (NT >= RSV_PASS_THREADS || NT == RSV_LAST_THREADS) ? 1 : 2)
    pass_kernel_tma(const __grid_constant__ PassArgs A) {
  pass_tma_body<TB, KIND, NT, DIAG, NPEER>(A);
}
template <int TB, int KIND, int NT, bool DIAG>
__global__ void __launch_bounds__(NT, (NT >= RSV_PASS_THREADS || NT == RSV_LAST_THREADS) ? 1 : 2)
    pass_kernel_rot(const __grid_constant__ PassArgs A) {
  pass_rot_body<TB, KIND, NT, DIAG>(A);
}

// ---------------------------------------------------------------- L2-resident chunk pass
// See ChunkArgs (rsv_kernels.cuh). Work item k in [0, 2 Nt) -> (kind, tile):
//   k < lag                 : M tile k
//   lag <= k < 2 Nt - lag   : alternating M tile lag + (k-lag)/2 and L tile (k-lag)/2
//   k >= 2 Nt - lag         : the remaining L tiles
// so an L tile of chunk c is handed out ~(lag - 2^gm) x 2 items after the last M tile of c.
// Items come from one atomic ticket (fetched one item ahead, so its latency is hidden); an L
// tile's operand u' is requested only after thread 0 has acquired the chunk's M counter.
#ifndef RSV_CHUNK_HINTS
#define RSV_CHUNK_HINTS 1
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gsrc, unsigned bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_load_5d_hint(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 int c3, int c4, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;"
      ::"r"(smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(cplx* p, cplx v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
  asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct ChunkItem {
  bool is_l;
  uint64_t t;
};
__device__ __forceinline__ ChunkItem chunk_item(uint64_t k, uint64_t nt, uint64_t lag) {
  if (k < lag) return {false, k};
  if (k < 2 * nt - lag) {
    const uint64_t rel = k - lag;
    return (rel & 1) ? ChunkItem{true, rel >> 1} : ChunkItem{false, lag + (rel >> 1)};
  }
  return {true, nt - lag + (k - (2 * nt - lag))};
}

template <int NT, bool DIAG>
__global__ void __launch_bounds__(NT, 1) chunk_kernel(const __grid_constant__ ChunkArgs A) {
  constexpr int TILE = 1 << kLoBits;
  constexpr int EPT = TILE / NT;
  constexpr int RB = RegBits<EPT>::value;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  cplx* xbuf = reinterpret_cast<cplx*>(smem_al);             // [2][TILE]
  cplx* ebuf = xbuf + 2 * TILE;                               // [TILE]
  double* rows = reinterpret_cast<double*>(ebuf + TILE);     // [2][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rows + 32);   // xbar[0], xbar[1], ebar
  __shared__ double red[32];
  __shared__ unsigned long long s_item[2];   // next item (decoded), double-buffered by stage parity

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* sc = A.sc;
  const double xs = sc[A.x_scale_slot];
  const bool has_prev = A.prev != nullptr;
  const double ecoef_m = has_prev ? -(sc[SC_BE + A.j - 1] * sc[SC_SG + A.j - 1]) : 0.0;
  double acc_a = 0.0;
  const uint64_t Sm = elem_offset(A.shm, NT), Sl = elem_offset(A.shl, NT);
  const uint64_t nt = A.shl.n_tiles;
  const uint64_t total = 2 * nt;
  const uint64_t lag = A.lag;
  const unsigned tiles_per_chunk = 1u << A.gm;
#if RSV_CHUNK_HINTS
  const uint64_t pol_keep = policy_evict_last();
  const uint64_t pol_drop = policy_evict_first();
#endif

  // M-tile copy geometry (LOAD_RUNS: per-warp runs of R amplitudes)
  const int R = (1 << A.shm.a) < 32 ? (1 << A.shm.a) : 32;
  const int RUNS = 32 / R;
  auto issue_m = [&](const cplx* base, const CUtensorMap* map, uint64_t tt, cplx* dst, uint64_t* bar, bool keep) {
#if RSV_CHUNK_HINTS
    const uint64_t pol = keep ? pol_keep : pol_drop;
#endif
    if (A.load_m == LOAD_TENSOR) {
      if (tid == 0) {
        const int m = A.shm.p - A.shm.a;
#if RSV_CHUNK_HINTS
        tma_load_5d_hint(dst, map, 0, (int)(tt & ((1ull << m) - 1ull)), 0, 0, (int)(tt >> m), bar, pol);
#else
        tma_load_5d(dst, map, 0, (int)(tt & ((1ull << m) - 1ull)), 0, 0, (int)(tt >> m), bar);
#endif
      }
      return;
    }
    if (lane < RUNS) {
      const uint32_t e0 = (uint32_t)(warp * 32 + lane * R);
      const cplx* src = base + tile_index(A.shm, tt, e0);
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
#if RSV_CHUNK_HINTS
        bulk_g2s_hint(dst + e0 + i * NT, src + i * Sm, R * sizeof(cplx), bar, pol);
#else
        bulk_g2s(dst + e0 + i * NT, src + i * Sm, R * sizeof(cplx), bar);
#endif
      }
    }
  };
  // items travel decoded: code = tile << 1 | is_l, kEnd past the last item (thread 0 decodes)
  constexpr unsigned long long kEnd = ~0ull;
  auto encode = [&](unsigned long long raw) -> unsigned long long {
    if (raw >= total) return kEnd;
    const ChunkItem it = chunk_item(raw, nt, lag);
    return (it.t << 1) | (it.is_l ? 1ull : 0ull);
  };
  auto issue_x = [&](unsigned long long code, int st) {
    const ChunkItem it{(code & 1ull) != 0, code >> 1};
    if (it.is_l) {
      if (tid == 0) {
#if RSV_CHUNK_HINTS
        bulk_g2s_hint(xbuf + st * TILE, A.x + (it.t << kLoBits), TILE * sizeof(cplx), &bars[st], pol_drop);
#else
        bulk_g2s(xbuf + st * TILE, A.x + (it.t << kLoBits), TILE * sizeof(cplx), &bars[st]);
#endif
        if (DIAG) bulk_g2s(rows + st * 16, A.dg.gc + it.t * kGcStride, 112, &bars[st]);
      }
    } else {
      issue_m(A.x, &A.tm_x, it.t, xbuf + st * TILE, &bars[st], true);
    }
  };
  auto x_bytes = [&](unsigned long long code) -> unsigned {
    return TILE * sizeof(cplx) + ((DIAG && (code & 1ull)) ? 112u : 0u);
  };

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    mbar_init_fence();
    s_item[1] = encode(atomicAdd(A.ticket, 1ull));
  }
  __syncthreads();
  unsigned long long cur = s_item[1];
  unsigned long long pend = 0;
  if (tid == 0) pend = atomicAdd(A.ticket, 1ull);   // the item after cur (consumed next iteration)
  unsigned xphase = 0u, ephase = 0u;   // bit s = parity of x stage s (a register, not a local array)
  if (cur != kEnd) {
    if (tid == 0) mbar_arrive_expect_tx(&bars[0], x_bytes(cur));
    __syncthreads();
    issue_x(cur, 0);
  }
  int stage = 0;
  bool signal_pending = false;   // the previous item was an M tile whose writes are not yet published
  uint64_t signal_chunk = 0;
  while (cur != kEnd) {
    const ChunkItem it{(cur & 1ull) != 0, cur >> 1};
    const bool has_e = it.is_l || has_prev;
    if (tid == 0) {
      const unsigned long long nx = encode(pend);
      s_item[stage] = nx;
      pend = atomicAdd(A.ticket, 1ull);
      if (nx != kEnd) mbar_arrive_expect_tx(&bars[stage ^ 1], x_bytes(nx));
      if (has_e) mbar_arrive_expect_tx(&bars[2], TILE * sizeof(cplx));
    }
    mbar_wait(&bars[stage], (xphase >> stage) & 1u);
    xphase ^= 1u << stage;
    __syncthreads();   // tile cur-1 fully consumed and stored; s_item[stage] visible
    const unsigned long long next = s_item[stage];
    if (tid == 0 && signal_pending) red_release_gpu(A.done + signal_chunk, 1u);
    signal_pending = false;
    if (next != kEnd) issue_x(next, stage ^ 1);
    const uint64_t chunk = it.t >> A.gm;
    if (has_e) {
      if (it.is_l) {
        if (tid == 0) {
          while (ld_acquire_gpu(A.done + chunk) < tiles_per_chunk) __nanosleep(64);
          fence_proxy_async_global();   // generic-proxy writes of other CTAs -> async-proxy (TMA) reads
#if RSV_CHUNK_HINTS
          bulk_g2s_hint(ebuf, A.out + (it.t << kLoBits), TILE * sizeof(cplx), &bars[2], pol_drop);
#else
          bulk_g2s(ebuf, A.out + (it.t << kLoBits), TILE * sizeof(cplx), &bars[2]);
#endif
        }
      } else {
        issue_m(A.prev, &A.tm_e, it.t, ebuf, &bars[2], false);
      }
    }
    const cplx* s = xbuf + stage * TILE;
    const uint64_t g0 = it.is_l ? (it.t << kLoBits) + tid : tile_index(A.shm, it.t, tid);
    const uint64_t S = it.is_l ? Sl : Sm;
    const FlipSet& fl = it.is_l ? A.fll : A.flm;

    cplx xv[EPT], ac[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      xv[i] = s[tid + i * NT];
      ac[i] = make_double2(0.0, 0.0);
    }
    #pragma unroll
    for (int b = 0; b < RB; ++b) {
      const double c = (it.is_l ? A.fll.rcoef[b] : A.flm.rcoef[b]) * xs;
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        ac[i].x = fma(c, xv[i ^ (1 << b)].x, ac[i].x);
        ac[i].y = fma(c, xv[i ^ (1 << b)].y, ac[i].y);
      }
    }
    const int nfl = fl.count;
    for (int f = 0; f < nfl; ++f) {
      const cplx* ps = s + (tid ^ fl.mask[f]);
      const double c = fl.coef[f] * xs;
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const cplx p = ps[i * NT];
        ac[i].x = fma(c, p.x, ac[i].x);
        ac[i].y = fma(c, p.y, ac[i].y);
      }
    }
    if (DIAG && it.is_l) {
      DiagRow<NT, EPT> dr;
      dr.setup(A.dg, A.shl, it.t, tid, rows + stage * 16);
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double d = dr.d[i];
        if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + i * S);
        d *= xs;
        ac[i].x = fma(d, xv[i].x, ac[i].x);
        ac[i].y = fma(d, xv[i].y, ac[i].y);
      }
    }
    if (has_e) {
      mbar_wait(&bars[2], ephase);
      ephase ^= 1u;
    }
    const double ecoef = it.is_l ? 1.0 : ecoef_m;
    cplx* po = A.out + g0;
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      double cr = ac[i].x, ci = ac[i].y;
      acc_a = fma(xv[i].x, cr, fma(xv[i].y, ci, acc_a));
      if (has_e) {
        const cplx u = ebuf[tid + i * NT];
        cr = fma(ecoef, u.x, cr);
        ci = fma(ecoef, u.y, ci);
      }
#if RSV_CHUNK_HINTS
      st_hint(po + i * S, make_double2(cr, ci), it.is_l ? pol_drop : pol_keep);
#else
      st_stream(po + i * S, make_double2(cr, ci));
#endif
    }
    if (!it.is_l) {
      signal_pending = true;
      signal_chunk = chunk;
    }
    cur = next;
    stage ^= 1;
  }
  if (signal_pending) {
    __syncthreads();
    if (tid == 0) red_release_gpu(A.done + signal_chunk, 1u);
  }
  acc_a *= xs;

  double mine[3];
  mine[0] = block_sum<NT>(acc_a, red);
  mine[1] = 0.0;
  mine[2] = 0.0;
  double tot[3];
  if (!grid_finalize<3, NT>(mine, A.part, A.counter, tot, red)) return;
  // every CTA has left the item loop: reset the scheduler for the next launch
  const uint64_t nchunks = nt >> A.gm;
  for (uint64_t c = tid; c < nchunks; c += NT) A.done[c] = 0u;
  if (tid == 0) {
    *A.ticket = 0ull;
    A.sc[SC_AP + A.j] = tot[0];
  }
}

// ---------------------------------------------------------------- fused two-pass Lanczos iteration
#ifndef RSV_ITER2_PREFETCH
#define RSV_ITER2_PREFETCH 1
#endif
// Registers of 16..21 qubits have two passes per iteration (lo, last; 4096-amplitude tiles) over a state that lives in
// L2; each pass is then a few tiles per SM, so launch latency, the pipeline fill and the tail of
// the grid reduction are a large part of it. One cooperative launch runs both: the lo pass, a grid
// barrier (after it the lo pass's alpha share and every partial sum u are visible), the last pass.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire_gpu(bar) < gridDim.x) __nanosleep(32);
    fence_proxy_async_global();   // other CTAs' generic writes (u) -> this CTA's TMA reads
  }
  __syncthreads();
  fence_proxy_async_smem();
}

// The last pass's first x tile (s_j, ready since the launch) is requested before the grid barrier,
// so its load overlaps the wait for the other CTAs' lo tiles (contiguous / tensor-map tiles only).
__device__ __forceinline__ bool rot_issue_x0(const PassArgs& A) {
  if (A.load != LOAD_CONTIG && A.load != LOAD_TENSOR) return false;
  constexpr int TILE = 1 << kLoBits;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  cplx* buf = reinterpret_cast<cplx*>(smem_al);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(buf + 3 * TILE) + 48);
  __syncthreads();   // every thread is done with the lo pass's buffers
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    mbar_init_fence();
    const uint64_t t0 = blockIdx.x;
    if (t0 < A.sh.n_tiles) {
      mbar_arrive_expect_tx(&bars[0], TILE * sizeof(cplx));
      if (A.load == LOAD_CONTIG) {
        bulk_g2s(buf, A.x + tile_index(A.sh, t0, 0), TILE * sizeof(cplx), &bars[0]);
      } else {
        const int m = A.sh.p - A.sh.a;
        tma_load_5d(buf, &A.tm_x, 0, (int)(t0 & ((1ull << m) - 1ull)), 0, 0, (int)(t0 >> m), &bars[0]);
      }
    }
  }
  return true;
}

template <bool DIAG>
__global__ void __launch_bounds__(RSV_ITER2_THREADS, 1) iter2_kernel(const __grid_constant__ Iter2Args A) {
  pass_tma_body<kLoBits, PASS_FIRST, RSV_ITER2_THREADS, DIAG>(A.lo);
#if RSV_ITER2_PREFETCH
  const bool x0 = rot_issue_x0(A.last);
#else
  const bool x0 = false;
#endif
  grid_barrier(A.gridbar);
  if (x0) pass_rot_body<kLoBits, PASS_LAST_LANCZOS, RSV_ITER2_THREADS, false, true>(A.last);
  else pass_rot_body<kLoBits, PASS_LAST_LANCZOS, RSV_ITER2_THREADS, false>(A.last);
  // second arrival: the last CTA to get here resets the barrier for the next launch
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(A.gridbar, 1u) == 2u * gridDim.x - 1u) *A.gridbar = 0u;
}

// ---------------------------------------------------------------- Krylov combination
// psi_new = sum_i coef_i v_i streamed tile by tile, fused with the next step's ||psi||^2,
// q_0 (q-sweep with the next step's coefficients) and the observable masks. Observables
// are reduced per warp into shared rows (no block barriers inside the tile loop).
template <int TB, int NT>
__global__ void __launch_bounds__(NT, NT >= RSV_COMBINE_THREADS ? 1 : 2) combine_kernel(const __grid_constant__ CombineArgs A) {
  constexpr int TILE = 1 << TB;
  constexpr int EPT = TILE / NT;
  constexpr int RB = RegBits<EPT>::value;
  constexpr int NW = (NT + 31) / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cplx* s = reinterpret_cast<cplx*>(smem_raw);
  __shared__ double red[32];
  __shared__ double s_obs[NW][kMaxMasks];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool has_diag = A.qsweep && A.dg.mode != DIAG_NONE;
  for (int m = lane; m < A.nmask; m += 32) s_obs[warp][m] = 0.0;
  // single-bit masks (occupations): a bit is a register bit of the thread, a thread-index bit or
  // constant over the tile; per-thread accumulators replace the per-mask warp reduction of every
  // tile (one warp sum per tile for the tile-constant bits, block sums once at the end)
  constexpr int LT = Log2<NT>::value;
  const bool single = A.obs_single != 0;
  double occ_p = 0.0, occ_r[RB > 0 ? RB : 1];
  #pragma unroll
  for (int b = 0; b < RB; ++b) occ_r[b] = 0.0;
  double acc_n = 0.0, acc_q = 0.0;
  uint64_t off[EPT];
  #pragma unroll
  for (int i = 0; i < EPT; ++i) off[i] = elem_offset(A.sh, i * NT);

  // The k vectors of a tile stream through a 3-stage cp.async ring (two items in flight per
  // thread). Each thread copies and reads only its own amplitudes, so the ring needs no block
  // barriers; the q-sweep reuses the stage of a tile's last vector.
  constexpr int RING = 3;
  const uint64_t G = gridDim.x;
  const int kv = A.k;
  uint64_t is_t = blockIdx.x;   // next (tile, vector, stage) to request
  int is_v = 0, is_s = 0;
#if RSV_COMBINE_TMA
  // TMA variant: each warp's amplitudes arrive by bulk copies of their contiguous runs, completion
  // on a per-warp mbarrier per stage (no LSU traffic for the copies; the ring stays warp-private)
  uint64_t* wbar = reinterpret_cast<uint64_t*>(s + RING * TILE);   // [RING][NW]
  const int R = (1 << A.sh.a) < 32 ? (1 << A.sh.a) : (NT < 32 ? NT : 32);
  const int RUNS = (NT < 32 ? NT : 32) / R;
  const unsigned warp_bytes = (unsigned)((NT < 32 ? NT : 32) * EPT * sizeof(cplx));
  if (lane == 0)
    for (int st = 0; st < RING; ++st) mbar_init(&wbar[st * NW + warp], 1);
  mbar_init_fence();
  __syncthreads();
  unsigned wphase = 0u;
  auto issue_next = [&]() {
    if (is_t < A.sh.n_tiles) {
      uint64_t* bar = &wbar[is_s * NW + warp];
      __syncwarp();                 // the warp is done with this stage's previous contents
      fence_proxy_async_smem();
      if (lane == 0) mbar_arrive_expect_tx(bar, warp_bytes);
      __syncwarp();
      if (lane < RUNS) {
        const uint32_t e0 = (uint32_t)(warp * 32 + lane * R);
        const cplx* src = A.v[is_v] + tile_index(A.sh, is_t, e0);
        cplx* dst = s + is_s * TILE + e0;
        #pragma unroll
        for (int i = 0; i < EPT; ++i) bulk_g2s(dst + i * NT, src + off[i], R * sizeof(cplx), bar);
      }
      if (++is_v == kv) {
        is_v = 0;
        is_t += G;
      }
    }
    is_s = is_s == RING - 1 ? 0 : is_s + 1;
  };
  auto wait_item = [&](int st) {
    mbar_wait(&wbar[st * NW + warp], (wphase >> st) & 1u);
    wphase ^= 1u << st;
  };
#else
  auto issue_next = [&]() {
    if (is_t < A.sh.n_tiles) {
      const cplx* src = A.v[is_v] + tile_index(A.sh, is_t, tid);
      cplx* dst = s + is_s * TILE + tid;
      #pragma unroll
      for (int i = 0; i < EPT; ++i) cp_async16(dst + i * NT, src + off[i]);
      if (++is_v == kv) {
        is_v = 0;
        is_t += G;
      }
    }
    cp_async_commit();
    is_s = is_s == RING - 1 ? 0 : is_s + 1;
  };
  auto wait_item = [&](int) { cp_async_wait<1>(); };   // this item landed; the next may be in flight
#endif
  issue_next();
  issue_next();
  int stage = 0;
  for (uint64_t t = blockIdx.x; t < A.sh.n_tiles; t += gridDim.x) {
    const uint64_t g0 = tile_index(A.sh, t, tid);
    cplx wv[EPT];
    #pragma unroll
    for (int i = 0; i < EPT; ++i) wv[i] = make_double2(0.0, 0.0);
    int qstage = 0;
    for (int k = 0; k < kv; ++k) {
      wait_item(stage);
      const cplx* src = s + stage * TILE + tid;
      const double2 c = A.coef[k];
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const cplx x = src[i * NT];
        wv[i].x = fma(c.x, x.x, fma(-c.y, x.y, wv[i].x));
        wv[i].y = fma(c.x, x.y, fma(c.y, x.x, wv[i].y));
      }
      issue_next();         // into the stage consumed one item ago
      qstage = stage;
      stage = stage == RING - 1 ? 0 : stage + 1;
    }
    #pragma unroll
    for (int i = 0; i < EPT; ++i) {
      if (A.out != nullptr) st_stream(A.out + g0 + off[i], wv[i]);
      acc_n = fma(wv[i].x, wv[i].x, fma(wv[i].y, wv[i].y, acc_n));
    }
    if (A.qsweep) {
      DiagRow<NT, EPT> dr;
      if (has_diag) dr.setup(A.dg, A.sh, t, tid, nullptr);
      cplx* sw = s + qstage * TILE;   // refilled only after the second barrier below
      #pragma unroll
      for (int i = 0; i < EPT; ++i) sw[tid + i * NT] = wv[i];
      __syncthreads();
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        double hr = 0.0, hi = 0.0;
        #pragma unroll
        for (int b = 0; b < RB; ++b) {
          hr = fma(A.fl.rcoef[b], wv[i ^ (1 << b)].x, hr);
          hi = fma(A.fl.rcoef[b], wv[i ^ (1 << b)].y, hi);
        }
        if (has_diag) {
          double d = dr.d[i];
          if (A.dg.mode == DIAG_VEC) d += __ldcs(A.dg.dvec + g0 + off[i]);
          hr = fma(d, wv[i].x, hr);
          hi = fma(d, wv[i].y, hi);
        }
        acc_q = fma(wv[i].x, hr, fma(wv[i].y, hi, acc_q));
      }
      for (int f = 0; f < A.fl.count; ++f) {
        const int m = A.fl.mask[f];
        const double c = A.fl.coef[f];
        #pragma unroll
        for (int i = 0; i < EPT; ++i) {
          const cplx p = sw[(tid + i * NT) ^ m];
          acc_q = fma(c, fma(wv[i].x, p.x, wv[i].y * p.y), acc_q);
        }
      }
      __syncthreads();
    } else {
      // keep the CTA's warps on the same tile: without it they drift apart over (tile, vector) items
      // and the k-vector stream loses DRAM locality (measured: 21 vectors at 1.9 vs 5.3 TB/s)
      __syncthreads();
    }
    if (A.nmask > 0 && single) {
      double ps = 0.0;
      #pragma unroll
      for (int i = 0; i < EPT; ++i) {
        const double pi = wv[i].x * wv[i].x + wv[i].y * wv[i].y;
        ps += pi;
        #pragma unroll
        for (int b = 0; b < RB; ++b)
          if ((i >> b) & 1) occ_r[b] += pi;
      }
      occ_p += ps;
      const double wsum = warp_sum<NT>(ps);
      if (lane == 0)
        for (int m = 0; m < A.nmask; ++m)
          if (A.obs_cat[m] == 0 && ((g0 >> A.obs_pos[m]) & 1ull)) s_obs[warp][m] += wsum;
    } else if (A.nmask > 0) {
      double p[EPT];
      #pragma unroll
      for (int i = 0; i < EPT; ++i) p[i] = wv[i].x * wv[i].x + wv[i].y * wv[i].y;
      for (int m = 0; m < A.nmask; ++m) {
        const uint64_t M = A.mask[m];
        double v = 0.0;
        #pragma unroll
        for (int i = 0; i < EPT; ++i) v += (((g0 + off[i]) & M) == M) ? p[i] : 0.0;
        v = warp_sum<NT>(v);
        if (lane == 0) s_obs[warp][m] += v;
      }
    }
  }

#if !RSV_COMBINE_TMA
  cp_async_wait<0>();
#endif
  double mine[2];
  mine[0] = block_sum<NT>(acc_n, red);
  mine[1] = block_sum<NT>(acc_q, red);
  constexpr int stride = 2 + kMaxMasks;
  if (tid == 0) {
    A.part[(size_t)blockIdx.x * stride + 0] = mine[0];
    A.part[(size_t)blockIdx.x * stride + 1] = mine[1];
  }
  __shared__ double s_bit[16];   // single-bit masks: CTA sums per thread-index bit / register bit
  if (single && A.nmask > 0) {
    for (int pos = 0; pos < LT; ++pos) {
      const double v = block_sum<NT>(((tid >> pos) & 1) ? occ_p : 0.0, red);
      if (tid == 0) s_bit[pos] = v;
    }
    #pragma unroll
    for (int b = 0; b < RB; ++b) {
      const double v = block_sum<NT>(occ_r[b], red);
      if (tid == 0) s_bit[LT + b] = v;
    }
    __syncthreads();
  }
  for (int m = tid; m < A.nmask; m += NT) {
    double v = 0.0;
    if (single && A.obs_cat[m] != 0) {
      v = s_bit[A.obs_cat[m] == 1 ? A.obs_pos[m] : LT + A.obs_pos[m]];
    } else {
      #pragma unroll
      for (int w = 0; w < NW; ++w) v += s_obs[w][m];
    }
    A.part[(size_t)blockIdx.x * stride + 2 + m] = v;
  }
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned tk = atomicAdd(A.counter, 1u);
    s_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ncol = 2 + A.nmask;
  double tot[2] = {0.0, 0.0};
  for (int c = 0; c < ncol; ++c) {
    double v = 0.0;
    for (unsigned r = tid; r < gridDim.x; r += NT) v += __ldcg(A.part + (size_t)r * stride + c);
    const double sum = block_sum<NT>(v, red);
    if (c < 2) tot[c] = sum;
    else if (tid == 0) A.sc[SC_OBS + c - 2] = sum;   // raw sums; the host divides by ||psi||^2
  }
  if (tid == 0) {
    *A.counter = 0u;
    if (A.sc_out >= 0) {   // re-orthogonalisation: raw ||w||^2 and <w|A_last|w> to scratch slots
      A.sc[A.sc_out] = tot[0];
      A.sc[A.sc_out + 1] = tot[1];
      return;
    }
    A.sc[SC_N0SQ] = tot[0];
    if (A.raw) {   // sharded: the host all-reduces ||psi||^2, <psi|A|psi> and the masks, then finishes
      A.sc[SC_Q + 0] = tot[1];
    } else {
      A.sc[SC_SG + 0] = tot[0] > 0.0 ? 1.0 / sqrt(tot[0]) : 0.0;
      A.sc[SC_Q + 0] = tot[0] > 0.0 ? tot[1] / tot[0] : 0.0;
    }
  }
}

// ---------------------------------------------------------------- tables and helpers
__global__ void build_dl_kernel(int a, int n, const double* __restrict__ umat, DiagArgs dg, int with_interaction,
                                double offset, double* __restrict__ dl) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (1 << a)) return;
  double v = offset;   // sharded runs: the constant energy of the shard's global bits
  for (int i = 0; i < a; ++i) {
    if (!((e >> i) & 1)) continue;
    v -= dg.delta[i];
    if (with_interaction)
      for (int j = i + 1; j < a; ++j)
        if ((e >> j) & 1) v += umat[(size_t)i * n + j];
  }
  dl[e] = v;
}

// Per-run tile table of the lo pass, row t: gc[t][i] = sum_{j>=a} U_ij bit_j(t) (i < a, cols 0..11),
// hh[t] = sum_{a<=i<j} U_ij bit_i(t) bit_j(t) (col 12); col 13 (tb) is filled per step.
__global__ void build_tile_table_kernel(int a, int n, const double* __restrict__ umat, uint64_t ntiles,
                                        double* __restrict__ gc) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    double* row = gc + t * kGcStride;
    for (int i = 0; i < 12; ++i) {
      double g = 0.0;
      if (i < a)
        for (int j = a; j < n; ++j)
          if ((t >> (j - a)) & 1ull) g += umat[(size_t)i * n + j];
      row[i] = g;
    }
    double hh = 0.0;
    for (int i = a; i < n; ++i) {
      if (!((t >> (i - a)) & 1ull)) continue;
      for (int j = i + 1; j < n; ++j)
        if ((t >> (j - a)) & 1ull) hh += umat[(size_t)i * n + j];
    }
    row[12] = hh;
    row[13] = hh;
  }
}

// Per-step tile base (col 13): tb[t] = hh[t] (fly) - sum_{j>=a} delta_j bit_j(t).
__global__ void build_tile_base_kernel(int a, int n, int fly, DiagArgs dg, uint64_t ntiles, double* __restrict__ gc) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    double v = fly ? gc[t * kGcStride + 12] : 0.0;
    for (int j = a; j < n; ++j)
      if ((t >> (j - a)) & 1ull) v -= dg.delta[j];
    gc[t * kGcStride + 13] = v;
  }
}

// Diagonal -sum_i delta_i bit_i + sum_{i<j} U_ij bit_i bit_j for every index
// (precomputed-vector variant, sv.py:116; rydsim/hamiltonian.py:114 build_diagonal).
__global__ void interaction_diag_kernel(int n, const double* __restrict__ umat, DiagArgs dg, int with_delta,
                                        double* __restrict__ dvec) {
  __shared__ double su[kMaxQubits * kMaxQubits];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) su[i] = umat[i];
  __syncthreads();
  const uint64_t total = 1ull << n;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < total; b += (uint64_t)gridDim.x * blockDim.x) {
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

__global__ void zdotc_kernel(const cplx* __restrict__ x, const cplx* __restrict__ y, uint64_t n, double* part,
                             unsigned* counter, double* result2) {
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
  if (threadIdx.x == 0) {
    result2[0] = tot[0];
    result2[1] = tot[1];
  }
}

// sum |x - y|^2 (norm_difference, observables.py:137, without cancellation)
__global__ void diff_norm_kernel(const cplx* __restrict__ x, const cplx* __restrict__ y, uint64_t n, double* part,
                                 unsigned* counter, double* result) {
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
__global__ void lanczos_update_kernel(cplx* __restrict__ w, const cplx* __restrict__ v, const cplx* __restrict__ vprev,
                                      double alpha, double beta, uint64_t n, double* part, unsigned* counter,
                                      double* result) {
  __shared__ double red[32];
  double nn = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    cplx a = w[i];
    const cplx b = v[i];
    a.x -= alpha * b.x;
    a.y -= alpha * b.y;
    if (vprev != nullptr) {
      const cplx c = vprev[i];
      a.x -= beta * c.x;
      a.y -= beta * c.y;
    }
    w[i] = a;
    nn = fma(a.x, a.x, fma(a.y, a.y, nn));
  }
  double mine[1] = {block_sum<kThreads>(nn, red)};
  double tot[1];
  if (!grid_finalize<1, kThreads>(mine, part, counter, tot, red)) return;
  if (threadIdx.x == 0) result[0] = tot[0];
}

// Flip of a sharded (global) qubit: u += c * x_peer (the partner shard's amplitudes, same local
// index) and dot = Re <x|x_peer> for the qubit's share of alpha (sharding.py; krylov.py:96-99).
__global__ void global_flip_kernel(cplx* __restrict__ u, const cplx* __restrict__ xp, const cplx* __restrict__ x,
                                   double c, uint64_t n, double* part, unsigned* counter, double* result) {
  __shared__ double red[32];
  double dot = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const cplx p = xp[i], xi = x[i];
    cplx a = u[i];
    a.x = fma(c, p.x, a.x);
    a.y = fma(c, p.y, a.y);
    u[i] = a;
    dot = fma(xi.x, p.x, fma(xi.y, p.y, dot));
  }
  double mine[1] = {block_sum<kThreads>(dot, red)};
  double tot[1];
  if (!grid_finalize<1, kThreads>(mine, part, counter, tot, red)) return;
  if (threadIdx.x == 0) result[0] = tot[0];
}

// ---- bitstring sampling (observables.py:167 sample_bitstrings, dense inverse-CDF path)
// chunk sums of |psi|^2 in a fixed order; the host prefixes them (float64) and each shot is
// resolved by one warp: binary search over the chunk prefixes, then a warp-scan walk inside
// the chunk to the first index whose running sum exceeds u * total (searchsorted side="right").
constexpr int kSampleChunkLog2 = 12;

__global__ void chunk_norms_kernel(const cplx* __restrict__ psi, uint64_t n, double* __restrict__ sums) {
  __shared__ double red[32];
  const uint64_t chunk = 1ull << kSampleChunkLog2;
  const uint64_t base = (uint64_t)blockIdx.x * chunk;
  const uint64_t len = n - base < chunk ? n - base : chunk;
  double v = 0.0;
  for (uint64_t i = threadIdx.x; i < len; i += kThreads) {
    const cplx a = psi[base + i];
    v = fma(a.x, a.x, fma(a.y, a.y, v));
  }
  v = block_sum<kThreads>(v, red);
  if (threadIdx.x == 0) sums[blockIdx.x] = v;
}

__global__ void sample_kernel(const cplx* __restrict__ psi, uint64_t n, const double* __restrict__ prefix,
                              uint64_t nchunks, const double* __restrict__ u, double total, int64_t shots,
                              int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t shot = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (shot >= shots) return;
  const double target = u[shot] * total;
  // largest chunk c with prefix[c] <= target (prefix[0] = 0, prefix[nchunks] = total)
  uint64_t lo = 0, hi = nchunks;   // invariant: prefix[lo] <= target, answer < hi
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= target) lo = mid;
    else hi = mid;
  }
  const uint64_t chunk = 1ull << kSampleChunkLog2;
  int64_t result = (int64_t)n - 1;   // cdf[-1] = 1: a target at or past the total maps to the last index
  for (uint64_t c = lo; c < nchunks; ++c) {
    double running = prefix[c];
    const uint64_t base = c * chunk;
    const uint64_t len = n - base < chunk ? n - base : chunk;
    bool found = false;
    for (uint64_t off = 0; off < len; off += 32) {
      double v = 0.0;
      if (off + lane < len) {
        const cplx a = psi[base + off + lane];
        v = fma(a.x, a.x, a.y * a.y);
      }
      #pragma unroll
      for (int d = 1; d < 32; d <<= 1) {   // inclusive warp scan (fixed order)
        const double t = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += t;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, (off + lane < len) && (running + v > target));
      if (hit) {
        result = (int64_t)(base + off + (uint64_t)(__ffs(hit) - 1));
        found = true;
        break;
      }
      running += __shfl_sync(0xffffffffu, v, 31);
    }
    if (found) break;
  }
  if (lane == 0) out[shot] = result;
}

// <s_i|w> for i < k (complex), one pass over w and the k vectors; deterministic per-CTA rows
// (re-orthogonalisation of the fused Lanczos step, krylov.py:103-104).
// <v_i|w> for the whole basis in ONE pass over w (re-orthogonalisation, krylov.py:104): a CTA holds
// kThreads x 8 amplitudes of w in registers and streams every v_i over them, so w is read once and
// each v_i once ((k+1) x 16 B per amplitude). Per vector and chunk each warp reduces its share with
// shuffles into its own row of shared accumulators; rows and CTAs are summed in fixed order.
__global__ void __launch_bounds__(kThreads) multidot_kernel(const MultiDotArgs A) {
  constexpr int EPT = 8;
  constexpr int NW = kThreads / 32;
  __shared__ double s_acc[NW][2 * kMaxKrylov];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n = A.n;
  const int ncol = 2 * A.k;
  for (int c = lane; c < ncol; c += 32) s_acc[warp][c] = 0.0;
  const uint64_t chunk = (uint64_t)kThreads * EPT;
  for (uint64_t base = blockIdx.x * chunk; base < n; base += (uint64_t)gridDim.x * chunk) {
    cplx wv[EPT];
    #pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const uint64_t e = base + threadIdx.x + (uint64_t)j * kThreads;
      wv[j] = e < n ? __ldcs(A.w + e) : make_double2(0.0, 0.0);
    }
    for (int i = 0; i < A.k; ++i) {
      const cplx* v = A.v[i];
      double re = 0.0, im = 0.0;
      #pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const uint64_t e = base + threadIdx.x + (uint64_t)j * kThreads;
        const cplx a = e < n ? __ldcs(v + e) : make_double2(0.0, 0.0);
        re = fma(a.x, wv[j].x, fma(a.y, wv[j].y, re));   // conj(a) w
        im = fma(a.x, wv[j].y, fma(-a.y, wv[j].x, im));
      }
      re = warp_sum<32>(re);
      im = warp_sum<32>(im);
      if (lane == 0) {
        s_acc[warp][2 * i] += re;
        s_acc[warp][2 * i + 1] += im;
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncol; c += kThreads) {
    double v = 0.0;
    #pragma unroll
    for (int w = 0; w < NW; ++w) v += s_acc[w][c];
    A.part[(size_t)blockIdx.x * A.stride + c] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(A.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int c = threadIdx.x; c < ncol; c += kThreads) {
    double v = 0.0;
    for (unsigned r = 0; r < gridDim.x; ++r) v += __ldcg(A.part + (size_t)r * A.stride + c);   // fixed order
    A.out[c] = v;
  }
  if (threadIdx.x == 0) *A.counter = 0u;
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

unsigned flat_grid(uint64_t n, int grid) {
  if (grid > 0) return (unsigned)grid;
  uint64_t blocks = (n + kThreads - 1) / kThreads;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

// Launch with grid = min(tiles, SMs x resident CTAs); the occupancy query is done once per kernel.
// Experiment switch: grid of the HBM-bound lo pass (0 = one CTA per SM); fewer CTAs draw less
// power under the 1 kW cap, which the SM-bound passes could use as clock.
#ifndef RSV_GRID_LO
#define RSV_GRID_LO 0
#endif

template <typename Kernel, typename Args>
cudaError_t launch_persistent(Kernel kern, const Args& args, uint64_t ntiles, int nt, size_t smem, int* occ_cache,
                              cudaStream_t st, unsigned grid_cap = 0) {
  if (*occ_cache == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
    if (e != cudaSuccess) return e;
    *occ_cache = occ > 0 ? occ : 1;
  }
  uint64_t cap = (uint64_t)num_sms() * (uint64_t)*occ_cache;
  if (grid_cap > 0 && grid_cap < cap) cap = grid_cap;
  const unsigned grid = (unsigned)(ntiles < cap ? ntiles : cap);
  kern<<<grid, nt, smem, st>>>(args);
  return cudaGetLastError();
}

template <int TB, int KIND, bool DIAG, int NPEER>
cudaError_t launch_peer_pass(const PassArgs& args, cudaStream_t st) {
  constexpr size_t smem_peer = 3 * (1 << TB) * sizeof(cplx) + 32 * sizeof(double) + 4 * sizeof(uint64_t) + 128 +
                               kPeerRingBytes;
  if (peer_pass_threads(KIND, args.sh.a) == RSV_LAST_THREADS) {
    static int occ_p256 = 0;
    return launch_persistent(pass_kernel_tma<TB, KIND, RSV_LAST_THREADS, DIAG, NPEER>, args, args.sh.n_tiles,
                             RSV_LAST_THREADS, smem_peer, &occ_p256, st);
  }
  if constexpr (pass_threads(TB) != RSV_LAST_THREADS) {
    static int occ_p = 0;
    return launch_persistent(pass_kernel_tma<TB, KIND, pass_threads(TB), DIAG, NPEER>, args, args.sh.n_tiles,
                             pass_threads(TB), smem_peer, &occ_p, st);
  }
  return cudaErrorInvalidValue;
}

template <int TB, int KIND, bool DIAG>
cudaError_t launch_pass_tbkd(const PassArgs& args, cudaStream_t st) {
  constexpr int NT = pass_threads(TB);
#if RSV_TMA && RSV_ROT
  // measured at N=26/29: the prefetched operand pays off in the last pass (its q-sweep leaves
  // less time to hide the operand load); the lo/mid passes are faster without the extra barrier
  if constexpr (TB >= 3 && (KIND == PASS_LAST_LANCZOS || (RSV_ROT_MID && KIND == PASS_MID))) {
    constexpr size_t smem_rot = 3 * (1 << TB) * sizeof(cplx) + 48 * sizeof(double) + 4 * sizeof(uint64_t) + 128;
    if constexpr (TB == kLoBits && RSV_LAST_THREADS != NT) {
      if (pass_threads_for(TB, KIND, args.sh.a) == RSV_LAST_THREADS) {
        static int occ_last = 0;
        return launch_persistent(pass_kernel_rot<TB, KIND, RSV_LAST_THREADS, DIAG>, args, args.sh.n_tiles,
                                 RSV_LAST_THREADS, smem_rot, &occ_last, st);
      }
    }
    static int occ_rot = 0;
    return launch_persistent(pass_kernel_rot<TB, KIND, NT, DIAG>, args, args.sh.n_tiles, NT, smem_rot, &occ_rot,
                             st);
  }
#endif
#if RSV_TMA
  if constexpr (TB == kLoBits && (KIND == PASS_FIRST || KIND == PASS_MID)) {
    if (args.npeer > 0 && args.npeer <= 2 && args.peer_tma) {   // partner tiles through the TMA ring
      if (args.npeer == 1) return launch_peer_pass<TB, KIND, DIAG, 1>(args, st);
      return launch_peer_pass<TB, KIND, DIAG, 2>(args, st);
    }
  }
  if constexpr (TB >= 3) {
    constexpr size_t smem_tma = 3 * (1 << TB) * sizeof(cplx) + 32 * sizeof(double) + 4 * sizeof(uint64_t) + 128;
    if constexpr (DIAG && TB == kLoBits) {
      // diag="vec" on contiguous tiles: the diagonal tile is staged in shared memory (+32 KB)
      if (args.dg.mode == DIAG_VEC && args.load == LOAD_CONTIG && RSV_DVEC_SMEM) {
        constexpr size_t pring_off = (3 * (1 << TB) * sizeof(cplx) + 32 * sizeof(double) + 4 * sizeof(uint64_t) + 127) &
                                     ~size_t(127);
        constexpr size_t smem_dv = pring_off + (1 << TB) * sizeof(double) + 128;
        PassArgs a2 = args;
        a2.dvec_smem = 1;
        if (pass_threads_for(TB, KIND, args.sh.a) == RSV_LAST_THREADS) {
          static int occ_dv256 = 0;
          return launch_persistent(pass_kernel_tma<TB, KIND, RSV_LAST_THREADS, DIAG>, a2, args.sh.n_tiles,
                                   RSV_LAST_THREADS, smem_dv, &occ_dv256, st);
        }
        static int occ_dv = 0;
        return launch_persistent(pass_kernel_tma<TB, KIND, NT, DIAG>, a2, args.sh.n_tiles, NT, smem_dv, &occ_dv, st);
      }
    }
    if constexpr (TB == kLoBits && KIND == PASS_MID && RSV_MID_THREADS != RSV_LAST_THREADS &&
                  RSV_MID_THREADS != NT) {
      if (pass_threads_for(TB, KIND, args.sh.a) == RSV_MID_THREADS) {
        static int occ_mid128 = 0;
        return launch_persistent(pass_kernel_tma<TB, KIND, RSV_MID_THREADS, DIAG>, args, args.sh.n_tiles,
                                 RSV_MID_THREADS, smem_tma, &occ_mid128, st);
      }
    }
    if constexpr (TB == kLoBits && (KIND == PASS_MID || (RSV_LO_LAST_THREADS && KIND == PASS_FIRST)) &&
                  RSV_LAST_THREADS != NT) {
      if (pass_threads_for(TB, KIND, args.sh.a) == RSV_LAST_THREADS) {
        static int occ_mid = 0;
        return launch_persistent(pass_kernel_tma<TB, KIND, RSV_LAST_THREADS, DIAG>, args, args.sh.n_tiles,
                                 RSV_LAST_THREADS, smem_tma, &occ_mid, st);
      }
    }
    static int occ_tma = 0;
    return launch_persistent(pass_kernel_tma<TB, KIND, NT, DIAG>, args, args.sh.n_tiles, NT, smem_tma, &occ_tma,
                             st, (KIND == PASS_FIRST && DIAG) ? RSV_GRID_LO : 0u);
  }
#endif
  constexpr int STAGES = TB >= 8 ? RSV_STAGES : 2;
  static int occ = 0;
  constexpr size_t smem = (STAGES + 1) * (1 << TB) * sizeof(cplx) + STAGES * 16 * sizeof(double);
  return launch_persistent(pass_kernel<TB, KIND, NT, DIAG>, args, args.sh.n_tiles, NT, smem, &occ, st);
}

template <int TB, int KIND>
cudaError_t launch_pass_tbk(const PassArgs& args, cudaStream_t st) {
  // the diagonal lives in the lo pass only: the middle passes never carry it
  if constexpr (KIND == PASS_MID) {
    return launch_pass_tbkd<TB, KIND, false>(args, st);
  } else {
    if (args.dg.mode != DIAG_NONE) return launch_pass_tbkd<TB, KIND, true>(args, st);
    return launch_pass_tbkd<TB, KIND, false>(args, st);
  }
}

template <int TB>
cudaError_t launch_pass_tb(const PassArgs& args, cudaStream_t st) {
  switch (args.kind) {
    case PASS_FIRST: return launch_pass_tbk<TB, PASS_FIRST>(args, st);
    case PASS_MID: return launch_pass_tbk<TB, PASS_MID>(args, st);
    case PASS_LAST_APPLY: return launch_pass_tbk<TB, PASS_LAST_APPLY>(args, st);
    case PASS_LAST_LANCZOS: return launch_pass_tbk<TB, PASS_LAST_LANCZOS>(args, st);
    default: return cudaErrorInvalidValue;
  }
}

template <bool DIAG>
cudaError_t launch_chunk_d(const ChunkArgs& args, cudaStream_t st) {
  constexpr int NT = RSV_CHUNK_THREADS;
  static int occ = 0;
  constexpr size_t smem = 3 * (1 << kLoBits) * sizeof(cplx) + 32 * sizeof(double) + 4 * sizeof(uint64_t) + 128;
  // tiles are handed out dynamically: the grid only needs to be resident (persistent)
  return launch_persistent(chunk_kernel<NT, DIAG>, args, 2 * args.shl.n_tiles, NT, smem, &occ, st);
}

template <bool DIAG>
cudaError_t launch_iter2_d(const Iter2Args& args, cudaStream_t st) {
  constexpr int NT = RSV_ITER2_THREADS;
  constexpr size_t smem = 3 * (1 << kLoBits) * sizeof(cplx) + 48 * sizeof(double) + 4 * sizeof(uint64_t) + 128;
  auto kern = iter2_kernel<DIAG>;
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorCooperativeLaunchTooLarge;
  }
  const uint64_t tiles = std::max(args.lo.sh.n_tiles, args.last.sh.n_tiles);
  const uint64_t cap = (uint64_t)num_sms() * (uint64_t)occ;   // every CTA resident: the grid barrier
  const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
  void* params[] = {const_cast<Iter2Args*>(&args)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(NT), params, smem, st);
}

template <int TB>
cudaError_t launch_combine_tb(const CombineArgs& args, cudaStream_t st) {
  constexpr int NT = combine_threads(TB);
  static int occ = 0;
  return launch_persistent(combine_kernel<TB, NT>, args, args.sh.n_tiles, NT,
                           3 * (1 << TB) * sizeof(cplx) + (RSV_COMBINE_TMA ? 3 * 32 * sizeof(uint64_t) : 0), &occ, st);
}

}  // namespace

cudaError_t launch_iter2(const Iter2Args& args, cudaStream_t st) {
  if (args.lo.sh.a + args.lo.sh.g != kLoBits || args.last.sh.a + args.last.sh.g != kLoBits)
    return cudaErrorInvalidValue;
  return args.lo.dg.mode != DIAG_NONE ? launch_iter2_d<true>(args, st) : launch_iter2_d<false>(args, st);
}

cudaError_t launch_pass(const PassArgs& args, cudaStream_t st) {
  switch (args.sh.a + args.sh.g) {
    case 1: return launch_pass_tb<1>(args, st);
    case 2: return launch_pass_tb<2>(args, st);
    case 3: return launch_pass_tb<3>(args, st);
    case 4: return launch_pass_tb<4>(args, st);
    case 5: return launch_pass_tb<5>(args, st);
    case 6: return launch_pass_tb<6>(args, st);
    case 7: return launch_pass_tb<7>(args, st);
    case 8: return launch_pass_tb<8>(args, st);
    case 9: return launch_pass_tb<9>(args, st);
    case 10: return launch_pass_tb<10>(args, st);
    case 11: return launch_pass_tb<11>(args, st);
    case 12: return launch_pass_tb<12>(args, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_combine(const CombineArgs& args, cudaStream_t st) {
  switch (args.sh.a + args.sh.g) {
    case 1: return launch_combine_tb<1>(args, st);
    case 2: return launch_combine_tb<2>(args, st);
    case 3: return launch_combine_tb<3>(args, st);
    case 4: return launch_combine_tb<4>(args, st);
    case 5: return launch_combine_tb<5>(args, st);
    case 6: return launch_combine_tb<6>(args, st);
    case 7: return launch_combine_tb<7>(args, st);
    case 8: return launch_combine_tb<8>(args, st);
    case 9: return launch_combine_tb<9>(args, st);
    case 10: return launch_combine_tb<10>(args, st);
    case 11: return launch_combine_tb<11>(args, st);
    case 12: return launch_combine_tb<12>(args, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_chunk(const ChunkArgs& args, cudaStream_t st) {
  if (args.dg.mode != DIAG_NONE) return launch_chunk_d<true>(args, st);
  return launch_chunk_d<false>(args, st);
}

cudaError_t launch_build_dl(int a, int n, const double* umat, const double* delta_host, int with_interaction,
                            double offset, double* dl, cudaStream_t st) {
  DiagArgs dg{};
  if (delta_host != nullptr)
    for (int i = 0; i < n && i < kMaxQubits; ++i) dg.delta[i] = delta_host[i];
  const int total = 1 << a;
  const int nt = total < 256 ? total : 256;
  build_dl_kernel<<<(total + nt - 1) / nt, nt, 0, st>>>(a, n, umat, dg, with_interaction, offset, dl);
  return cudaGetLastError();
}

cudaError_t launch_tile_table(int a, int n, const double* umat, double* gc, cudaStream_t st) {
  const uint64_t ntiles = 1ull << (n - a);
  uint64_t blocks = (ntiles + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  build_tile_table_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, n, umat, ntiles, gc);
  return cudaGetLastError();
}

cudaError_t launch_tile_base(int a, int n, int fly, const double* delta_host, double* gc, cudaStream_t st) {
  const uint64_t ntiles = 1ull << (n - a);
  uint64_t blocks = (ntiles + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  DiagArgs dg{};
  for (int i = 0; i < n && i < kMaxQubits; ++i) dg.delta[i] = delta_host[i];
  build_tile_base_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, n, fly, dg, ntiles, gc);
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

cudaError_t launch_zdotc(const cplx* x, const cplx* y, uint64_t n, double* part, unsigned* counter, double* result2,
                         int grid, cudaStream_t st) {
  zdotc_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(x, y, n, part, counter, result2);
  return cudaGetLastError();
}

cudaError_t launch_diff_norm(const cplx* x, const cplx* y, uint64_t n, double* part, unsigned* counter, double* result,
                             int grid, cudaStream_t st) {
  diff_norm_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(x, y, n, part, counter, result);
  return cudaGetLastError();
}

cudaError_t launch_lanczos_update(cplx* w, const cplx* v, const cplx* vprev, double alpha, double beta, uint64_t n,
                                  double* part, unsigned* counter, double* result, int grid, cudaStream_t st) {
  lanczos_update_kernel<<<flat_grid(n, grid), kThreads, 0, st>>>(w, v, vprev, alpha, beta, n, part, counter, result);
  return cudaGetLastError();
}

cudaError_t launch_global_flip(cplx* u, const cplx* xp, const cplx* x, double c, uint64_t n, double* part,
                               unsigned* counter, double* result, cudaStream_t st) {
  global_flip_kernel<<<flat_grid(n, 0), kThreads, 0, st>>>(u, xp, x, c, n, part, counter, result);
  return cudaGetLastError();
}

cudaError_t launch_chunk_norms(const cplx* psi, uint64_t n, double* sums, uint64_t* nchunks, cudaStream_t st) {
  const uint64_t chunk = 1ull << kSampleChunkLog2;
  *nchunks = (n + chunk - 1) / chunk;
  chunk_norms_kernel<<<(unsigned)*nchunks, kThreads, 0, st>>>(psi, n, sums);
  return cudaGetLastError();
}

cudaError_t launch_sample(const cplx* psi, uint64_t n, const double* prefix, uint64_t nchunks, const double* u,
                          double total, int64_t shots, int64_t* out, cudaStream_t st) {
  const int warps = kThreads / 32;
  const uint64_t blocks = (uint64_t)(shots + warps - 1) / warps;
  sample_kernel<<<(unsigned)blocks, kThreads, 0, st>>>(psi, n, prefix, nchunks, u, total, shots, out);
  return cudaGetLastError();
}

cudaError_t launch_multidot(const MultiDotArgs& args, cudaStream_t st) {
  // a fixed grid: the reduction rows must fit the partial buffer (max_grid_rows)
  multidot_kernel<<<(unsigned)std::min<uint64_t>(flat_grid(args.n, 0), (uint64_t)num_sms() * 2), kThreads, 0, st>>>(args);
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

// Sharded runs, device-side scalars: after the all-reduce of (||w_j||^2, <w_j|A_last|w_j>) in red[0..1]
// finish beta_j, sigma_{j+1}, q_{j+1} (what lanczos_scalars does for one GPU) and post alpha_j, beta_j
// (and ||psi||^2 at j = 0) to the host mailbox -- no host round trip inside the iteration.
__global__ void shard_scalars_kernel(double* sc, int j, const double* red, double* mail) {
  const double nrm2 = red[0];
  const double beta = sqrt(fmax(0.0, nrm2));
  sc[SC_BE + j] = beta;
  sc[SC_SG + j + 1] = beta > 0.0 ? 1.0 / beta : 0.0;
  sc[SC_Q + j + 1] = nrm2 > 0.0 ? red[1] / nrm2 : 0.0;
  if (mail != nullptr) {
    if (j == 0) mail[0] = sc[SC_N0SQ];
    mail[1 + 2 * j] = sc[SC_AL + j];
    mail[2 + 2 * j] = beta;
    __threadfence_system();
  }
}

cudaError_t launch_shard_scalars(double* sc, int j, const double* red, double* mail, cudaStream_t st) {
  shard_scalars_kernel<<<1, 1, 0, st>>>(sc, j, red, mail);
  return cudaGetLastError();
}

int max_grid_rows() { return num_sms() * 8; }

}  // namespace rsv
