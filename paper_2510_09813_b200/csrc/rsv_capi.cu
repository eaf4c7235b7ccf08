// rsv_capi.cu -- C ABI (include/rsv.h) and the host-side Lanczos step driver.
//
// The driver restates rydsim/krylov.py:67-125 (expm_multiply) around the fused
// pass kernels: per Lanczos iteration it launches the bit-group passes (the last
// one writes w_j and reduces beta_j and q_{j+1}), copies (alpha_j, beta_j) to
// pinned host memory, and runs the reference's a-posteriori convergence test on
// the host with a tridiagonal implicit-QL eigen-solver (k <= 96).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rsv.h"
#include "rsv_kernels.cuh"

#ifndef RSV_L2_PROMOTION
#define RSV_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B   // strided tile loads pull whole 256 B sectors
#endif
#ifndef RSV_TENSOR_MAPS
#define RSV_TENSOR_MAPS 1   // 5-D TMA descriptors for the strided tiles (0: per-warp bulk runs)
#endif

using rsv::cplx;
typedef std::complex<double> zc;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(RSV_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                   \
  } while (0)

constexpr double kNsToUs = 1e-3;          // krylov.py:21
constexpr double kBreakdownRtol = 1e-14;  // krylov.py:25
constexpr int kScratchJ = 127;            // alpha-partial slot used by plain H.psi
constexpr int kRegenMax = rsv::kMaxKrylov; // Lanczos vectors of one run (device scalar arrays hold 128)
constexpr int kSpeculateMaxQubits = 24;    // auto speculation: Lanczos iterations of <= ~0.5 ms
constexpr int kFuseMaxQubits = 21;         // auto fused two-pass iteration (every 2-pass plan)
constexpr int kPartStride = 2 * rsv::kMaxKrylov > 2 + rsv::kMaxMasks ? 2 * rsv::kMaxKrylov
                                                                      : 2 + rsv::kMaxMasks;   // widest partial row

// ---------------------------------------------------------------- exp(-i tau T) e1 of the Lanczos tridiagonal
// krylov.py:54 (_tridiag_exp_e1: dense eigh of T) restated as a Chebyshev expansion of exp(-i z s) on
// the Gershgorin interval [c - rho, c + rho] of T:
//   exp(-i tau T) e1 = e^{-i tau c} sum_n eps_n (-i)^n J_n(tau rho) T_n(S) e1,  S = (T - c) / rho,
// eps_0 = 1, eps_n = 2. The Bessel values J_n come from Miller's downward recurrence (normalised with
// J_0 + 2 sum_m J_2m = 1), the vectors T_n(S) e1 from the three-term recurrence (T is tridiagonal: O(k)
// each, nonzero in their first n+1 entries), the sum stops where J_n(tau rho) < 1e-30. Cost
// O(k (tau rho + 40)) flops: at k = 38 about 7 us on the host against 50-80 us for implicit-QL sweeps
// (which at small N took longer than one Lanczos iteration on the GPU, stalling the speculative
// pipeline) and ~0.2 ms for the QL with every eigenvector row the combination needs. Accuracy: the
// absolute error of each component is at rounding level (~1e-16 of |y| = 1), the same noise floor as
// the reference's eigh; the convergence test (krylov.py:107-111) reads the last component only.
// Returns the last component; `all` (optional) receives every component.
zc tridiag_exp(const std::vector<double>& a, const std::vector<double>& b, double tau, std::vector<zc>* all) {
  const int k = (int)a.size();
  if (k == 1) {
    const zc y = std::exp(zc(0.0, -tau * a[0]));
    if (all) all->assign(1, y);
    return y;
  }
  double lo = INFINITY, hi = -INFINITY;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  const double c = 0.5 * (lo + hi);
  const double rho = std::max(0.5 * (hi - lo), 1e-300);
  const double z = std::fabs(tau) * rho;
  const int nmax = (int)std::ceil(z + 10.0 * std::cbrt(z + 1.0) + 30.0);   // J_n(z) < 1e-30 beyond
  std::vector<double> J(nmax + 1, 0.0);
  if (z == 0.0) {
    J[0] = 1.0;
  } else {
    double jp1 = 0.0, jn = 1e-300, norm = 0.0;
    for (int n = nmax + 30; n >= 1; --n) {
      const double jm1 = (2.0 * n / z) * jn - jp1;   // J_{n-1}
      jp1 = jn;
      jn = jm1;
      if (n - 1 <= nmax) J[n - 1] = jn;
      if (n - 1 > 0 && (n - 1) % 2 == 0) norm += 2.0 * jn;
      if (std::fabs(jn) > 1e250) {   // keep the unnormalised values in range
        for (int m = n - 1; m <= nmax; ++m) J[m] *= 1e-250;
        jn *= 1e-250;
        jp1 *= 1e-250;
        norm *= 1e-250;
      }
    }
    norm += J[0];
    for (double& v : J) v /= norm;
  }
  if (tau < 0.0)   // exp(+i |tau| T): J_n(-z) = (-1)^n J_n(z)
    for (int n = 1; n <= nmax; n += 2) J[n] = -J[n];
  // coefficient of T_n(S) e1: eps_n (-i)^n J_n, the phase e^{-i tau c} applied at the end
  const zc mi(0.0, -1.0);
  std::vector<zc> acc;
  if (all) acc.assign(k, zc(0.0, 0.0));
  zc last(0.0, 0.0);
  std::vector<double> w0(k, 0.0), w1(k, 0.0), w2(k, 0.0);
  const double inv = 1.0 / rho;
  w0[0] = 1.0;                       // T_0(S) e1
  w1[0] = (a[0] - c) * inv;          // T_1(S) e1
  w1[1] = b[0] * inv;
  if (all) {
    acc[0] += J[0];
    acc[0] += 2.0 * J[1] * mi * w1[0];
    acc[1] += 2.0 * J[1] * mi * w1[1];
  } else if (k == 2) {
    last = 2.0 * J[1] * mi * w1[1];
  }
  zc ph = mi;   // (-i)^n
  for (int n = 1; n < nmax; ++n) {
    const int len = std::min(k, n + 2);   // nonzeros of T_{n+1}(S) e1
    for (int i = 0; i < len; ++i) {
      double t = (a[i] - c) * w1[i];
      if (i > 0) t += b[i - 1] * w1[i - 1];
      if (i + 1 < k) t += b[i] * w1[i + 1];
      w2[i] = 2.0 * inv * t - w0[i];
    }
    std::swap(w0, w1);
    std::swap(w1, w2);
    ph *= mi;
    const zc cf = 2.0 * J[n + 1] * ph;
    if (all) {
      for (int i = 0; i < len; ++i) acc[i] += cf * w1[i];
    } else if (len == k) {
      last += cf * w1[k - 1];
    }
  }
  const zc phase = std::exp(zc(0.0, -tau * c));
  if (all) {
    for (zc& v : acc) v *= phase;
    *all = std::move(acc);
    return all->back();
  }
  return phase * last;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 5-D view of a 2^n complex128 vector whose box is one strided tile of shape sh:
// [2^(a+1) doubles | 2^(p-a) mid tiles | 2^g1 group rows | 2^g2 group rows | 2^(n-p-g) hi tiles]
bool encode_tile_map(CUtensorMap* m, const void* base, const rsv::Shape& sh) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr || sh.a > 7 || base == nullptr) return false;
  const int g1 = std::min(sh.g, 8), g2 = sh.g - g1, hb = sh.n - sh.p - sh.g;
  cuuint64_t dim[5] = {2ull << sh.a, 1ull << (sh.p - sh.a), 1ull << g1, 1ull << g2, 1ull << hb};
  cuuint64_t stride[4] = {16ull << sh.a, 16ull << sh.p, 16ull << (sh.p + g1), 16ull << (sh.p + sh.g)};
  cuuint32_t box[5] = {2u << sh.a, 1u, 1u << g1, 1u << g2, 1u};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(base), dim, stride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)RSV_L2_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// The same tile geometry with the group split as [g-3 rows | 3 eighth bits]: the box is one eighth
// of a tile (coordinate 3 selects it), the unit of the peer-memory TMA ring (PassArgs::tm_peer).
bool encode_eighth_map(CUtensorMap* m, const void* base, const rsv::Shape& sh) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr || sh.a > 7 || sh.g < 3 || sh.g - 3 > 8 || base == nullptr) return false;
  const int g1 = sh.g - 3, hb = sh.n - sh.p - sh.g;
  cuuint64_t dim[5] = {2ull << sh.a, 1ull << (sh.p - sh.a), 1ull << g1, 8ull, 1ull << hb};
  cuuint64_t stride[4] = {16ull << sh.a, 16ull << sh.p, 16ull << (sh.p + g1), 16ull << (sh.p + sh.g)};
  cuuint32_t box[5] = {2u << sh.a, 1u, 1u << g1, 1u, 1u};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(base), dim, stride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)RSV_L2_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace
struct rsv_context;
namespace {
bool cached_tile_map(rsv_context* c, CUtensorMap* m, const void* base, const rsv::Shape& sh, bool eighth = false);

// Choose the tile-load mode of a pass and set its TMA descriptors (encoded once per vector and
// shape, rsv_context::maps).
void set_tile_load(rsv_context* c, rsv::PassArgs& A) {
  const rsv::Shape& sh = A.sh;
  A.tstore = 0;
  if (sh.g == 0) {
    A.load = rsv::LOAD_CONTIG;
    A.tstore = A.out != nullptr ? 1 : 0;   // one bulk copy per output tile
    return;
  }
  A.load = rsv::LOAD_RUNS;
  if (RSV_TENSOR_MAPS && sh.a <= 7 && cached_tile_map(c, &A.tm_x, A.x, sh) &&
      (A.ein == nullptr || cached_tile_map(c, &A.tm_e, A.ein, sh))) {
    A.load = rsv::LOAD_TENSOR;
    // output tiles by TMA tensor stores through the same tile geometry
    if (A.out != nullptr && cached_tile_map(c, &A.tm_o, A.out, sh)) A.tstore = 1;
  }
}

// Peer-memory passes: partner tiles by TMA into the kernel's shared-memory ring when the pass has
// full 4096-amplitude tiles, >= 8 amplitudes a thread and a TMA tile load (RSV_PEER_TMA=0 in the
// environment keeps the per-thread P2P loads, for comparison).
void set_peer_load(rsv_context* c, rsv::PassArgs& A) {
  A.peer_tma = 0;
  if (A.npeer == 0 || A.sh.a + A.sh.g != rsv::kLoBits) return;
  static const bool off = [] {
    const char* e = std::getenv("RSV_PEER_TMA");
    return e != nullptr && e[0] == '0';
  }();
  if (off) return;
  if ((A.kind != rsv::PASS_FIRST && A.kind != rsv::PASS_MID) || A.npeer > 2) return;
  if ((1 << rsv::kLoBits) / rsv::peer_pass_threads(A.kind, A.sh.a) < 8) return;
  if (A.load == rsv::LOAD_CONTIG) {
    A.peer_tma = 1;
    return;
  }
  if (A.load != rsv::LOAD_TENSOR) return;
  for (int g = 0; g < A.npeer; ++g)
    if (!cached_tile_map(c, &A.tm_peer[g], A.peer[g], A.sh, true)) return;
  A.peer_tma = 1;
}

struct PassPlan {
  rsv::Shape sh;
  std::vector<int> qubits;   // qubits whose flips this pass applies (all inside its tile)
  bool lo;    // lo tile (bits [0, a)) carries the diagonal
  // chunk pass (rsv::ChunkArgs): sh/qubits are its L tiles, shm/qubits_m its M tiles
  bool chunk = false;
  int gm = 0;
  rsv::Shape shm{};
  std::vector<int> qubits_m;
};

}  // namespace

struct rsv_context {
  int n = 0;
  int diag_mode = RSV_DIAG_FLY;
  cudaStream_t st = nullptr;
  int device = 0;
  double* d_u = nullptr;
  double* d_sc = nullptr;
  double* d_part = nullptr;
  unsigned* d_counter = nullptr;
  double* d_dl = nullptr;
  double* d_gc = nullptr;         // lo-pass tile table (per run)
  double* d_dvec = nullptr;
  double* h_pin = nullptr;
  double* d_red = nullptr;          // sharded runs: caller's device buffer for on-stream all-reduces
  int red_count = 0;                //   (rsv_set_shard_scratch; RSV_COMM_ALLREDUCE_DEVICE)
  double* h_mail = nullptr;         // mapped pinned mailbox: [n0sq, alpha_0, beta_0, alpha_1, ...]
  double* d_mail = nullptr;         //   its device address (written by the last pass)
  struct MapEntry {
    const void* base;
    int n, a, p, g;
    CUtensorMap map;
  };
  std::vector<MapEntry> maps;       // TMA descriptors by (vector, tile shape): encoded once
  std::vector<void*> phys;        // bound slots
  std::vector<int> logical;       // logical slot -> physical; logical 0..K = Krylov s_j, K+1 = work
  std::vector<PassPlan> plan;
  // sharding by the top qubits (row e; sharding.py): this context holds one shard's local qubits
  bool sharded = false;
  rsv_comm_fn comm = nullptr;
  void* comm_user = nullptr;
  cplx* xbuf = nullptr;             // exchange buffer (the partner shard's copy of s_j)
  double offset = 0.0, next_offset = 0.0;   // constant energy of this shard's global bits
  std::vector<double> gcoef;        // Omega_g / 2 of each global qubit this step (0: no flip)
  std::vector<int> gpeer;           // partner rank of each global qubit
  double n0sq_global = 0.0;         // ||psi||^2 over all shards from the last combination
  double local_n0sq = 0.0;          // this shard's share of it
  // peer-memory mode: the partner shards' slots mapped into this process (CUDA IPC / UVA);
  // peer_slots[g][physical slot] for global qubit g (empty: exchange through the callback)
  std::vector<std::vector<const cplx*>> peer_slots;
  long long peer_passes[2] = {0, 0};   // peer-memory passes launched: TMA ring, per-thread loads
  bool reorth = false;              // full re-orthogonalisation (krylov.py:103-104), opt-in
  bool tail_regen = true;           // beyond the resident basis: ring + regeneration (else split in time)
  int speculate = -1;               // launch iteration j+1 before testing j: -1 auto (N <= 24), 0 off, 1 on
  int fuse = -1;                    // two-pass plans in one cooperative launch: -1 auto (N <= 21), 0 off, 1 on
  cudaEvent_t iter_ev[2] = {nullptr, nullptr};
  double* d_dots = nullptr;         // <s_i|w> scratch (2 kMaxKrylov doubles)
  int plan_gm = -1;               // chunk group bits: -1 auto, 0 off, 3..9 forced (rsv_set_plan)
  long long plan_lag = -1;        // chunk scheduler lag in M tiles (-1 auto)
  unsigned long long* d_ticket = nullptr;
  unsigned* d_done = nullptr;     // per-chunk M-tile counters (2^(n-15) entries: any gm >= 3)
  std::vector<double> h_u;
  // caches
  bool prep_valid = false;
  std::vector<double> prep_key;
  bool dl_valid = false;
  std::vector<double> dl_key;
  std::vector<uint64_t> masks;
  cudaEvent_t obs_event = nullptr;
  bool obs_pending = false;
  int obs_count = 0;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_pending;   // (event index start, family)
  int ev_next = 0;
  double prof_ms[4] = {0, 0, 0, 0};   // event-timed launches: summed time and count
  long long prof_n[4] = {0, 0, 0, 0};
  long long prof_all[4] = {0, 0, 0, 0};   // every launch of the family
  int prof_every = 1;                     // time one launch in prof_every (per family)
  bool prof_skip = false;                 // the current launch is not timed
};

namespace {

bool cached_tile_map(rsv_context* c, CUtensorMap* m, const void* base, const rsv::Shape& sh, bool eighth) {
  const int gk = eighth ? -1 - sh.g : sh.g;   // eighth-tile maps keyed apart
  for (const auto& e : c->maps)
    if (e.base == base && e.n == sh.n && e.a == sh.a && e.p == sh.p && e.g == gk) {
      *m = e.map;
      return true;
    }
  if (!(eighth ? encode_eighth_map(m, base, sh) : encode_tile_map(m, base, sh))) return false;
  if (c->maps.size() >= 512) c->maps.clear();   // user vectors of rsv_apply_hamiltonian come and go
  c->maps.push_back({base, sh.n, sh.a, sh.p, gk, *m});
  return true;
}

// Slots 0..K: s_0 (the state) .. s_{K-1} are the Krylov basis; the partial sums u of iteration j
// live in slot j+1 (each pass reads and rewrites its own tiles in place, the last pass turns u
// into s_{j+1} there), so no separate work vector is needed and K = nslots - 1.
int kcap(const rsv_context* c) { return (int)c->logical.size() - 1; }
cplx* slot(const rsv_context* c, int logical_index) {
  return reinterpret_cast<cplx*>(c->phys[c->logical[logical_index]]);
}
// Logical slot of Krylov vector s_i. Up to the cap K the basis is resident (s_i in slot i); beyond
// it the recurrence continues in a ring of the last two slots (s_i for i > K overwrites s_{i-2}:
// iteration j writes s_{j+1} where it read s_{j-1}, elementwise), and the overwritten basis
// vectors are regenerated for the Krylov combination (lanczos_run, "tail regeneration").
int kidx(const rsv_context* c, int i) {
  const int K = kcap(c);
  return i <= K ? i : (K - 1) + ((i - (K - 1)) & 1);
}
cplx* kvec(const rsv_context* c, int i) { return slot(c, kidx(c, i)); }

// Pass plan: the lo pass (tile = bits [0, 12), carries the diagonal) and hi passes over groups
// of <= 9 high bits (tile = 2^a contiguous x 2^g strided rows). Smaller groups sit at the top
// of the index so the most strided passes get the longest contiguous runs; the lowest group
// runs last (it also carries the q-sweep). When a middle pass exists, the lowest qubits'
// flips move from the lo pass (the heaviest: 12 flips + diagonal) to the first middle pass,
// whose tile contains those bits too.
#ifndef RSV_TOP_BIG
#define RSV_TOP_BIG 0
#endif
#ifndef RSV_DELEGATE_LOW
#define RSV_DELEGATE_LOW 3
#endif
#ifndef RSV_LO_LAST
#define RSV_LO_LAST 0
#endif
#ifndef RSV_LAST_TOP
#define RSV_LAST_TOP 1
#endif
constexpr int kDelegateLow = RSV_DELEGATE_LOW;

#ifndef RSV_CHUNK_GM
#define RSV_CHUNK_GM 8
#endif
#ifndef RSV_CHUNK_AUTO
#define RSV_CHUNK_AUTO 0
#endif

// Chunk group bits for N qubits under the context's setting (0 = plain passes).
int chunk_gm_for(int n, int setting) {
  if (setting == 0) return 0;
  // M tiles keep a = 12 - gm <= log2(pass threads) so a thread's amplitudes sit at one stride
  const int gmin = std::max(3, rsv::kLoBits - rsv::ilog2(RSV_CHUNK_THREADS));
  if (setting > 0) return (setting >= gmin && setting <= 9 && n - rsv::kLoBits - setting >= 1) ? setting : 0;
  // auto: off. Measured at N=29 ("L2-resident chunk pass"): the chunk pass cuts a
  // Lanczos iteration's HBM bytes from 144 to 96 per amplitude, but its two tile passes stay
  // shared-memory-pipe bound, so the plain passes (HBM-bound at ~0.95 of the copy peak) are faster.
#if RSV_CHUNK_AUTO
  if (n - rsv::kLoBits > rsv::kLoBits - 3) return std::min(RSV_CHUNK_GM, n - rsv::kLoBits - 1);
#endif
  return 0;
}

// Groups of <= 9 bits covering [from, n), smallest at the top of the index, in execution order
// (lowest group last unless RSV_LAST_TOP).
std::vector<PassPlan> hi_groups(int n, int from) {
  std::vector<PassPlan> out;
  const int rem = n - from;
  if (rem <= 0) return out;
  const int gmax = rsv::kLoBits - 3;
  const int ng = (rem + gmax - 1) / gmax;
  std::vector<int> sizes;   // ascending: the top (most strided) groups are the smallest
  for (int i = 0; i < ng; ++i) sizes.push_back(rem / ng + (i >= ng - rem % ng ? 1 : 0));
#if RSV_TOP_BIG
  std::reverse(sizes.begin(), sizes.end());   // experiment: the top group takes the extra bit
#endif
  std::vector<PassPlan> hi;
  int top = n;
  const int lt = rsv::ilog2(rsv::pass_threads(rsv::kLoBits));
  for (int s : sizes) {
    PassPlan p;
    // contiguous run 2^a with a <= log2(pass threads): the register bits of a thread are then
    // all group bits, so its amplitudes sit at one uniform stride (pass_kernel, S)
    const int a = std::min(rsv::kLoBits - s, lt);
    p.sh = rsv::Shape{n, a, top - s, s, 1ull << (n - a - s)};
    for (int q = top - s; q < top; ++q) p.qubits.push_back(q);
    p.lo = false;
    hi.push_back(p);
    top -= s;
  }
#if RSV_LAST_TOP
  for (size_t i = hi.size() - 1; i >= 1; --i) out.push_back(hi[i]);
  out.push_back(hi[0]);
#else
  for (size_t i = 0; i + 1 < hi.size(); ++i) out.push_back(hi[i]);
  out.push_back(hi.back());
#endif
  return out;
}

#ifndef RSV_CHUNK_DELEGATE
#define RSV_CHUNK_DELEGATE 3
#endif
#ifndef RSV_CHUNK_DELEGATE_M
#define RSV_CHUNK_DELEGATE_M 0
#endif

void build_plan(rsv_context* c) {
  const int n = c->n;
  c->plan.clear();
  const int alo = std::min(n, rsv::kLoBits);
  PassPlan lo;
  lo.sh = rsv::Shape{n, alo, alo, 0, 1ull << (n - alo)};
  for (int q = 0; q < alo; ++q) lo.qubits.push_back(q);
  lo.lo = true;
  const int gm = chunk_gm_for(n, c->plan_gm);
  if (gm > 0) {
    // chunk pass: L tiles = the lo tile, M tiles = 2^(12-gm) contiguous x bits [12, 12+gm)
    lo.chunk = true;
    lo.gm = gm;
    lo.shm = rsv::Shape{n, rsv::kLoBits - gm, rsv::kLoBits, gm, 1ull << (n - rsv::kLoBits)};
    for (int q = rsv::kLoBits; q < rsv::kLoBits + gm; ++q) lo.qubits_m.push_back(q);
    c->plan.push_back(lo);
    for (auto& p : hi_groups(n, rsv::kLoBits + gm)) c->plan.push_back(p);
    // the lowest bits' flips move to the first hi pass (its tile holds them too): the chunk
    // pass carries two tiles' worth of shared-memory work per amplitude
    const int d = RSV_CHUNK_DELEGATE;
    if (d > 0 && c->plan[1].sh.a >= d) {
      PassPlan& l = c->plan[0];
      PassPlan& m = c->plan[1];
      l.qubits.erase(l.qubits.begin(), l.qubits.begin() + d);
      for (int q = 0; q < d; ++q) m.qubits.push_back(q);
    } else if (RSV_CHUNK_DELEGATE_M > 0 && lo.shm.a >= RSV_CHUNK_DELEGATE_M) {
      // or to the chunk's own M tiles (they hold bits [0, 12 - gm) too)
      PassPlan& l = c->plan[0];
      l.qubits.erase(l.qubits.begin(), l.qubits.begin() + RSV_CHUNK_DELEGATE_M);
      for (int q = 0; q < RSV_CHUNK_DELEGATE_M; ++q) l.qubits_m.push_back(q);
    }
    return;
  }
  c->plan.push_back(lo);
  for (auto& p : hi_groups(n, alo)) c->plan.push_back(p);
  if (kDelegateLow > 0 && c->plan.size() >= 3 && c->plan[1].sh.a >= kDelegateLow && alo > kDelegateLow) {
    PassPlan& l = c->plan[0];
    PassPlan& m = c->plan[1];
    l.qubits.erase(l.qubits.begin(), l.qubits.begin() + kDelegateLow);
    for (int q = 0; q < kDelegateLow; ++q) m.qubits.push_back(q);
  }
#if RSV_LO_LAST
  // lo pass last: the q-sweep and the Krylov combination then run on contiguous tiles, the
  // strided passes (top group first) carry no q-sweep
  if (c->plan.size() >= 2) {
    std::vector<PassPlan> hi(c->plan.begin() + 1, c->plan.end());
    std::vector<PassPlan> order;
    for (size_t i = hi.size(); i-- > 0;) order.push_back(hi[i]);
    order.push_back(c->plan[0]);
    c->plan = order;
  }
#endif
}

rsv::FlipSet flips_for(const PassPlan& p, const double* omegas, int nthreads) {
  // Tile bits below log2(threads per CTA) are flipped through shared memory, the
  // ones above are register permutations inside a thread (pass_kernel, RegBits).
  rsv::FlipSet f{};
  f.count = 0;
  const int lt = rsv::ilog2(nthreads);
  for (int q : p.qubits) {
    const double cq = 0.5 * omegas[q];
    if (cq == 0.0) continue;   // zero drives are skipped, as in _kernels.py:19
    const int local = (p.lo || q < p.sh.a) ? q : p.sh.a + (q - p.sh.p);
    if (local >= lt) {
      f.rcoef[local - lt] = cq;
    } else {
      f.mask[f.count] = 1 << local;
      f.coef[f.count] = cq;
      ++f.count;
    }
  }
  return f;
}

rsv::DiagArgs diag_for(const rsv_context* c, const PassPlan& p, const double* deltas) {
  rsv::DiagArgs d{};
  d.mode = rsv::DIAG_NONE;
  if (!p.lo) return d;
  d.mode = c->diag_mode == RSV_DIAG_VEC ? rsv::DIAG_VEC : rsv::DIAG_FLY;
  d.dl = c->d_dl;
  d.gc = c->d_gc;
  d.umat = c->d_u;
  d.dvec = c->d_dvec;
  for (int i = 0; i < c->n; ++i) d.delta[i] = deltas[i];
  return d;
}

int ensure_dl(rsv_context* c, const double* deltas, double offset = 0.0) {
  const int alo = std::min(c->n, rsv::kLoBits);   // the lo tile (wherever it sits in the plan)
  std::vector<double> key(deltas, deltas + c->n);
  key.push_back(offset);
  if (c->dl_valid && key == c->dl_key) return RSV_OK;
  const bool fly = c->diag_mode == RSV_DIAG_FLY;
  CUDA_TRY(rsv::launch_build_dl(alo, c->n, c->d_u, deltas, fly ? 1 : 0, offset, c->d_dl, c->st));
  CUDA_TRY(rsv::launch_tile_base(alo, c->n, fly ? 1 : 0, deltas, c->d_gc, c->st));
  c->dl_key = key;
  c->dl_valid = true;
  return RSV_OK;
}

// Key of everything the prepared q_0 depends on: last-pass drives (+ detunings if it holds the diagonal).
std::vector<double> prep_key_for(const rsv_context* c, const double* omegas, const double* deltas, double off) {
  const PassPlan& last = c->plan.back();
  std::vector<double> k;
  for (int q : last.qubits) k.push_back(omegas[q]);
  if (last.lo) {
    k.insert(k.end(), deltas, deltas + c->n);
    k.push_back(off);
  }
  return k;
}

void prof_begin(rsv_context* c, int family) {
  if (!c->prof) return;
  // sampled timing: the event pair costs host time per launch, which on small registers (Lanczos
  // iterations of ~35 us, host-paced) would slow the timed loop by ~16 % if every launch carried one
  c->prof_skip = (c->prof_all[family]++ % c->prof_every) != 0;
  if (c->prof_skip) return;
  if (c->ev_next + 2 > (int)c->ev_pool.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->ev_pool.push_back(e);
    }
  }
  cudaEventRecord(c->ev_pool[c->ev_next], c->st);
  c->ev_pending.push_back({c->ev_next, family});
  c->ev_next += 2;
}
void prof_end(rsv_context* c) {
  if (!c->prof || c->prof_skip) return;
  cudaEventRecord(c->ev_pool[c->ev_pending.back().first + 1], c->st);
}
void prof_collect(rsv_context* c) {   // collects the kernels that have finished (speculation may leave some)
  if (!c->prof) return;
  std::vector<std::pair<int, int>> left;
  for (auto& pe : c->ev_pending) {
    if (cudaEventQuery(c->ev_pool[pe.first + 1]) != cudaSuccess) {
      left.push_back(pe);
      continue;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_pool[pe.first], c->ev_pool[pe.first + 1]);
    c->prof_ms[pe.second] += ms;
    c->prof_n[pe.second] += 1;
  }
  c->ev_pending.swap(left);
  if (c->ev_pending.empty()) c->ev_next = 0;
}

int family_of(size_t pass_index, size_t npass) {
  if (pass_index + 1 == npass) return 2;
  return pass_index == 0 ? 0 : 1;
}

// ---- sharded runs: the host side of the all-reduces and the global-qubit exchanges
int comm_call(rsv_context* c, int op, int slot_index, int peer, double* host, int count) {
  const int rc = c->comm(c->comm_user, op, slot_index, peer, host, count);
  if (rc != 0) return fail(RSV_ERR_CUDA, "shard communication callback failed (op %d, rc %d)", op, rc);
  return RSV_OK;
}

// After a raw combination: all-reduce ||psi||^2, <psi|A_last|psi> and the mask sums, finish the scalars.
int shard_finish_combine(rsv_context* c, int nmask) {
  double* h = c->h_pin;
  CUDA_TRY(cudaMemcpyAsync(h + rsv::SC_N0SQ, c->d_sc + rsv::SC_N0SQ, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaMemcpyAsync(h + rsv::SC_Q, c->d_sc + rsv::SC_Q, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  if (nmask > 0)
    CUDA_TRY(cudaMemcpyAsync(h + rsv::SC_OBS, c->d_sc + rsv::SC_OBS, sizeof(double) * nmask, cudaMemcpyDeviceToHost,
                             c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  std::vector<double> buf(2 + nmask);
  buf[0] = h[rsv::SC_N0SQ];
  buf[1] = h[rsv::SC_Q];
  for (int m = 0; m < nmask; ++m) buf[2 + m] = h[rsv::SC_OBS + m];
  c->local_n0sq = buf[0];
  int rc = comm_call(c, RSV_COMM_ALLREDUCE, -1, -1, buf.data(), (int)buf.size());
  if (rc) return rc;
  const double nsq = buf[0];
  c->n0sq_global = nsq;
  double fin[3] = {nsq, nsq > 0.0 ? 1.0 / std::sqrt(nsq) : 0.0, nsq > 0.0 ? buf[1] / nsq : 0.0};
  h[rsv::SC_N0SQ] = nsq;
  for (int m = 0; m < nmask; ++m) h[rsv::SC_OBS + m] = buf[2 + m];
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_N0SQ, &fin[0], sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_SG, &fin[1], sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_Q, &fin[2], sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if (nmask > 0) {
    CUDA_TRY(cudaEventRecord(c->obs_event, c->st));
    c->obs_pending = true;
    c->obs_count = nmask;
  }
  return RSV_OK;
}

// Before the last pass of iteration j: the global-qubit flips (partner shard's s_j, exchanged by the
// host) are added to the partial sums u (slot j+1), and alpha's partial share is all-reduced.
// The first exchange was started before the local passes (overlapped with them).
int shard_before_last(rsv_context* c, int j, double sigma, bool started, bool p2p) {
  double add = 0.0;
  const uint64_t nloc = 1ull << c->n;
  bool first = true;
  for (size_t g = 0; g < c->gcoef.size() && !p2p; ++g) {
    if (c->gcoef[g] == 0.0) continue;
    if (c->xbuf == nullptr) return fail(RSV_ERR_STATE, "exchange mode without an exchange buffer (rsv_set_shard)");
    int rc;
    if (!(first && started)) {
      CUDA_TRY(cudaStreamSynchronize(c->st));
      rc = comm_call(c, RSV_COMM_EXCHANGE_START, c->logical[kidx(c, j)], c->gpeer[g], nullptr, 0);
      if (rc) return rc;
    }
    first = false;
    rc = comm_call(c, RSV_COMM_EXCHANGE_WAIT, c->logical[kidx(c, j)], c->gpeer[g], nullptr, 0);
    if (rc) return rc;
    const double cs = c->gcoef[g] * sigma;
    CUDA_TRY(rsv::launch_global_flip(kvec(c, j + 1), c->xbuf, kvec(c, j), cs, nloc, c->d_part, c->d_counter,
                                     c->d_sc + rsv::SC_GF, c->st));
    double dot = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&c->h_pin[rsv::SC_GF], c->d_sc + rsv::SC_GF, sizeof(double), cudaMemcpyDeviceToHost,
                             c->st));
    CUDA_TRY(cudaStreamSynchronize(c->st));   // the exchange buffer is free again
    dot = c->h_pin[rsv::SC_GF];
    add += cs * sigma * dot;
  }
  if (p2p && c->d_red != nullptr) {   // on-stream all-reduce of alpha's partial share (no host sync)
    CUDA_TRY(cudaMemcpyAsync(c->d_red, c->d_sc + rsv::SC_AP + j, sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    int rc = comm_call(c, RSV_COMM_ALLREDUCE_DEVICE, -1, -1, c->d_red, 1);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_AP + j, c->d_red, sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    return RSV_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(&c->h_pin[rsv::SC_AP + j], c->d_sc + rsv::SC_AP + j, sizeof(double),
                           cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  double ap = c->h_pin[rsv::SC_AP + j] + add;
  int rc = comm_call(c, RSV_COMM_ALLREDUCE, -1, -1, &ap, 1);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_AP + j, &ap, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return RSV_OK;
}

// After the (raw) last pass of iteration j: all-reduce ||w_j||^2 and <w_j|A_last|w_j>, write back
// beta_j, sigma_{j+1}, q_{j+1}.
int shard_finish_iteration(rsv_context* c, int j) {
  if (c->d_red != nullptr && c->red_count >= 2) {   // on-stream: all-reduce + finishing kernel + mailbox
    CUDA_TRY(cudaMemcpyAsync(c->d_red, c->d_sc + rsv::SC_BE + j, sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CUDA_TRY(cudaMemcpyAsync(c->d_red + 1, c->d_sc + rsv::SC_Q + j + 1, sizeof(double), cudaMemcpyDeviceToDevice,
                             c->st));
    int rc = comm_call(c, RSV_COMM_ALLREDUCE_DEVICE, -1, -1, c->d_red, 2);
    if (rc) return rc;
    CUDA_TRY(rsv::launch_shard_scalars(c->d_sc, j, c->d_red, c->d_mail, c->st));
    return RSV_OK;
  }
  double* h = c->h_pin;
  CUDA_TRY(cudaMemcpyAsync(h + rsv::SC_BE + j, c->d_sc + rsv::SC_BE + j, sizeof(double), cudaMemcpyDeviceToHost,
                           c->st));
  CUDA_TRY(cudaMemcpyAsync(h + rsv::SC_Q + j + 1, c->d_sc + rsv::SC_Q + j + 1, sizeof(double),
                           cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  double buf[2] = {h[rsv::SC_BE + j], h[rsv::SC_Q + j + 1]};
  int rc = comm_call(c, RSV_COMM_ALLREDUCE, -1, -1, buf, 2);
  if (rc) return rc;
  const double nrm2 = buf[0], beta = std::sqrt(std::max(0.0, nrm2));
  const double sg = beta > 0.0 ? 1.0 / beta : 0.0, q = nrm2 > 0.0 ? buf[1] / nrm2 : 0.0;
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_BE + j, &beta, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_SG + j + 1, &sg, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_Q + j + 1, &q, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return RSV_OK;
}

// Single-bit observable masks (occupations) are reduced per bit class in the combination kernel:
// a bit of the combine tile is a thread-index bit (tile position < log2 threads) or a register bit,
// any other bit is constant over a tile.
void classify_masks(rsv::CombineArgs& A) {
  A.obs_single = A.nmask > 0 ? 1 : 0;
  const int lt = rsv::ilog2(rsv::combine_threads(A.sh.a + A.sh.g));
  for (int m = 0; m < A.nmask; ++m) {
    const uint64_t M = A.mask[m];
    if (M == 0 || (M & (M - 1))) {
      A.obs_single = 0;
      return;
    }
    int q = 0;
    while (!((M >> q) & 1ull)) ++q;
    int pos = -1;   // tile position
    if (q < A.sh.a) pos = q;
    else if (q >= A.sh.p && q < A.sh.p + A.sh.g) pos = A.sh.a + (q - A.sh.p);
    if (pos < 0) {
      A.obs_cat[m] = 0;
      A.obs_pos[m] = (unsigned char)q;
    } else if (pos < lt) {
      A.obs_cat[m] = 1;
      A.obs_pos[m] = (unsigned char)pos;
    } else {
      A.obs_cat[m] = 2;
      A.obs_pos[m] = (unsigned char)(pos - lt);
    }
  }
}

// Krylov combination (also "prepare": k = 1, coefficient 1, in place). vecs (optional): the vectors
// to combine (default: s_0..s_{k-1} in their resident slots).
int run_combine(rsv_context* c, int k, const std::vector<zc>& coef, cplx* out, const double* q_omegas,
                const double* q_deltas, int observe, double q_offset = 0.0,
                const std::vector<const cplx*>* vecs = nullptr) {
  rsv::CombineArgs A{};
  const PassPlan& last = c->plan.back();
  A.sh = last.sh;
  A.qsweep = q_omegas != nullptr ? 1 : 0;
  if (A.qsweep) {
    A.fl = flips_for(last, q_omegas, rsv::combine_threads(last.sh.a + last.sh.g));
    A.dg = diag_for(c, last, q_deltas);
    if (last.lo) {
      int rc = ensure_dl(c, q_deltas, q_offset);
      if (rc) return rc;
    }
  } else {
    A.fl.count = 0;
    A.dg.mode = rsv::DIAG_NONE;
  }
  if (k > rsv::kMaxKrylov) return fail(RSV_ERR_ARG, "Krylov combination of %d vectors exceeds %d", k, rsv::kMaxKrylov);
  A.k = k;
  for (int i = 0; i < k; ++i) {
    A.v[i] = vecs ? (*vecs)[i] : slot(c, i);
    A.coef[i] = make_double2(coef[i].real(), coef[i].imag());
  }
  A.out = out;
  A.nmask = observe ? (int)c->masks.size() : 0;
  for (int m = 0; m < A.nmask; ++m) A.mask[m] = c->masks[m];
  classify_masks(A);
  A.sc = c->d_sc;
  A.part = c->d_part;
  A.counter = c->d_counter;
  A.raw = c->sharded ? 1 : 0;
  prof_begin(c, 3);
  CUDA_TRY(rsv::launch_combine(A, c->st));
  prof_end(c);
  if (c->sharded) return shard_finish_combine(c, A.nmask);
  if (A.nmask > 0) {
    CUDA_TRY(cudaMemcpyAsync(c->h_pin + rsv::SC_OBS, c->d_sc + rsv::SC_OBS, sizeof(double) * A.nmask,
                             cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaMemcpyAsync(c->h_pin + rsv::SC_N0SQ, c->d_sc + rsv::SC_N0SQ, sizeof(double),
                             cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaEventRecord(c->obs_event, c->st));
    c->obs_pending = true;
    c->obs_count = A.nmask;
  }
  return RSV_OK;
}

int prepare(rsv_context* c, const double* omegas, const double* deltas) {
  std::vector<zc> one(1, zc(1.0, 0.0));
  int rc = run_combine(c, 1, one, slot(c, 0), omegas, deltas, 0, c->offset);
  if (rc) return rc;
  c->prep_key = prep_key_for(c, omegas, deltas, c->offset);
  c->prep_valid = true;
  return RSV_OK;
}

// The chunk pass (first kernel of an iteration): out = (A_M + A_L + D) v - beta' prev.
int launch_chunk_pass(rsv_context* c, const PassPlan& p, const double* omegas, const double* deltas,
                      const cplx* x, int x_scale_slot, const cplx* prev, cplx* out, int j) {
  rsv::ChunkArgs A{};
  A.shm = p.shm;
  A.shl = p.sh;
  PassPlan pm;
  pm.sh = p.shm;
  pm.qubits = p.qubits_m;
  pm.lo = false;
  const int nt = RSV_CHUNK_THREADS;
  A.flm = flips_for(pm, omegas, nt);
  A.fll = flips_for(p, omegas, nt);
  A.dg = diag_for(c, p, deltas);
  A.x = x;
  A.x_scale_slot = x_scale_slot;
  A.prev = prev;
  A.out = out;
  A.j = j;
  A.gm = p.gm;
  const unsigned long long tiles = 1ull << p.gm;
  unsigned long long lag = c->plan_lag > 0 ? (unsigned long long)c->plan_lag : tiles + tiles / 2;
  if (lag < tiles) lag = tiles;   // an L tile may never precede the M tiles of its chunk
  A.lag = std::min<unsigned long long>(lag, p.sh.n_tiles);
  A.sc = c->d_sc;
  A.part = c->d_part;
  A.counter = c->d_counter;
  A.ticket = c->d_ticket;
  A.done = c->d_done;
  A.load_m = rsv::LOAD_RUNS;
  if (RSV_TENSOR_MAPS && p.shm.a <= 7 && encode_tile_map(&A.tm_x, x, p.shm) &&
      (prev == nullptr || encode_tile_map(&A.tm_e, prev, p.shm)))
    A.load_m = rsv::LOAD_TENSOR;
  prof_begin(c, 0);
  CUDA_TRY(rsv::launch_chunk(A, c->st));
  prof_end(c);
  return RSV_OK;
}

// The plan is [lo, last] with 4096-amplitude tiles and the context may run it as one cooperative
// launch (iter2_kernel): single-GPU runs of 16..21 qubits.
bool fused_iteration(const rsv_context* c) {
  if (c->fuse == 0 || c->sharded || c->plan.size() != 2) return false;
  const PassPlan& lo = c->plan[0];
  const PassPlan& last = c->plan[1];
  if (!lo.lo || lo.chunk || lo.sh.a + lo.sh.g != rsv::kLoBits || last.sh.a + last.sh.g != rsv::kLoBits) return false;
  if (last.sh.a > rsv::ilog2(RSV_ITER2_THREADS)) return false;   // a thread's amplitudes at one stride
  return c->fuse > 0 || c->n <= kFuseMaxQubits;
}

int launch_lanczos_iteration(rsv_context* c, int j, const double* omegas, const double* deltas, double sigma,
                             double prev_coef) {
  const size_t np = c->plan.size();
  if (fused_iteration(c)) {
    rsv::Iter2Args F{};
    for (int pi = 0; pi < 2; ++pi) {
      rsv::PassArgs& A = pi == 0 ? F.lo : F.last;
      const PassPlan& p = c->plan[pi];
      A.kind = pi == 0 ? rsv::PASS_FIRST : rsv::PASS_LAST_LANCZOS;
      A.sh = p.sh;
      A.fl = flips_for(p, omegas, RSV_ITER2_THREADS);
      A.dg = diag_for(c, p, deltas);
      A.x = kvec(c, j);
      A.x_scale_slot = rsv::SC_SG + j;
      A.j = j;
      A.sc = c->d_sc;
      A.part = c->d_part;
      A.counter = c->d_counter;
      A.ein = pi == 0 ? (j > 0 ? kvec(c, j - 1) : nullptr) : kvec(c, j + 1);
      A.ein_is_prev = pi == 0 ? 1 : 0;
      A.out = kvec(c, j + 1);
      A.qsweep = pi == 1 ? 1 : 0;
      A.mail = pi == 1 ? c->d_mail : nullptr;
      set_tile_load(c, A);
    }
    F.gridbar = c->d_counter + 2;
    prof_begin(c, 0);
    CUDA_TRY(rsv::launch_iter2(F, c->st));
    prof_end(c);
    return RSV_OK;
  }
  // sharded: start the first global-qubit exchange of s_j so it overlaps the local passes
  // (peer-memory mode: no exchange, the first pass reads the partner shards directly)
  bool started = false;
  // (the opt-in chunk pass has no peer operands: with it the exchange mode is required)
  const bool p2p = c->sharded && !c->peer_slots.empty() && np > 1 && !c->plan[0].chunk;
  if (c->sharded && !p2p) {
    for (size_t g = 0; g < c->gcoef.size(); ++g) {
      if (c->gcoef[g] == 0.0) continue;
      if (c->xbuf == nullptr) return fail(RSV_ERR_STATE, "exchange mode without an exchange buffer (rsv_set_shard)");
      CUDA_TRY(cudaStreamSynchronize(c->st));
      int rc = comm_call(c, RSV_COMM_EXCHANGE_START, c->logical[kidx(c, j)], c->gpeer[g], nullptr, 0);
      if (rc) return rc;
      started = true;
      break;
    }
  }
  for (size_t pi = 0; pi < np; ++pi) {
    const PassPlan& p = c->plan[pi];
    if (c->sharded && pi + 1 == np) {
      if (np == 1) {
        // a single pass has no partial sums to add the global flips to: seed u = -beta' s_{j-1}
        // (its elementwise operand) in slot j+1 and let the pass read u instead
        const uint64_t nloc = 1ull << c->n;
        if (j > 0) {
          CUDA_TRY(rsv::launch_scale(kvec(c, j + 1), kvec(c, j - 1), make_double2(prev_coef, 0.0), nloc, 0, c->st));
        } else {
          CUDA_TRY(cudaMemsetAsync(kvec(c, j + 1), 0, sizeof(cplx) * nloc, c->st));
        }
      }
      int rc = shard_before_last(c, j, sigma, started, p2p);
      if (rc) return rc;
    }
    if (p.chunk) {
      int rc = launch_chunk_pass(c, p, omegas, deltas, kvec(c, j), rsv::SC_SG + j, j > 0 ? kvec(c, j - 1) : nullptr,
                                 kvec(c, j + 1), j);
      if (rc) return rc;
      continue;
    }
    rsv::PassArgs A{};
    const bool last = pi + 1 == np;
    A.kind = last ? rsv::PASS_LAST_LANCZOS : (pi == 0 ? rsv::PASS_FIRST : rsv::PASS_MID);
    A.sh = p.sh;
    A.fl = flips_for(p, omegas, rsv::pass_threads_for(p.sh.a + p.sh.g, A.kind, p.sh.a));
    A.dg = diag_for(c, p, deltas);
    A.x = kvec(c, j);
    A.x_scale_slot = rsv::SC_SG + j;
    A.j = j;
    A.sc = c->d_sc;
    A.part = c->d_part;
    A.counter = c->d_counter;
    // elementwise operand: -beta' s_{j-1} joins in the first pass, the partial sum u in the others
    if (pi == 0) {
      A.ein = j > 0 ? kvec(c, j - 1) : nullptr;
      A.ein_is_prev = 1;
      if (c->sharded && np == 1) {
        A.ein = kvec(c, j + 1);
        A.ein_is_prev = 0;
      }
    } else {
      A.ein = kvec(c, j + 1);
      A.ein_is_prev = 0;
    }
    A.out = kvec(c, j + 1);   // u in place, then s_{j+1}
    if (p2p && !last) {
      // the partner reads (NVLink) are spread over the passes before the last one so they overlap
      // more local work: active global qubit number i goes to pass i mod (np - 1)
      int active = 0;
      for (size_t g = 0; g < c->gcoef.size(); ++g) {
        if (c->gcoef[g] == 0.0) continue;
        if (active++ % (int)(np - 1) != (int)pi) continue;
        A.peer[A.npeer] = c->peer_slots[g][c->logical[kidx(c, j)]];
        A.peer_coef[A.npeer] = c->gcoef[g];
        ++A.npeer;
      }
    }
    A.qsweep = last ? 1 : 0;
    A.raw = (last && c->sharded) ? 1 : 0;
    A.mail = (last && !c->sharded) ? c->d_mail : nullptr;
    set_tile_load(c, A);
    set_peer_load(c, A);
    // with the TMA ring the lo pass runs 256 threads x 16 amplitudes (the 512-thread variant spills
    // under its 128-register cap); the kernel launcher picks the same count (rsv::peer_pass_threads)
    if (A.peer_tma) A.fl = flips_for(p, omegas, rsv::peer_pass_threads(A.kind, A.sh.a));
    if (A.npeer > 0) ++c->peer_passes[A.peer_tma ? 0 : 1];
    prof_begin(c, family_of(pi, np));
    CUDA_TRY(rsv::launch_pass(A, c->st));
    prof_end(c);
  }
  return RSV_OK;
}

// Full re-orthogonalisation of w_j = s_{j+1} against s_0..s_j (krylov.py:103-104, classical
// Gram-Schmidt: one multi-dot pass, then one Krylov-combination pass that subtracts the projections
// in place and recomputes ||w||^2 and the q-sweep of the last pass). Returns the new beta_j and
// rewrites beta_j, sigma_{j+1}, q_{j+1} on the device.
int reorthogonalize(rsv_context* c, int j, double n0, const std::vector<double>& betas, const double* omegas,
                    const double* deltas, double* beta_out) {
  const int k = j + 1;
  if (k + 1 > rsv::kMaxKrylov) return fail(RSV_ERR_ARG, "re-orthogonalisation of %d vectors exceeds %d", k, rsv::kMaxKrylov - 1);
  rsv::MultiDotArgs M{};
  for (int i = 0; i < k; ++i) M.v[i] = slot(c, i);
  M.w = slot(c, j + 1);
  M.k = k;
  M.n = 1ull << c->n;
  M.part = c->d_part;
  M.stride = kPartStride;
  M.counter = c->d_counter;
  M.out = c->d_dots;
  CUDA_TRY(rsv::launch_multidot(M, c->st));
  std::vector<double> dots(2 * k);
  CUDA_TRY(cudaMemcpyAsync(dots.data(), c->d_dots, sizeof(double) * 2 * k, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  rsv::CombineArgs A{};
  const PassPlan& last = c->plan.back();
  A.sh = last.sh;
  A.qsweep = 1;
  A.fl = flips_for(last, omegas, rsv::combine_threads(last.sh.a + last.sh.g));
  A.dg = diag_for(c, last, deltas);
  A.k = k + 1;
  A.v[0] = slot(c, j + 1);
  A.coef[0] = make_double2(1.0, 0.0);
  for (int i = 0; i < k; ++i) {
    const double sg = i == 0 ? 1.0 / n0 : 1.0 / betas[i - 1];
    A.v[i + 1] = slot(c, i);
    A.coef[i + 1] = make_double2(-sg * sg * dots[2 * i], -sg * sg * dots[2 * i + 1]);
  }
  A.out = slot(c, j + 1);   // elementwise: in place
  A.nmask = 0;
  A.sc = c->d_sc;
  A.part = c->d_part;
  A.counter = c->d_counter;
  A.sc_out = rsv::SC_GF + 1;
  prof_begin(c, 3);
  CUDA_TRY(rsv::launch_combine(A, c->st));
  prof_end(c);
  double raw[2];
  CUDA_TRY(cudaMemcpyAsync(raw, c->d_sc + rsv::SC_GF + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  const double nrm2 = raw[0], beta = std::sqrt(std::max(0.0, nrm2));
  const double sg = beta > 0.0 ? 1.0 / beta : 0.0, q = nrm2 > 0.0 ? raw[1] / nrm2 : 0.0;
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_BE + j, &beta, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_SG + j + 1, &sg, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sc + rsv::SC_Q + j + 1, &q, sizeof(double), cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  *beta_out = beta;
  return RSV_OK;
}

// Krylov combination when the basis outgrew the resident slots (k > K = cap >= 4): s_0..s_{K-2} are
// resident, the ring (slots K-1, K) holds s_{k-1} and s_k. (1) psi = sum over the resident vectors
// and s_{k-1}, in place in slot 0; (2) iterations K-2 .. k-3 are re-run (same kernels, same inputs:
// the same vectors bit for bit) to regenerate s_{K-1} .. s_{k-2} through the ring, and every two of
// them are added to psi by an in-place combination; the last one also carries the next step's
// q-sweep, the norm and the observables. (K >= 4: the first re-run iteration reads s_{K-3} as its
// previous vector, which must not be slot 0, where psi is being accumulated.)
int combine_with_regeneration(rsv_context* c, int k, const std::vector<zc>& coef, const std::vector<double>& betas,
                              const double* omegas, const double* deltas, const double* qo, const double* qd,
                              int obs, double qoff) {
  const int K = kcap(c);
  cplx* psi = slot(c, 0);
  {
    std::vector<const cplx*> v;
    std::vector<zc> cf;
    for (int i = 0; i <= K - 2; ++i) {
      v.push_back(kvec(c, i));
      cf.push_back(coef[i]);
    }
    v.push_back(kvec(c, k - 1));
    cf.push_back(coef[k - 1]);
    int rc = run_combine(c, (int)v.size(), cf, psi, nullptr, nullptr, 0, 0.0, &v);
    if (rc) return rc;
  }
  // regenerate s_{K-1} .. s_{k-2}: iteration j writes s_{j+1}
  std::vector<int> pending;
  for (int j = K - 2; j <= k - 3; ++j) {
    const double sigma = betas[j - 1] > 0.0 ? 1.0 / betas[j - 1] : 0.0;   // j >= K-2 >= 1
    const double sg_prev = j == 1 ? (c->n0sq_global > 0.0 ? 1.0 / std::sqrt(c->n0sq_global) : 0.0)
                                  : (betas[j - 2] > 0.0 ? 1.0 / betas[j - 2] : 0.0);
    int rc = launch_lanczos_iteration(c, j, omegas, deltas, sigma, -betas[j - 1] * sg_prev);
    if (rc) return rc;
    if (c->sharded) {
      rc = shard_finish_iteration(c, j);
      if (rc) return rc;
    }
    pending.push_back(j + 1);
    const bool final = j + 1 == k - 2;
    if (pending.size() == 2 || final) {
      std::vector<const cplx*> v(1, psi);
      std::vector<zc> cf(1, zc(1.0, 0.0));
      for (int i : pending) {
        v.push_back(kvec(c, i));
        cf.push_back(coef[i]);
      }
      pending.clear();
      rc = run_combine(c, (int)v.size(), cf, psi, final ? qo : nullptr, final ? qd : nullptr, final ? obs : 0,
                       qoff, &v);
      if (rc) return rc;
    }
  }
  return RSV_OK;
}

// One Lanczos run on the resident state for a time step of dt_rest (<= the requested step).
// Returns the fraction of dt_rest actually advanced (1 when converged on the full step, < 1
// when the Krylov basis hit the HBM cap and the step was split).
int lanczos_run(rsv_context* c, const double* omegas, const double* deltas, double dt_rest, double tol, int kmax,
                double norm_eps, const double* q_omegas, const double* q_deltas, bool last_run, int observe,
                rsv_krylov_report* rep, bool first_run, double* advanced, bool* zero_vector) {
  *zero_vector = false;
  bool need_prep = !c->prep_valid || c->prep_key != prep_key_for(c, omegas, deltas, c->offset);
  if (c->sharded) {   // collectives must be entered by every shard: decide together
    double flag = need_prep ? 1.0 : 0.0;
    int rc = comm_call(c, RSV_COMM_ALLREDUCE, -1, -1, &flag, 1);
    if (rc) return rc;
    need_prep = flag > 0.0;
  }
  if (need_prep) {
    int rc = prepare(c, omegas, deltas);
    if (rc) return rc;
  }
  int rc = ensure_dl(c, deltas, c->offset);
  if (rc) return rc;
  CUDA_TRY(cudaMemsetAsync(c->d_sc + rsv::SC_AP, 0, sizeof(double) * 128, c->st));

  const double tau = dt_rest * kNsToUs;
  const int cap = kcap(c);
  std::vector<double> alphas, betas;
  std::vector<zc> y;
  double residual = INFINITY, n0 = 0.0, beta = 0.0;
  bool converged = false;
  int k = 0;
  // Speculative launch (small registers, where the host round trip per iteration is comparable to
  // the kernels): iteration j+1 is enqueued before the host tests iteration j, when its output slot
  // s_{j+2} is resident (never a ring slot holding a basis vector the combination may still need).
  // A speculative iteration after convergence is wasted GPU time but touches nothing in use.
  const bool spec = !c->sharded && !c->reorth &&
                    (c->speculate > 0 || (c->speculate < 0 && c->n <= kSpeculateMaxQubits));
  int launched = 0;
  auto enqueue = [&](int j) -> int {
    // host copies of sigma_j and -beta_{j-1} sigma_{j-1} (sharded runs only: the global flips and
    // single-pass plans; the kernels read the device scalars)
    double sigma = 0.0, prev_coef = 0.0;
    if (c->sharded)
      sigma = j == 0 ? (c->n0sq_global > 0.0 ? 1.0 / std::sqrt(c->n0sq_global) : 0.0)
                     : (betas.back() > 0.0 ? 1.0 / betas.back() : 0.0);
    if (j > 0 && c->sharded) {
      const double sg_prev = j == 1 ? (c->n0sq_global > 0.0 ? 1.0 / std::sqrt(c->n0sq_global) : 0.0)
                                    : (betas[j - 2] > 0.0 ? 1.0 / betas[j - 2] : 0.0);
      prev_coef = -betas[j - 1] * sg_prev;
    }
    int rc2 = launch_lanczos_iteration(c, j, omegas, deltas, sigma, prev_coef);
    if (rc2) return rc2;
    if (c->sharded) {
      rc2 = shard_finish_iteration(c, j);
      if (rc2) return rc2;
    }
    if (c->sharded && c->d_red == nullptr) {   // scalars finished by the host (all-reduced): copy them
      CUDA_TRY(cudaMemcpyAsync(c->h_mail + 1 + 2 * j, c->d_sc + rsv::SC_AL + j, sizeof(double),
                               cudaMemcpyDeviceToHost, c->st));
      CUDA_TRY(cudaMemcpyAsync(c->h_mail + 2 + 2 * j, c->d_sc + rsv::SC_BE + j, sizeof(double),
                               cudaMemcpyDeviceToHost, c->st));
      if (j == 0)
        CUDA_TRY(cudaMemcpyAsync(c->h_mail, c->d_sc + rsv::SC_N0SQ, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    }   // else the last pass wrote them to the mapped mailbox
    CUDA_TRY(cudaEventRecord(c->iter_ev[j & 1], c->st));
    ++launched;
    return RSV_OK;
  };
  for (int j = 0;; ++j) {
    if (launched == j) {
      rc = enqueue(j);
      if (rc) return rc;
    }
    if (spec && launched == j + 1 && j + 2 <= cap && j + 1 < kmax) {
      rc = enqueue(j + 1);
      if (rc) return rc;
    }
    CUDA_TRY(cudaEventSynchronize(c->iter_ev[j & 1]));
    rep->matvecs += 1;   // products the step uses (a discarded speculative iteration is not counted)
    prof_collect(c);
    const volatile double* mail = c->h_mail;
    if (j == 0) {
      n0 = std::sqrt(std::max(0.0, (double)mail[0]));
      if (first_run) {
        rep->norm_in = n0;
        rep->alpha0 = mail[1];
      }
      if (n0 <= norm_eps) {   // krylov.py:83-84: zero vector returned unchanged
        *zero_vector = true;
        *advanced = 1.0;
        return RSV_OK;
      }
    }
    alphas.push_back((double)mail[1 + 2 * j]);
    beta = mail[2 + 2 * j];
    if (c->reorth) {
      rc = reorthogonalize(c, j, n0, betas, omegas, deltas, &beta);
      if (rc) return rc;
    }
    residual = beta * std::abs(tridiag_exp(alphas, betas, tau, nullptr));
    k = (int)alphas.size();
    double scale = 1.0;
    for (double a : alphas) scale = std::max(scale, std::fabs(a));
    for (double b : betas) scale = std::max(scale, b);
    if (residual <= tol || beta <= kBreakdownRtol * scale) {   // krylov.py:111
      converged = true;
      break;
    }
    if (k >= kmax) break;                                       // krylov.py:114
    // resident-basis cap: continue in the slot ring and regenerate the overwritten vectors for the
    // combination (exact: the same deterministic kernels recompute them bit for bit); the opt-in
    // re-orthogonalisation needs the whole basis resident and splits the step in time instead
    if (k >= (c->reorth || !c->tail_regen ? cap : kRegenMax) || (cap < 4 && k >= cap)) break;
    betas.push_back(beta);
  }

  double frac = 1.0;
  if (!converged && k >= cap && k < kmax) {
    // HBM cap reached: exp(-i tau H) = exp(-i (tau - tau') H) exp(-i tau' H) exactly. The basis
    // already built gives the largest tau' whose a-posteriori estimate meets the tolerance
    // (bisection on the same T_k); the caller continues with the rest of the step.
    double lo = 0.0, hi = 1.0, r_lo = 0.0;
    for (int it = 0; it < 48; ++it) {
      const double mid = 0.5 * (lo + hi);
      const double r = beta * std::abs(tridiag_exp(alphas, betas, mid * tau, nullptr));
      if (r <= tol) {
        lo = mid;
        r_lo = r;
      } else {
        hi = mid;
      }
    }
    if (lo > 0.0) {
      frac = lo;
      residual = r_lo;
      converged = true;
    }
  }
  tridiag_exp(alphas, betas, frac * tau, &y);
  rep->iterations = std::max(rep->iterations, k);
  rep->residual = std::max(rep->residual, residual);
  if (!converged) rep->converged = 0;

  // psi_new = n0 * sum_i y_i v_i, v_0 = s_0/n0, v_i = s_i / beta_{i-1}
  std::vector<zc> coef(k);
  for (int i = 0; i < k; ++i) {
    const double sigma = i == 0 ? 1.0 / n0 : 1.0 / betas[i - 1];
    coef[i] = y[i] * (n0 * sigma);
  }
  const bool more = frac < 1.0;
  const double* qo = more ? omegas : q_omegas;
  const double* qd = more ? deltas : q_deltas;
  const int obs = (!more && last_run && observe) ? 1 : 0;
  const double qoff = more ? c->offset : c->next_offset;
  if (k <= cap) {
    // elementwise, so in place: every amplitude of s_0 is read before it is overwritten
    rc = run_combine(c, k, coef, slot(c, 0), qo, qd, obs, qoff);
    if (rc) return rc;
  } else {
    rc = combine_with_regeneration(c, k, coef, betas, omegas, deltas, qo, qd, obs, qoff);
    if (rc) return rc;
    rep->regenerated += k - cap;
    rep->matvecs += k - cap;
  }
  if (qo != nullptr) {
    c->prep_key = prep_key_for(c, qo, qd, more ? c->offset : c->next_offset);
    c->prep_valid = true;
  } else {
    c->prep_valid = false;
  }
  *advanced = frac;
  return RSV_OK;
}

// One exact step of length dt on the resident state, split into as many Lanczos runs as the
// resident Krylov basis requires.
int expm_step_impl(rsv_context* c, const double* omegas, const double* deltas, double dt_ns, double tol,
                   int kmax, double norm_eps, const double* next_omegas, const double* next_deltas,
                   int observe, rsv_krylov_report* rep) {
  rep->converged = 1;
  rep->residual = 0.0;
  double remaining = dt_ns;
  for (int run = 0;; ++run) {
    if (run > 100000) return fail(RSV_ERR_NOT_CONVERGED, "step split into more than 1e5 Krylov runs");
    double frac = 1.0;
    bool zero = false;
    int rc = lanczos_run(c, omegas, deltas, remaining, tol, kmax, norm_eps, next_omegas, next_deltas, true,
                         observe, rep, run == 0, &frac, &zero);
    if (rc) return rc;
    if (zero) {   // krylov.py:83-84 returns the zero vector unchanged; the observables still report it
      if (observe) {
        std::vector<double> tmp(c->masks.size() + 1);
        double nsq = 0.0;
        rc = rsv_measure(c, tmp.data(), &nsq);
        if (rc) return rc;
      }
      return RSV_OK;
    }
    if (!rep->converged || frac >= 1.0) return RSV_OK;
    remaining *= (1.0 - frac);
    rep->substeps += 1;
  }
}

}  // namespace

extern "C" {

int rsv_version(void) { return 10000; }

const char* rsv_last_error(void) { return g_err.c_str(); }

int rsv_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return fail(RSV_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *out = n;
  return RSV_OK;
}

int rsv_create(int n_qubits, const double* interaction_u, int diag_mode, void* stream, rsv_context** out) {
  if (out == nullptr) return fail(RSV_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > rsv::kMaxQubits)
    return fail(RSV_ERR_ARG, "n_qubits=%d outside [1, %d]", n_qubits, rsv::kMaxQubits);
  if (diag_mode != RSV_DIAG_FLY && diag_mode != RSV_DIAG_VEC)
    return fail(RSV_ERR_ARG, "unknown diag_mode %d", diag_mode);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(RSV_ERR_CUDA, "no CUDA device: the rsv hot path has no CPU fallback");
  rsv_context* c = new rsv_context();
  c->n = n_qubits;
  c->diag_mode = diag_mode;
  c->st = reinterpret_cast<cudaStream_t>(stream);
  cudaGetDevice(&c->device);
  c->h_u.assign(interaction_u, interaction_u + (size_t)n_qubits * n_qubits);
  build_plan(c);
  const int maxgrid = rsv::max_grid_rows();
  const int alo = std::min(n_qubits, rsv::kLoBits);
  const size_t gc_rows = size_t(1) << (n_qubits - alo);
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = cudaMalloc(&c->d_u, sizeof(double) * n_qubits * n_qubits);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_sc, sizeof(double) * rsv::SC_SIZE);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_part, sizeof(double) * (size_t)maxgrid * kPartStride);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_counter, sizeof(unsigned) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_dl, sizeof(double) << rsv::kLoBits);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_gc, sizeof(double) * rsv::kGcStride * gc_rows);
  const size_t done_rows = n_qubits > 15 ? size_t(1) << (n_qubits - 15) : 1;
  if (e == cudaSuccess) e = cudaMalloc(&c->d_dots, sizeof(double) * 2 * rsv::kMaxKrylov);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_ticket, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_done, sizeof(unsigned) * done_rows);
  if (e == cudaSuccess) e = cudaMemset(c->d_ticket, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->d_done, 0, sizeof(unsigned) * done_rows);

  if (e == cudaSuccess) e = cudaMallocHost(&c->h_pin, sizeof(double) * rsv::SC_SIZE);
  if (e == cudaSuccess) e = cudaHostAlloc(&c->h_mail, sizeof(double) * (2 * 128 + 2), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&c->d_mail, c->h_mail, 0);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->obs_event, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->iter_ev[0], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->iter_ev[1], cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaMemcpy(c->d_u, c->h_u.data(), sizeof(double) * n_qubits * n_qubits, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(c->d_counter, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess) e = cudaMemset(c->d_sc, 0, sizeof(double) * rsv::SC_SIZE);
  double one = 1.0;
  if (e == cudaSuccess) e = cudaMemcpy(c->d_sc + rsv::SC_ONE, &one, sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = rsv::launch_tile_table(alo, n_qubits, c->d_u, c->d_gc, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    rsv_destroy(c);
    return fail(RSV_ERR_CUDA, "rsv_create: %s", cudaGetErrorString(e));
  }
  *out = c;
  return RSV_OK;
}

void rsv_destroy(rsv_context* c) {
  if (c == nullptr) return;
  cudaFree(c->d_u);
  cudaFree(c->d_sc);
  cudaFree(c->d_part);
  cudaFree(c->d_counter);
  cudaFree(c->d_dl);
  cudaFree(c->d_gc);
  cudaFree(c->d_ticket);
  cudaFree(c->d_dots);
  cudaFree(c->d_done);
  if (c->h_pin) cudaFreeHost(c->h_pin);
  if (c->h_mail) cudaFreeHost(c->h_mail);
  if (c->obs_event) cudaEventDestroy(c->obs_event);
  for (cudaEvent_t ev : c->iter_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  delete c;
}

int rsv_set_stream(rsv_context* c, void* stream) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  c->st = reinterpret_cast<cudaStream_t>(stream);
  return RSV_OK;
}

int rsv_bind_slots(rsv_context* c, void* const* slots, int nslots) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (nslots < 2) return fail(RSV_ERR_ARG, "need at least 2 slots (state + one Lanczos vector), got %d", nslots);
  if (nslots - 1 > rsv::kMaxKrylov)
    nslots = rsv::kMaxKrylov + 1;   // extra slots are never used
  c->phys.assign(slots, slots + nslots);
  c->maps.clear();
  for (int i = 0; i < nslots; ++i) {
    if (c->phys[i] == nullptr || (reinterpret_cast<uintptr_t>(c->phys[i]) & 15u))
      return fail(RSV_ERR_ARG, "slot %d is NULL or not 16-byte aligned", i);
  }
  c->logical.resize(nslots);
  for (int i = 0; i < nslots; ++i) c->logical[i] = i;
  c->prep_valid = false;
  return RSV_OK;
}

int rsv_state_slot(rsv_context* c, int* out) {
  if (!c || c->logical.empty()) return fail(RSV_ERR_STATE, "no slots bound");
  *out = c->logical[0];
  return RSV_OK;
}

int rsv_bind_diag_vector(rsv_context* c, double* dev_diag, int fill_interaction) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  c->d_dvec = dev_diag;
  if (dev_diag != nullptr && fill_interaction) {
    CUDA_TRY(rsv::launch_interaction_diag(c->n, c->d_u, nullptr, dev_diag, c->st));
  }
  c->prep_valid = false;
  return RSV_OK;
}

int rsv_build_diagonal(rsv_context* c, const double* deltas, double* dev_out) {
  if (!c || !deltas || !dev_out) return fail(RSV_ERR_ARG, "NULL argument");
  CUDA_TRY(rsv::launch_interaction_diag(c->n, c->d_u, deltas, dev_out, c->st));
  return RSV_OK;
}

int rsv_state_modified(rsv_context* c) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  c->prep_valid = false;
  return RSV_OK;
}

int rsv_apply_hamiltonian(rsv_context* c, const double* omegas, const double* deltas, const void* psi, void* out) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (psi == nullptr || out == nullptr) return fail(RSV_ERR_ARG, "NULL vector");
  if (c->diag_mode == RSV_DIAG_VEC && c->d_dvec == nullptr)
    return fail(RSV_ERR_STATE, "diag_mode VEC needs rsv_bind_diag_vector first");
  const size_t np = c->plan.size();
  if (np > 1 && psi == out) return fail(RSV_ERR_ARG, "psi and out must not alias for N > %d", rsv::kLoBits);
  if (c->sharded) return fail(RSV_ERR_STATE, "rsv_apply_hamiltonian applies the local operator only: unset the shard");
  int rc = ensure_dl(c, deltas);
  if (rc) return rc;
  for (size_t pi = 0; pi < np; ++pi) {
    const PassPlan& p = c->plan[pi];
    if (p.chunk) {
      rc = launch_chunk_pass(c, p, omegas, deltas, reinterpret_cast<const cplx*>(psi), rsv::SC_ONE, nullptr,
                             reinterpret_cast<cplx*>(out), kScratchJ);
      if (rc) return rc;
      continue;
    }
    rsv::PassArgs A{};
    A.kind = pi + 1 == np ? rsv::PASS_LAST_APPLY : (pi == 0 ? rsv::PASS_FIRST : rsv::PASS_MID);
    A.sh = p.sh;
    A.fl = flips_for(p, omegas, rsv::pass_threads_for(p.sh.a + p.sh.g, A.kind, p.sh.a));
    A.dg = diag_for(c, p, deltas);
    A.x = reinterpret_cast<const cplx*>(psi);
    A.x_scale_slot = rsv::SC_ONE;
    A.j = kScratchJ;
    A.sc = c->d_sc;
    A.part = c->d_part;
    A.counter = c->d_counter;
    A.out = reinterpret_cast<cplx*>(out);
    A.ein = pi == 0 ? nullptr : reinterpret_cast<const cplx*>(out);
    A.ein_is_prev = 0;
    set_tile_load(c, A);
    prof_begin(c, family_of(pi, np));
    CUDA_TRY(rsv::launch_pass(A, c->st));
    prof_end(c);
  }
  return RSV_OK;
}

int rsv_expm_step(rsv_context* c, const double* omegas, const double* deltas, double dt_ns, double tolerance,
                  int max_krylov_dim, double norm_epsilon, const double* next_omegas, const double* next_deltas,
                  int observe, rsv_krylov_report* report) {
  if (!c || !report || !omegas || !deltas) return fail(RSV_ERR_ARG, "NULL argument");
  if (c->logical.empty()) return fail(RSV_ERR_STATE, "no slots bound");
  if (c->diag_mode == RSV_DIAG_VEC && c->d_dvec == nullptr)
    return fail(RSV_ERR_STATE, "diag_mode VEC needs rsv_bind_diag_vector first");
  if (max_krylov_dim < 2) return fail(RSV_ERR_ARG, "max_krylov_dim must be >= 2");
  // max_krylov_dim above the resident basis (<= kMaxKrylov vectors) is not clamped: the reference's
  // not-converged decision (krylov.py:115) uses the caller's value, the basis limit splits the step
  std::memset(report, 0, sizeof(*report));
  c->obs_pending = false;   // observables of an earlier step are never reported as this step's
  if (dt_ns == 0.0) {   // krylov.py:85-86: identity, one iteration
    report->iterations = 1;
    report->converged = 1;
    if (observe) {
      double nsq = 0.0;
      std::vector<double> tmp(c->masks.size());
      int rc = rsv_measure(c, tmp.data(), &nsq);
      if (rc) return rc;
      report->norm_in = std::sqrt(nsq);
    }
    return RSV_OK;
  }
  return expm_step_impl(c, omegas, deltas, dt_ns, tolerance, max_krylov_dim, norm_epsilon, next_omegas,
                        next_deltas, observe, report);
}

int rsv_set_observables(rsv_context* c, const uint64_t* masks, int nmask) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (nmask < 0 || nmask > rsv::kMaxMasks) return fail(RSV_ERR_ARG, "nmask %d outside [0, %d]", nmask, rsv::kMaxMasks);
  c->masks.assign(masks, masks + nmask);
  return RSV_OK;
}

int rsv_get_observables(rsv_context* c, double* out) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (!c->obs_pending) return fail(RSV_ERR_STATE, "no observables were requested on the last step");
  CUDA_TRY(cudaEventSynchronize(c->obs_event));
  const double nsq = c->h_pin[rsv::SC_N0SQ];
  for (int m = 0; m < c->obs_count; ++m) out[m] = nsq > 0.0 ? c->h_pin[rsv::SC_OBS + m] / nsq : 0.0;
  return RSV_OK;
}

int rsv_measure(rsv_context* c, double* out, double* norm_sq) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (c->logical.empty()) return fail(RSV_ERR_STATE, "no slots bound");
  std::vector<zc> one(1, zc(1.0, 0.0));
  int rc = run_combine(c, 1, one, slot(c, 0), nullptr, nullptr, 1);
  if (rc) return rc;
  c->prep_valid = false;
  if (!c->obs_pending) {   // no masks: still report the norm
    CUDA_TRY(cudaMemcpyAsync(c->h_pin + rsv::SC_N0SQ, c->d_sc + rsv::SC_N0SQ, sizeof(double),
                             cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaStreamSynchronize(c->st));
    prof_collect(c);
    if (norm_sq) *norm_sq = c->h_pin[rsv::SC_N0SQ];
    return RSV_OK;
  }
  rc = rsv_get_observables(c, out);
  prof_collect(c);
  if (norm_sq) *norm_sq = c->h_pin[rsv::SC_N0SQ];
  return rc;
}

int rsv_observe(rsv_context* c, const void* psi, const uint64_t* masks, int nmask, double* out, double* norm_sq) {
  if (!c || !psi) return fail(RSV_ERR_ARG, "NULL argument");
  if (nmask < 0 || nmask > rsv::kMaxMasks) return fail(RSV_ERR_ARG, "nmask %d outside [0, %d]", nmask, rsv::kMaxMasks);
  rsv::CombineArgs A{};
  A.sh = c->plan.back().sh;
  A.fl.count = 0;
  A.dg.mode = rsv::DIAG_NONE;
  A.k = 1;
  A.v[0] = reinterpret_cast<const cplx*>(psi);
  A.coef[0] = make_double2(1.0, 0.0);
  A.out = nullptr;   // read-only
  A.qsweep = 0;
  A.nmask = nmask;
  for (int m = 0; m < nmask; ++m) A.mask[m] = masks[m];
  classify_masks(A);
  A.sc = c->d_sc;
  A.part = c->d_part;
  A.counter = c->d_counter;
  // the combine overwrites SC_N0SQ / SC_SG / SC_Q: the resident state is re-prepared on its next step
  CUDA_TRY(rsv::launch_combine(A, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->h_pin + rsv::SC_OBS, c->d_sc + rsv::SC_OBS, sizeof(double) * (nmask > 0 ? nmask : 1),
                           cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaMemcpyAsync(c->h_pin + rsv::SC_SIZE - 3, c->d_sc + rsv::SC_N0SQ, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  c->prep_valid = false;
  const double nsq = c->h_pin[rsv::SC_SIZE - 3];
  for (int m = 0; m < nmask; ++m) out[m] = nsq > 0.0 ? c->h_pin[rsv::SC_OBS + m] / nsq : 0.0;
  if (norm_sq) *norm_sq = nsq;
  return RSV_OK;
}

int rsv_sample(rsv_context* c, const void* psi, const double* uniforms, int64_t shots, int64_t* out_indices,
               double* norm_sq) {
  if (!c || !psi || !uniforms || !out_indices) return fail(RSV_ERR_ARG, "NULL argument");
  if (shots < 1) return fail(RSV_ERR_ARG, "shots must be >= 1, got %lld", (long long)shots);
  const uint64_t n = 1ull << c->n;
  const uint64_t chunks = (n + 4095) / 4096;
  double* d_sums = nullptr;
  double* d_u = nullptr;
  int64_t* d_out = nullptr;
  int rc = RSV_OK;
  cudaError_t e = cudaMallocAsync(&d_sums, sizeof(double) * (chunks + 1), c->st);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_u, sizeof(double) * shots, c->st);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_out, sizeof(int64_t) * shots, c->st);
  uint64_t nchunks = 0;
  std::vector<double> pre(chunks + 1, 0.0);
  if (e == cudaSuccess) e = rsv::launch_chunk_norms(reinterpret_cast<const cplx*>(psi), n, d_sums, &nchunks, c->st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pre.data() + 1, d_sums, sizeof(double) * nchunks, cudaMemcpyDeviceToHost, c->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (e == cudaSuccess) {
    for (uint64_t i = 1; i <= nchunks; ++i) pre[i] += pre[i - 1];   // exclusive chunk prefix, in order
    if (norm_sq) *norm_sq = pre[nchunks];
    e = cudaMemcpyAsync(d_sums, pre.data(), sizeof(double) * (nchunks + 1), cudaMemcpyHostToDevice, c->st);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_u, uniforms, sizeof(double) * shots, cudaMemcpyHostToDevice, c->st);
  if (e == cudaSuccess)
    e = rsv::launch_sample(reinterpret_cast<const cplx*>(psi), n, d_sums, nchunks, d_u, pre[nchunks], shots, d_out,
                           c->st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out_indices, d_out, sizeof(int64_t) * shots, cudaMemcpyDeviceToHost, c->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (e != cudaSuccess) rc = fail(RSV_ERR_CUDA, "rsv_sample: %s", cudaGetErrorString(e));
  cudaFreeAsync(d_sums, c->st);
  cudaFreeAsync(d_u, c->st);
  cudaFreeAsync(d_out, c->st);
  return rc;
}

int rsv_diff_norm_sq(rsv_context* c, const void* x, const void* y, uint64_t n, double* out) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  CUDA_TRY(rsv::launch_diff_norm(reinterpret_cast<const cplx*>(x), reinterpret_cast<const cplx*>(y), n, c->d_part,
                                 c->d_counter, c->d_sc + rsv::SC_OBS, 0, c->st));
  CUDA_TRY(cudaMemcpyAsync(out, c->d_sc + rsv::SC_OBS, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return RSV_OK;
}

int rsv_zdotc(rsv_context* c, const void* x, const void* y, uint64_t n, double* out) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  CUDA_TRY(rsv::launch_zdotc(reinterpret_cast<const cplx*>(x), reinterpret_cast<const cplx*>(y), n, c->d_part,
                             c->d_counter, c->d_sc + rsv::SC_OBS, 0, c->st));
  CUDA_TRY(cudaMemcpyAsync(out, c->d_sc + rsv::SC_OBS, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return RSV_OK;
}

int rsv_lanczos_update(rsv_context* c, void* w, const void* v, const void* vprev, double alpha, double beta,
                       uint64_t n, double* out_norm_sq) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  CUDA_TRY(rsv::launch_lanczos_update(reinterpret_cast<cplx*>(w), reinterpret_cast<const cplx*>(v),
                                      reinterpret_cast<const cplx*>(vprev), alpha, beta, n, c->d_part,
                                      c->d_counter, c->d_sc + rsv::SC_OBS, 0, c->st));
  CUDA_TRY(cudaMemcpyAsync(out_norm_sq, c->d_sc + rsv::SC_OBS, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return RSV_OK;
}

int rsv_axpy(rsv_context* c, void* y, const void* x, double are, double aim, uint64_t n) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  CUDA_TRY(rsv::launch_axpy(reinterpret_cast<cplx*>(y), reinterpret_cast<const cplx*>(x), make_double2(are, aim),
                            n, 0, c->st));
  return RSV_OK;
}

int rsv_scale(rsv_context* c, void* y, const void* x, double are, double aim, uint64_t n) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  CUDA_TRY(rsv::launch_scale(reinterpret_cast<cplx*>(y), reinterpret_cast<const cplx*>(x), make_double2(are, aim),
                             n, 0, c->st));
  return RSV_OK;
}

int rsv_tridiag_exp_e1(const double* alphas, const double* betas, int k, double tau, int full, double* out) {
  if (alphas == nullptr || out == nullptr || k < 1 || (k > 1 && betas == nullptr))
    return fail(RSV_ERR_ARG, "bad tridiagonal arguments");
  std::vector<double> a(alphas, alphas + k), b;
  if (k > 1) b.assign(betas, betas + (k - 1));
  std::vector<zc> y;
  const zc yl = tridiag_exp(a, b, tau, full ? &y : nullptr);
  if (!full) {
    out[0] = yl.real();
    out[1] = yl.imag();
    return RSV_OK;
  }
  for (int i = 0; i < k; ++i) {
    out[2 * i] = y[i].real();
    out[2 * i + 1] = y[i].imag();
  }
  return RSV_OK;
}

int rsv_pass_plan(rsv_context* c, int* out, int max_ints) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  const int np = (int)c->plan.size();
  if (max_ints < 1 + 6 * np) return fail(RSV_ERR_ARG, "buffer too small");
  out[0] = np;
  for (int i = 0; i < np; ++i) {
    out[1 + 6 * i] = c->plan[i].sh.a;
    out[2 + 6 * i] = c->plan[i].sh.p;
    out[3 + 6 * i] = c->plan[i].sh.g;
    out[4 + 6 * i] = c->plan[i].lo ? 1 : 0;
    out[5 + 6 * i] = fused_iteration(c) ? 3 : family_of(i, np);   // 3: both passes in iter2_kernel
    out[6 + 6 * i] = c->plan[i].chunk ? c->plan[i].gm : 0;
  }
  return RSV_OK;
}

int rsv_set_shard(rsv_context* c, rsv_comm_fn comm, void* user, void* exchange_buffer) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (comm == nullptr) {
    c->sharded = false;
    c->comm = nullptr;
    c->xbuf = nullptr;
    return RSV_OK;
  }
  if (c->reorth) return fail(RSV_ERR_STATE, "re-orthogonalisation is on: it is not available for sharded runs");
  if (reinterpret_cast<uintptr_t>(exchange_buffer) & 15u)   // NULL: peer-memory mode only
    return fail(RSV_ERR_ARG, "exchange buffer is not 16-byte aligned");
  c->sharded = true;
  c->comm = comm;
  c->comm_user = user;
  c->xbuf = reinterpret_cast<cplx*>(exchange_buffer);
  c->prep_valid = false;
  return RSV_OK;
}

int rsv_set_shard_scratch(rsv_context* c, double* dev_buf, int count) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (dev_buf != nullptr && count < 2) return fail(RSV_ERR_ARG, "the scratch buffer needs >= 2 doubles");
  c->d_red = dev_buf;
  c->red_count = dev_buf ? count : 0;
  return RSV_OK;
}

int rsv_set_shard_step(rsv_context* c, double offset, double next_offset, int n_global, const double* coef,
                       const int* peer) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (!c->sharded) return fail(RSV_ERR_STATE, "rsv_set_shard_step needs rsv_set_shard first");
  if (n_global < 0 || n_global > 16 || (n_global > 0 && (coef == nullptr || peer == nullptr)))
    return fail(RSV_ERR_ARG, "bad global-qubit list (%d entries)", n_global);
  c->offset = offset;   // enters the prepared-q_0 key (prep_key_for) when the last pass holds the diagonal
  c->next_offset = next_offset;
  c->gcoef.assign(coef, coef + n_global);
  c->gpeer.assign(peer, peer + n_global);
  return RSV_OK;
}

int rsv_enable_peer_access(const void* ptr) {
  if (ptr == nullptr) return fail(RSV_ERR_ARG, "NULL pointer");
  cudaPointerAttributes at{};
  CUDA_TRY(cudaPointerGetAttributes(&at, ptr));
  if (at.type != cudaMemoryTypeDevice) return fail(RSV_ERR_ARG, "not a device pointer");
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  if (at.device == cur) return RSV_OK;
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, cur, at.device));
  if (!can) return fail(RSV_ERR_CUDA, "device %d cannot access device %d's memory (no P2P)", cur, at.device);
  const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();   // clear the non-sticky status
    return RSV_OK;
  }
  if (e != cudaSuccess) return fail(RSV_ERR_CUDA, "cudaDeviceEnablePeerAccess(%d): %s", at.device, cudaGetErrorString(e));
  return RSV_OK;
}

int rsv_shard_peer_stats(rsv_context* c, long long* out2) {
  if (!c || !out2) return fail(RSV_ERR_ARG, "NULL argument");
  out2[0] = c->peer_passes[0];
  out2[1] = c->peer_passes[1];
  return RSV_OK;
}

int rsv_set_shard_peers(rsv_context* c, int n_global, const void* const* ptrs, int nslots) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (n_global == 0 || ptrs == nullptr) {
    c->peer_slots.clear();
    return RSV_OK;
  }
  if (n_global < 0 || n_global > 4) return fail(RSV_ERR_ARG, "peer-memory mode supports 1..4 global qubits, got %d", n_global);
  if (nslots != (int)c->phys.size()) return fail(RSV_ERR_ARG, "peer table has %d slots, %d are bound", nslots, (int)c->phys.size());
  c->peer_slots.assign(n_global, std::vector<const cplx*>(nslots, nullptr));
  for (int g = 0; g < n_global; ++g)
    for (int s = 0; s < nslots; ++s) {
      const void* p = ptrs[(size_t)g * nslots + s];
      if (p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u))
        return fail(RSV_ERR_ARG, "peer slot (%d, %d) is NULL or misaligned", g, s);
      c->peer_slots[g][s] = reinterpret_cast<const cplx*>(p);
    }
  return RSV_OK;
}

int rsv_shard_local_norm_sq(rsv_context* c, double* out) {
  if (!c || !out) return fail(RSV_ERR_ARG, "NULL argument");
  *out = c->local_n0sq;
  return RSV_OK;
}

int rsv_set_speculation(rsv_context* c, int mode) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (mode < -1 || mode > 1) return fail(RSV_ERR_ARG, "speculation mode %d not in {-1, 0, 1}", mode);
  c->speculate = mode;
  return RSV_OK;
}

int rsv_set_fusion(rsv_context* c, int mode) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (mode < -1 || mode > 1) return fail(RSV_ERR_ARG, "fusion mode %d not in {-1, 0, 1}", mode);
  c->fuse = mode;
  return RSV_OK;
}

int rsv_set_tail_regeneration(rsv_context* c, int on) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  c->tail_regen = on != 0;
  return RSV_OK;
}

int rsv_set_reorthogonalize(rsv_context* c, int on) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (on && c->sharded) return fail(RSV_ERR_STATE, "re-orthogonalisation is not available for sharded runs");
  c->reorth = on != 0;
  return RSV_OK;
}

int rsv_set_plan(rsv_context* c, int chunk_group_bits, long long chunk_lag) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (chunk_group_bits != -1 && chunk_group_bits != 0 && (chunk_group_bits < 3 || chunk_group_bits > 9))
    return fail(RSV_ERR_ARG, "chunk_group_bits must be -1 (auto), 0 (off) or 3..9, got %d", chunk_group_bits);
  if (chunk_group_bits > 0 && chunk_gm_for(c->n, chunk_group_bits) == 0)
    return fail(RSV_ERR_ARG, "chunk group of %d bits is invalid at N=%d (needs M tiles of <= 2^%d contiguous and a hi pass)",
                chunk_group_bits, c->n, rsv::ilog2(RSV_CHUNK_THREADS));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  c->plan_gm = chunk_group_bits;
  c->plan_lag = chunk_lag;
  build_plan(c);
  c->prep_valid = false;
  c->dl_valid = false;
  return RSV_OK;
}

int rsv_set_profiling(rsv_context* c, int on) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  if (on < 0) return fail(RSV_ERR_ARG, "profiling period %d < 0", on);
  c->prof = on != 0;
  c->prof_every = on > 0 ? on : 1;
  return RSV_OK;
}

int rsv_get_profile(rsv_context* c, double* ms4, long long* n4) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  CUDA_TRY(cudaStreamSynchronize(c->st));
  prof_collect(c);
  for (int i = 0; i < 4; ++i) {   // sampled: mean of the timed launches x every launch
    ms4[i] = c->prof_n[i] > 0 ? c->prof_ms[i] / (double)c->prof_n[i] * (double)c->prof_all[i] : 0.0;
    n4[i] = c->prof_all[i];
  }
  return RSV_OK;
}

int rsv_reset_profile(rsv_context* c) {
  if (!c) return fail(RSV_ERR_ARG, "NULL context");
  for (int i = 0; i < 4; ++i) {
    c->prof_ms[i] = 0;
    c->prof_n[i] = 0;
    c->prof_all[i] = 0;
  }
  return RSV_OK;
}

}  // extern "C"
