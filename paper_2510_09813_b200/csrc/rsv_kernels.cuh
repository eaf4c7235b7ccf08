// rsv_kernels.cuh -- sm_100a kernels for the matrix-free Rydberg H.psi and the fused Lanczos step.
//
// State layout in HBM: one complex128 (double2, 16 B) per basis index b in [0, 2^N);
// qubit i is bit i of b (reference convention, rydsim/hamiltonian.py:1-8).
//
// H.psi (rydsim/hamiltonian.py:164 apply_hamiltonian, rydsim/_kernels.py:14) is
//   out[b] = d[b] psi[b] + sum_i (Omega_i/2) psi[b ^ (1<<i)]
// Every bit flip must see both partners on chip, but one CTA can hold only 2^12
// amplitudes (64 KB of shared memory), so the N qubits are partitioned into
// "bit groups", one streaming pass each:
//   * the lo pass: tile = bits [0, a) contiguous (a = min(N, 12)); applies the
//     flips on those bits plus the diagonal (on the fly from U, or from a
//     precomputed vector);
//   * hi passes: tile = 2^a contiguous amplitudes (128..512 B runs) x 2^g
//     amplitudes strided along a group of g high bits; applies the flips on
//     the group (the first also the lowest bits, which its tile holds too).
// A tile is moved once into shared memory by the TMA engine (one bulk copy for a
// contiguous tile, a 5-D tensor map for a strided one, completion on mbarriers);
// each partner of a flip is then one 16-byte shared load (bank-conflict free:
// e ^ mask permutes aligned groups of 8 lanes), flips on a thread's own register
// bits are register permutations.
//
// The Lanczos recurrence is fused into the passes (no separate vdot/axpy/norm
// passes): the first/middle passes reduce their part of alpha_j = <v_j|H|v_j>,
// the last pass knows alpha_j completely (its own part q_j was computed one
// iteration earlier from w_{j-1} while that tile was on chip, the "q-sweep"),
// so it writes w_j = H v_j - alpha_j v_j - beta_{j-1} v_{j-1} directly and
// reduces ||w_j||^2 and q_{j+1}. Vectors are kept unnormalised with scales in a
// device scalar array, so normalisation costs no pass.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsv {

typedef double2 cplx;

constexpr int kMaxQubits = 48;
constexpr int kMaxFlips = 16;     // flips per pass (tile bits <= 12)
constexpr int kMaxKrylov = 120;   // vectors in one Krylov combination
constexpr int kMaxMasks = 128;    // observable masks per combine
constexpr int kLoBits = 12;       // tile bits: 2^12 complex128 = 64 KB per tile buffer
constexpr int kGcStride = 14;     // lo-pass tile table row: gc[0..11], hh, tb (112 B, cp.async-able)

// CTA size of the pass kernels (host and device agree on it: the flip split depends on it).
// 512 threads x 8 amplitudes: the top 3 tile bits are register bits.
#ifndef RSV_PASS_THREADS
#define RSV_PASS_THREADS 512
#endif
constexpr int pass_threads(int tb) { return (1 << tb) < RSV_PASS_THREADS ? (1 << tb) : RSV_PASS_THREADS; }
// The middle and last Lanczos passes of a full tile may run fewer threads with more amplitudes
// each (more register bits: fewer shared-memory flips, and in the last pass a cheaper q-sweep),
// when the contiguous run still fits below the thread bits (a <= log2 threads).
#ifndef RSV_LAST_THREADS
#define RSV_LAST_THREADS 256   // measured at N=29: last pass 5.16 -> 5.01 ms (4 register bits)
#endif
constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }
// threads of the fused two-pass iteration kernel (iter2_kernel; registers of 16..21 qubits)
#ifndef RSV_ITER2_THREADS
#define RSV_ITER2_THREADS RSV_LAST_THREADS
#endif
// threads of the L2 chunk pass (its M tiles need 12 - gm <= log2 of this)
#ifndef RSV_CHUNK_THREADS
#define RSV_CHUNK_THREADS RSV_PASS_THREADS
#endif
// the lo pass (PASS_FIRST, contiguous tile) with RSV_LAST_THREADS threads too: 16 amplitudes a thread,
// 4 register bits, one shared-memory flip fewer per amplitude (measured at N=29 on a 1537 MHz box:
// 4.04-4.06 -> 3.87 ms per launch, profiles/r2_last_pass.md); 0: 512 threads x 8 amplitudes
#ifndef RSV_LO_LAST_THREADS
#define RSV_LO_LAST_THREADS 1
#endif
// the mid passes with RSV_MID_THREADS: 128 threads x 32 amplitudes (5 register bits, computed in two
// halves so that 32 amplitudes of x and 16 accumulators fit the register file) -- experiment switch
#ifndef RSV_MID_THREADS
#define RSV_MID_THREADS RSV_LAST_THREADS
#endif
constexpr int pass_threads_for(int tb, int kind, int a) {
  return (kind == 1 && tb == kLoBits && a <= ilog2c(RSV_MID_THREADS))
             ? RSV_MID_THREADS
             : (((kind == 3 || kind == 1) && tb == kLoBits && a <= ilog2c(RSV_LAST_THREADS)) ||
                (RSV_LO_LAST_THREADS && kind == 0 && tb == kLoBits))
                   ? RSV_LAST_THREADS
                   : pass_threads(tb);
}
// Threads of a peer-memory pass with the TMA ring (full tiles): the lo pass too runs RSV_LAST_THREADS
// (its contiguous tile puts a thread's amplitudes at one stride for any count).
constexpr int peer_pass_threads(int kind, int a) {
  return (kind == 0 || kind == 1) ? RSV_LAST_THREADS : pass_threads_for(kLoBits, kind, a);
}
#ifndef RSV_COMBINE_THREADS
#define RSV_COMBINE_THREADS 512
#endif
constexpr int combine_threads(int tb) { return (1 << tb) < RSV_COMBINE_THREADS ? (1 << tb) : RSV_COMBINE_THREADS; }
constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }

// scalar slots (device double array, reset per step)
constexpr int SC_N0SQ = 0;        // ||psi||^2 of the step's input state
constexpr int SC_ONE = 1;         // constant 1.0
constexpr int SC_AP = 16;         // partial alpha (first+mid passes), per iteration
constexpr int SC_Q = SC_AP + 128; // q_j = <v_j|A_last|v_j>
constexpr int SC_AL = SC_Q + 128; // alpha_j
constexpr int SC_BE = SC_AL + 128;// beta_j
constexpr int SC_SG = SC_BE + 128;// sigma_j : v_j = sigma_j * s_j
constexpr int SC_OBS = SC_SG + 128;
constexpr int SC_GF = SC_OBS + kMaxMasks;   // global-flip dot (sharded runs)
constexpr int SC_SIZE = SC_OBS + kMaxMasks + 8;

enum PassKind : int {
  PASS_FIRST = 0,         // out = A x            ; ap[j]  = <x|A x>
  PASS_MID = 1,           // out = uin + A x      ; ap[j] += <x|A x>
  PASS_LAST_APPLY = 2,    // out = uin + A x       (plain H.psi)
  PASS_LAST_LANCZOS = 3,  // out = uin + A x - alpha x ; beta, q_{j+1} (-beta' prev enters in the first pass)
};

enum DiagMode : int { DIAG_NONE = 0, DIAG_FLY = 1, DIAG_VEC = 2 };

struct Shape {
  int n;        // local qubits
  int a;        // contiguous low bits in the tile
  int p;        // first bit of the strided group (p >= a)
  int g;        // bits in the group
  uint64_t n_tiles;
};

struct FlipSet {
  int count;                // flips through shared memory (tile bit < log2(threads))
  int mask[kMaxFlips];      // tile-local bit masks
  double coef[kMaxFlips];   // Omega_q / 2
  double rcoef[5];          // register flips: coefficient of tile bit log2(threads) + b (0 = inactive)
};

struct DiagArgs {
  int mode;                 // DiagMode (only for passes whose tile is [0, a))
  const double* dl;         // 2^a table: lo part of the diagonal (fly: detuning+interaction, vec: detuning)
  const double* gc;         // per-run tile table [tiles][kGcStride] (fly): lo-hi couplings + hi-hi energy
  const double* umat;       // n x n interaction matrix
  const double* dvec;       // 2^n precomputed interaction diagonal (vec)
  double delta[kMaxQubits]; // detunings
};

// How a pass kernel moves a tile into shared memory (TMA path).
enum TileLoad : int {
  LOAD_RUNS = 0,       // per-warp cp.async.bulk of each contiguous run
  LOAD_CONTIG = 1,     // the tile is one contiguous range: a single bulk copy
  LOAD_TENSOR = 2,     // 5-D TMA tensor map (box = the whole strided tile)
};

struct alignas(64) PassArgs {
  CUtensorMap tm_x;                     // TMA descriptors (LOAD_TENSOR) for x and ein
  CUtensorMap tm_e;
  CUtensorMap tm_o;                     // ... and for out (tstore with LOAD_TENSOR)
  int load;                             // TileLoad
  int tstore;                           // output tiles leave through shared memory by TMA stores
                                        // (LOAD_CONTIG: bulk copy, LOAD_TENSOR: tm_o) instead of
                                        // per-thread 16-byte global stores
  Shape sh;
  FlipSet fl;
  DiagArgs dg;
  int kind;
  const cplx* x; int x_scale_slot;      // operand s_j, v_j = sc[slot] * s_j
  const cplx* ein;                      // elementwise operand (may be null): the partial sum u of the
                                        // previous passes (coefficient 1) or, in the first pass of a
                                        // Lanczos iteration, s_{j-1} (coefficient -beta_{j-1} sigma_{j-1})
  int ein_is_prev;
  cplx* out;
  int j;                                // Lanczos iteration
  int qsweep;                           // LAST_LANCZOS: compute q_{j+1}
  int raw;                              // LAST_LANCZOS of a sharded run: store local sums (host all-reduces)
  int npeer;                            // sharded, peer-memory mode (passes before the last): global-qubit
  const cplx* peer[4];                  //   flips read the partner shards' x over NVLink
  double peer_coef[4];                  //   Omega_g / 2
  int peer_tma;                         // 1: partner tiles by TMA (bulk copy for LOAD_CONTIG, tm_peer for
  CUtensorMap tm_peer[4];               //   LOAD_TENSOR: box = one eighth of the tile) into a shared-memory
                                        //   ring; 0: per-thread P2P loads
  double* sc; double* part; unsigned* counter;
  double* mail;                         // LAST_LANCZOS (not raw): mapped pinned host memory receiving
                                        //   [n0sq (j=0)], alpha_j, beta_j -- the host reads them after the
                                        //   iteration's event, no device-to-host copies in the stream
  int dvec_smem;                        // set by the launcher: diag="vec" tiles are staged in shared memory
                                        //   by a bulk copy per tile (contiguous 4096-amplitude tiles)
};

struct CombineArgs {
  Shape sh;
  FlipSet fl;                           // next step's flips on this tile's group (q-sweep)
  DiagArgs dg;                          // next step's diagonal if the group is the lo tile
  int k;
  const cplx* v[kMaxKrylov];
  double2 coef[kMaxKrylov];             // psi_new = sum coef_i * v_i
  cplx* out;
  int qsweep;
  int nmask;                            // observables: sum_b |psi_b|^2 [b & M == M]
  uint64_t mask[kMaxMasks];
  int raw;                              // sharded run: store local sums (host all-reduces)
  int sc_out = -1;                      // >= 0: raw ||out||^2, <out|A|out> to sc[sc_out], sc[sc_out+1] only
  int obs_single;                       // every mask is one bit: obs_cat 0 = constant over the tile
  unsigned char obs_cat[kMaxMasks];     //   (obs_pos = global bit), 1 = thread-index bit, 2 = register
  unsigned char obs_pos[kMaxMasks];     //   bit of the thread (obs_pos = that bit's index)
  double* sc; double* part; unsigned* counter;
};

// L2-resident chunk pass (the first kernel of a Lanczos iteration at N >= 22).
// A chunk = the 2^(12+gm) amplitudes sharing bits [12+gm, n). Two kinds of 4096-amplitude
// tiles cover it: M tiles (2^(12-gm) contiguous x 2^gm rows strided along bits [12, 12+gm))
// and L tiles (bits [0, 12) contiguous). One persistent kernel hands out M and L tiles from a
// single ticket counter; the L tiles of a chunk start only once all of its M tiles are written
// (per-chunk release/acquire counters), M running ~1.5 chunks ahead. The M tiles read x and
// s_{j-1} from HBM and write the partial sum u' (kept in L2); the L tiles re-read x and u'
// from L2 and write u = (A_M + A_L + D) v - beta' s_{j-1} -- one HBM round trip for two bit
// groups. Everything else (reductions, scales, flips) is PASS_FIRST semantics.
struct alignas(64) ChunkArgs {
  CUtensorMap tm_x;                     // M-tile TMA descriptors over x and s_{j-1} (load_m == LOAD_TENSOR)
  CUtensorMap tm_e;
  int load_m;                           // TileLoad of the M tiles (LOAD_TENSOR or LOAD_RUNS)
  Shape shm, shl;                       // M / L tile shapes (n_tiles equal)
  FlipSet flm, fll;
  DiagArgs dg;                          // diagonal (L tiles)
  const cplx* x; int x_scale_slot;
  const cplx* prev;                     // s_{j-1} (may be null: first iteration / plain H.psi)
  cplx* out;                            // u' then u (in place)
  int j;
  int gm;                               // chunk group bits: 2^gm tiles of each kind per chunk
  unsigned long long lag;               // M tiles handed out before the first L tile
  double* sc; double* part; unsigned* counter;
  unsigned long long* ticket;           // work counter (reset by the last CTA)
  unsigned* done;                       // per-chunk finished M tiles (reset by the last CTA)
};

// Fused two-pass Lanczos iteration (plans of exactly [lo, last] with 4096-amplitude tiles, 16..21 qubits):
// both passes in one cooperative launch with a grid barrier between them (iter2_kernel).
struct alignas(64) Iter2Args {
  PassArgs lo;                          // PASS_FIRST, flips for RSV_LAST_THREADS threads
  PassArgs last;                        // PASS_LAST_LANCZOS
  unsigned* gridbar;                    // zero between launches
};

struct MultiDotArgs {
  const cplx* v[kMaxKrylov];
  const cplx* w;
  int k;
  uint64_t n;
  double* part; int stride; unsigned* counter;
  double* out;                          // 2k doubles: <v_i|w> (re, im)
};

// host-side launchers (rsv_kernels.cu); persistent grids sized from the occupancy query
cudaError_t launch_pass(const PassArgs& args, cudaStream_t st);
cudaError_t launch_combine(const CombineArgs& args, cudaStream_t st);
cudaError_t launch_chunk(const ChunkArgs& args, cudaStream_t st);
cudaError_t launch_iter2(const Iter2Args& args, cudaStream_t st);
cudaError_t launch_multidot(const MultiDotArgs& args, cudaStream_t st);
cudaError_t launch_build_dl(int a, int n, const double* umat, const double* delta_host, int with_interaction,
                            double offset, double* dl, cudaStream_t st);
cudaError_t launch_global_flip(cplx* u, const cplx* xp, const cplx* x, double c, uint64_t n, double* part,
                               unsigned* counter, double* result, cudaStream_t st);
cudaError_t launch_tile_table(int a, int n, const double* umat, double* gc, cudaStream_t st);
cudaError_t launch_tile_base(int a, int n, int fly, const double* delta_host, double* gc, cudaStream_t st);
cudaError_t launch_interaction_diag(int n, const double* umat, const double* delta_host, double* dvec,
                                    cudaStream_t st);
cudaError_t launch_zdotc(const cplx* x, const cplx* y, uint64_t n, double* part, unsigned* counter,
                         double* result2, int grid, cudaStream_t st);
cudaError_t launch_diff_norm(const cplx* x, const cplx* y, uint64_t n, double* part, unsigned* counter,
                             double* result, int grid, cudaStream_t st);
cudaError_t launch_lanczos_update(cplx* w, const cplx* v, const cplx* vprev, double alpha, double beta,
                                  uint64_t n, double* part, unsigned* counter, double* result, int grid,
                                  cudaStream_t st);
cudaError_t launch_axpy(cplx* y, const cplx* x, double2 a, uint64_t n, int grid, cudaStream_t st);
cudaError_t launch_chunk_norms(const cplx* psi, uint64_t n, double* sums, uint64_t* nchunks, cudaStream_t st);
cudaError_t launch_sample(const cplx* psi, uint64_t n, const double* prefix, uint64_t nchunks, const double* u,
                          double total, int64_t shots, int64_t* out, cudaStream_t st);
cudaError_t launch_scale(cplx* y, const cplx* x, double2 a, uint64_t n, int grid, cudaStream_t st);
cudaError_t launch_shard_scalars(double* sc, int j, const double* red, double* mail, cudaStream_t st);
int max_grid_rows();   // upper bound on the grid of any kernel writing partial rows

}  // namespace rsv
