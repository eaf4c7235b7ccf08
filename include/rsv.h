/* rsv.h -- C ABI of the B200 state-vector hot path (libprefix "rsv_").
 *
 * Drop-in boundary for the reference's state-vector path (rydsim, Python):
 * the reference's host API (rydsim/hamiltonian.py, rydsim/krylov.py, rydsim/sv.py,
 * rydsim/observables.py) is mirrored in Python by paper_2510_09813_b200/, which
 * binds exactly these symbols through ctypes. Plain pointers and sizes only.
 * Vectors are device pointers to 2^N complex128 values (interleaved re, im),
 * qubit i = bit i of the basis index (rydsim/hamiltonian.py:1-8).
 *
 * All functions return 0 on success and a negative code on failure; the
 * message is available from rsv_last_error(). There is no CPU fallback:
 * without a CUDA device every compute entry point fails with RSV_ERR_CUDA.
 */
#ifndef RSV_H
#define RSV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSV_OK 0
#define RSV_ERR_ARG (-1)
#define RSV_ERR_CUDA (-2)
#define RSV_ERR_STATE (-3)
#define RSV_ERR_NOT_CONVERGED (-4)

#define RSV_DIAG_FLY 1   /* diagonal computed on the fly from U and detunings */
#define RSV_DIAG_VEC 2   /* precomputed float64 interaction diagonal vector + detunings */

typedef struct rsv_context rsv_context;

/* Mirrors rydsim.krylov.KrylovReport (krylov.py:47) plus diagnostics. */
typedef struct {
  int iterations;     /* Lanczos vectors used (largest over sub-steps) */
  int converged;      /* 1 when the a-posteriori estimate met the tolerance */
  double residual;    /* final estimate |beta_k [exp(-i tau T_k)]_{k,1}| */
  double alpha0;      /* <v0|H|v0>: Rayleigh quotient of the input state (Energy observable) */
  double norm_in;     /* ||psi|| of the input state */
  int substeps;       /* >0 when the step was split in time (basis beyond kMaxKrylov, or re-orthogonalisation
                         with a basis beyond the resident slots) */
  int matvecs;        /* H.psi products issued (including regenerated ones) */
  int regenerated;    /* Lanczos vectors recomputed for the combination because the basis outgrew the
                         resident slots (the recurrence continues in a ring of two slots) */
} rsv_krylov_report;

int rsv_version(void);
const char* rsv_last_error(void);
int rsv_device_count(int* out);

/* Context for one register of n_qubits with interaction matrix U (n x n, row-major, host).
 * Replaces the state the reference keeps across evolve_sv (sv.py:80): interaction matrix
 * (hamiltonian.py:66), the interaction diagonal (sv.py:116) and the Krylov workspace.
 * stream: cudaStream_t (may be NULL = legacy default stream). */
int rsv_create(int n_qubits, const double* interaction_u, int diag_mode, void* stream, rsv_context** out);
void rsv_destroy(rsv_context* ctx);
int rsv_set_stream(rsv_context* ctx, void* stream);

/* Bind caller-allocated (e.g. torch) device vectors: nslots >= 2 vectors of 2^n complex128.
 * Slot layout: Krylov basis s_0..s_{nslots-2} (s_0 = state); Lanczos iteration j keeps its partial
 * sums in slot j+1 and turns them into s_{j+1} in place, so the last slot needs no basis vector.
 * The Krylov cap is nslots - 1 vectors; steps needing more are split (exactly) in time. */
int rsv_bind_slots(rsv_context* ctx, void* const* slots, int nslots);
/* Index of the bound slot holding the state (slot 0: the Krylov combination writes it in place). */
int rsv_state_slot(rsv_context* ctx, int* out);
/* Bind a caller-allocated device buffer of 2^n float64 used as the diagonal vector:
 * if fill_interaction != 0 it is filled with sum_{i<j} U_ij n_i n_j (sv.py:116),
 * otherwise the caller's contents are used as an explicit diagonal (HamiltonianSlice.diagonal). */
int rsv_bind_diag_vector(rsv_context* ctx, double* dev_diag, int fill_interaction);
/* Full 2^n diagonal -sum delta_i n_i + sum_{i<j} U_ij n_i n_j into a device buffer
 * (rydsim/hamiltonian.py:114 build_diagonal). Not used by the hot path (diag on the fly). */
int rsv_build_diagonal(rsv_context* ctx, const double* deltas, double* dev_out);
/* The state changed outside rsv (new initial state): invalidate cached per-state scalars. */
int rsv_state_modified(rsv_context* ctx);

/* H.psi, rydsim/hamiltonian.py:164 apply_hamiltonian (+ _kernels.py:14):
 * out = diag(deltas, U) psi + sum_i omegas_i/2 X_i psi. psi and out are device
 * pointers; they may alias only when n <= 12 (single pass). omegas, deltas: host
 * arrays of n values (rad/us). Asynchronous on the context stream. */
int rsv_apply_hamiltonian(rsv_context* ctx, const double* omegas, const double* deltas,
                          const void* psi, void* out);

/* One exact step psi <- exp(-i dt 1e-3 H) psi on the resident state
 * (rydsim/krylov.py:67 expm_multiply with the matvec of sv.py:125-128).
 * next_omegas/next_deltas (may be NULL): the following step's parameters, used to
 * pre-reduce that step's first Lanczos scalar inside the Krylov combination.
 * observe != 0 evaluates the masks set by rsv_set_observables on the new state. */
int rsv_expm_step(rsv_context* ctx, const double* omegas, const double* deltas, double dt_ns,
                  double tolerance, int max_krylov_dim, double norm_epsilon,
                  const double* next_omegas, const double* next_deltas, int observe,
                  rsv_krylov_report* report);

/* Observables as bit masks M: value = sum_b |psi_b|^2 [b & M == M] / sum_b |psi_b|^2.
 * occupation(q): M = 1<<q (observables.py:82); correlation(i,j): M = (1<<i)|(1<<j)
 * (observables.py:102). */
int rsv_set_observables(rsv_context* ctx, const uint64_t* masks, int nmask);
int rsv_get_observables(rsv_context* ctx, double* out_host);
/* Evaluate the masks on the resident state now (blocking). */
int rsv_measure(rsv_context* ctx, double* out_host, double* norm_sq);

/* Same masks on an arbitrary device vector psi (read-only), e.g. observables.occupations(). */
int rsv_observe(rsv_context* ctx, const void* psi, const uint64_t* masks, int nmask, double* out_host,
                double* norm_sq);
/* Basis-state indices drawn from |psi|^2 by inverse CDF (replaces observables.py:167 sample_bitstrings,
 * dense path): `uniforms` are the reference's per-batch PCG64 draws (host), out_indices[s] = the first
 * index whose cumulative |psi|^2 exceeds uniforms[s] * ||psi||^2 (searchsorted side="right"; cdf[-1] = 1).
 * norm_sq (may be NULL) returns ||psi||^2 for the caller's normalisation check. psi has 2^n amplitudes. */
int rsv_sample(rsv_context* ctx, const void* psi, const double* uniforms, int64_t shots, int64_t* out_indices,
               double* norm_sq);
/* sum_b |x_b - y_b|^2 (observables.py:137 norm_difference, computed without cancellation). */
int rsv_diff_norm_sq(rsv_context* ctx, const void* x, const void* y, uint64_t n, double* out);

/* Generic vector kernels for the callable-matvec Lanczos (krylov.py:96-121). */
int rsv_zdotc(rsv_context* ctx, const void* x, const void* y, uint64_t n, double* out_re_im);
int rsv_lanczos_update(rsv_context* ctx, void* w, const void* v, const void* vprev, double alpha,
                       double beta, uint64_t n, double* out_norm_sq);
int rsv_axpy(rsv_context* ctx, void* y, const void* x, double a_re, double a_im, uint64_t n);
int rsv_scale(rsv_context* ctx, void* y, const void* x, double a_re, double a_im, uint64_t n);

/* exp(-i tau T) e1 of the k x k Lanczos tridiagonal T (diagonal alphas[0..k), off-diagonal betas[0..k-1)),
 * host only, no context; the function the step driver uses (Chebyshev expansion on the Gershgorin
 * interval). Replaces rydsim/krylov.py:54 _tridiag_exp_e1 (dense eigh). full != 0: all k components (the
 * Krylov combination's coefficients), out_re_im[2k]; full == 0: only the last one (what the convergence
 * test krylov.py:107-111 reads), out_re_im[2]. */
int rsv_tridiag_exp_e1(const double* alphas, const double* betas, int k, double tau, int full, double* out_re_im);

/* Introspection / measurement support. */
int rsv_pass_plan(rsv_context* ctx, int* out, int max_ints);   /* [np, per pass: a, p, g, lo, family, chunk_gm];
                                                                   family 0 lo, 1 mid, 2 last, 3 fused [lo, last] */
/* Sharding by the top log2(P) qubits (north-star row e; paper_2510_09813_b200/sharding.py). The context
 * is created for the LOCAL qubits (n - log2 P) with the local interaction block; per step the host passes
 * the shard's effective detunings as `deltas` of rsv_expm_step and the rest through rsv_set_shard_step.
 * The driver calls `comm` synchronously (its stream idle):
 *   RSV_COMM_ALLREDUCE       host[0..count) summed over all ranks, in place;
 *   RSV_COMM_EXCHANGE_START  start sending bound slot `slot` to rank `peer` and receiving the peer's copy into
 *                            the exchange buffer (may run concurrently with the local passes);
 *   RSV_COMM_EXCHANGE_WAIT   complete that exchange.
 * Reference counterpart: none (the reference is single-process, rydsim/sv.py:80). */
#define RSV_COMM_ALLREDUCE 1
#define RSV_COMM_EXCHANGE_START 2
#define RSV_COMM_EXCHANGE_WAIT 3
#define RSV_COMM_ALLREDUCE_DEVICE 4   /* `host` is a DEVICE pointer into the buffer of rsv_set_shard_scratch:
                                         enqueue an in-place sum all-reduce of `count` doubles on the context
                                         stream (e.g. NCCL) and return without waiting for it */
typedef int (*rsv_comm_fn)(void* user, int op, int slot, int peer, double* host, int count);
int rsv_set_shard(rsv_context* ctx, rsv_comm_fn comm, void* user, void* exchange_buffer);   /* buffer may be NULL
                                                     in peer-memory mode (rsv_set_shard_peers) */
/* Device scratch (>= 2 doubles) for on-stream all-reduces of the Lanczos scalars (RSV_COMM_ALLREDUCE_DEVICE):
 * with it, a peer-memory sharded iteration has no host synchronisation (alpha's share before the last
 * pass, ||w||^2 and q after it are reduced on the stream and finished by a device kernel). NULL: the
 * host all-reduce path. */
int rsv_set_shard_scratch(rsv_context* ctx, double* dev_buf, int count);
/* This step's constant energy of the shard's global bits (and the next step's), and per global qubit
 * Omega_g/2 (0 = no flip) with the partner rank. */
int rsv_set_shard_step(rsv_context* ctx, double offset, double next_offset, int n_global, const double* coef,
                       const int* peer);
/* Peer-memory mode: ptrs[g * nslots + s] = bound slot s of the partner shard of global qubit g, mapped
 * into this process (CUDA IPC over NVLink / UVA). The first pass then reads the partner shards' s_j
 * directly (P2P loads) instead of exchanging copies; n_global = 0 returns to the exchange mode.
 * Plans with a single pass keep the exchange. */
int rsv_set_shard_peers(rsv_context* ctx, int n_global, const void* const* ptrs, int nslots);
/* Make a (mapped) device pointer of another GPU readable from kernels on the current device
 * (cudaDeviceEnablePeerAccess; a no-op on the same device). */
int rsv_enable_peer_access(const void* ptr);
/* Peer-memory passes launched so far: out[0] with the partner tiles moved by TMA into a shared-memory
 * ring, out[1] with per-thread P2P loads (tiles below 4096 amplitudes, RSV_PEER_TMA=0). */
int rsv_shard_peer_stats(rsv_context* ctx, long long* out2);
/* This shard's share of ||psi||^2 from the last Krylov combination / measurement. */
int rsv_shard_local_norm_sq(rsv_context* ctx, double* out);

/* Beyond the resident Krylov basis (nslots - 1 vectors) the fused step continues the recurrence in a
 * ring of the last two slots and regenerates the overwritten vectors for the combination (default,
 * on), or splits the step exactly in time (off; always the case with re-orthogonalisation). Either
 * way the result meets the reference's tolerance; regeneration keeps the reference's Krylov
 * dimension per step (krylov.py:96-117). */
int rsv_set_tail_regeneration(rsv_context* ctx, int on);
/* Launch Lanczos iteration j+1 before the host has tested iteration j for convergence (hides the host
 * round trip on small registers; a speculative iteration after convergence is discarded):
 * -1 auto (N <= 24, the default), 0 off, 1 on. Never in sharded or re-orthogonalised runs. */
int rsv_set_speculation(rsv_context* ctx, int mode);
/* Run a two-pass Lanczos iteration ([lo, last] plans: 16..21 local qubits, single GPU) as one cooperative
 * launch with a grid barrier between the passes: -1 auto (default: every such plan), 0 off, 1 on.
 * Reference counterpart: none (launch latency). Its kernel time is reported under profile family 0. */
int rsv_set_fusion(rsv_context* ctx, int mode);

/* Full re-orthogonalisation of every new Lanczos vector against the basis (the reference algorithm,
 * krylov.py:103-104; classical Gram-Schmidt, two extra passes over the basis per iteration). Off by
 * default: the fused step uses the plain three-term recurrence. */
int rsv_set_reorthogonalize(rsv_context* ctx, int on);

/* Pass-plan override (tests / tuning): chunk_group_bits -1 = auto (chunk pass at N >= 22), 0 = plain
 * bit-group passes, 3..9 = force the L2-resident chunk pass over bits [0, 12 + g); chunk_lag = M tiles
 * handed out ahead of the first L tile (-1 = auto, 1.5 chunks). No reference counterpart: the reference
 * has one matvec loop (rydsim/_kernels.py:14). */
int rsv_set_plan(rsv_context* ctx, int chunk_group_bits, long long chunk_lag);
/* Kernel timing by CUDA events on the context's stream: 0 off, P >= 1 times one launch in P per kernel
 * family (1: every launch). */
int rsv_set_profiling(rsv_context* ctx, int on);
/* per kernel family: [0]=lo pass, [1]=mid passes, [2]=last pass, [3]=combine; ms (the mean of the timed
 * launches times every launch) and launches */
int rsv_get_profile(rsv_context* ctx, double* ms4, long long* launches4);
int rsv_reset_profile(rsv_context* ctx);

#ifdef __cplusplus
}
#endif
#endif /* RSV_H */
