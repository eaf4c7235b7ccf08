/* A plain-C consumer of the drop-in boundary (include/rsv.h), the way a cgo/JNI/FFI binding would
 * drive it: device memory from the CUDA runtime, everything else through the rsv_* entry points.
 * Checks H.psi against the C restatement of the reference matvec (oracle/sv_ref.c, test
 * infrastructure only) and a few exact properties of rsv_expm_step.
 * usage: consumer [--expect-no-gpu] */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "rsv.h"

void svref_build_diagonal(int n, const double* deltas, const double* u, double* out);
void svref_matvec(int n, const double* psi, const double* diag, const double* half_omega, double* out);
void svref_fill(int64_t count, double* x, uint64_t seed);

#define CHECK(x)                                                                     \
  do {                                                                               \
    int rc_ = (x);                                                                   \
    if (rc_ != RSV_OK) {                                                             \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, rsv_last_error());            \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

int main(int argc, char** argv) {
  const int n = 14;
  const size_t dim = (size_t)1 << n;
  double u[14 * 14], om[14], de[14], half[14];
  for (int i = 0; i < n; ++i) {
    om[i] = 1.0 + 0.25 * i;
    half[i] = 0.5 * om[i];
    de[i] = -1.5 + 0.2 * i;
    for (int j = 0; j < n; ++j) {
      const double r = fabs((double)(i - j)) * 1.3 + 0.7 * ((i * 7 + j * 3) % 5 == 0);
      u[i * n + j] = i == j ? 0.0 : 40.0 / pow(r + 1.0, 6.0) * 64.0;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) u[i * n + j] = u[j * n + i];
  rsv_context* ctx = NULL;
  if (argc > 1 && strcmp(argv[1], "--expect-no-gpu") == 0) {
    const int rc = rsv_create(n, u, RSV_DIAG_FLY, NULL, &ctx);   /* no CPU fallback: must fail loudly */
    printf("create without GPU: rc=%d (%s)\n", rc, rsv_last_error());
    return rc == RSV_ERR_CUDA && ctx == NULL && strlen(rsv_last_error()) > 0 ? 0 : 1;
  }
  if (rsv_create(0, u, RSV_DIAG_FLY, NULL, &ctx) != RSV_ERR_ARG || strlen(rsv_last_error()) == 0) return 1;
  CHECK(rsv_create(n, u, RSV_DIAG_FLY, NULL, &ctx));

  /* H.psi through the boundary vs the C restatement of rydsim/_kernels.py:14 */
  double* psi = malloc(sizeof(double) * 2 * dim);
  double* out = malloc(sizeof(double) * 2 * dim);
  double* ref = malloc(sizeof(double) * 2 * dim);
  double* diag = malloc(sizeof(double) * dim);
  svref_fill((int64_t)(2 * dim), psi, 42);
  void *d_psi, *d_out;
  if (cudaMalloc(&d_psi, 16 * dim) != cudaSuccess || cudaMalloc(&d_out, 16 * dim) != cudaSuccess) return 1;
  cudaMemcpy(d_psi, psi, 16 * dim, cudaMemcpyHostToDevice);
  CHECK(rsv_apply_hamiltonian(ctx, om, de, d_psi, d_out));
  cudaMemcpy(out, d_out, 16 * dim, cudaMemcpyDeviceToHost);
  svref_build_diagonal(n, de, u, diag);
  svref_matvec(n, psi, diag, half, ref);
  double err = 0.0, mx = 1.0;
  for (size_t i = 0; i < 2 * dim; ++i) {
    err = fmax(err, fabs(out[i] - ref[i]));
    mx = fmax(mx, fabs(ref[i]));
  }
  printf("H.psi max relative error %.3e\n", err / mx);
  if (err / mx > 1e-12) return 1;

  /* exact time steps: norm and energy (alpha_0) are conserved under a constant H */
  enum { NSLOTS = 24 };
  void* slots[NSLOTS];
  for (int s = 0; s < NSLOTS; ++s)
    if (cudaMalloc(&slots[s], 16 * dim) != cudaSuccess) return 1;
  CHECK(rsv_bind_slots(ctx, slots, NSLOTS));
  int s0 = -1;
  CHECK(rsv_state_slot(ctx, &s0));
  double nrm = 0.0;
  for (size_t i = 0; i < 2 * dim; ++i) nrm += psi[i] * psi[i];
  for (size_t i = 0; i < 2 * dim; ++i) psi[i] /= sqrt(nrm);
  cudaMemcpy(slots[s0], psi, 16 * dim, cudaMemcpyHostToDevice);
  CHECK(rsv_state_modified(ctx));
  uint64_t masks[14];
  for (int q = 0; q < n; ++q) masks[q] = (uint64_t)1 << q;
  CHECK(rsv_set_observables(ctx, masks, n));
  double e0 = 0.0;
  for (int k = 0; k < 5; ++k) {
    rsv_krylov_report rep;
    CHECK(rsv_expm_step(ctx, om, de, 10.0, 1e-10, 100, 1e-14, om, de, 1, &rep));
    if (!rep.converged) return 1;
    if (k == 0) e0 = rep.alpha0;
    if (fabs(rep.alpha0 - e0) > 1e-9 * fmax(1.0, fabs(e0)) || fabs(rep.norm_in - 1.0) > 1e-9) {
      fprintf(stderr, "step %d: energy %.15g vs %.15g, norm %.15g\n", k, rep.alpha0, e0, rep.norm_in);
      return 1;
    }
  }
  double occ[14], nsq = 0.0;
  CHECK(rsv_get_observables(ctx, occ));
  CHECK(rsv_measure(ctx, occ, &nsq));
  for (int q = 0; q < n; ++q)
    if (!(occ[q] >= 0.0 && occ[q] <= 1.0)) return 1;
  if (fabs(nsq - 1.0) > 1e-9) return 1;
  rsv_destroy(ctx);
  for (int s = 0; s < NSLOTS; ++s) cudaFree(slots[s]);
  cudaFree(d_psi);
  cudaFree(d_out);
  printf("c-abi consumer ok: energy %.12f, norm^2 %.15f\n", e0, nsq);
  return 0;
}
