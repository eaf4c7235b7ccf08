/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference's compiled CPU hot loop.
 *
 * Used solely as the timed CPU baseline (bench.py cpu_baseline / --impl reference).
 * The product never links this file.
 *
 * svref_matvec restates rydsim/_kernels.py:14 (matvec_bitflip_diag, the numba
 * kernel the reference dispatches to for N >= 10, hamiltonian.py:180-187):
 *     out[b] = diag[b] * psi[b] + sum_i half_omega[i] * psi[b ^ (1 << i)]
 * with the same per-element arithmetic, parallelised over b with OpenMP
 * (element results do not depend on evaluation order across b).
 * svref_build_diagonal restates hamiltonian.py:83-122 (doubling construction).
 * svref_zdotc / svref_zaxpy / svref_zscal / svref_norm2 are the vector operations of the
 * reference's Lanczos loop (krylov.py:96-122: np.vdot, w -= c v, w / beta, np.linalg.norm),
 * in place and OpenMP-parallel so the oracle can run that loop at N = 27..30 on the host
 * (oracle/big.py) without numpy temporaries.
 */
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int svref_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Threads of the parallel loops (the CPU baseline uses every core of its affinity mask, whatever
 * OMP_NUM_THREADS a launcher such as torchrun has set). */
void svref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

void svref_matvec(int n, const double* psi, const double* diag, const double* half_omega, double* out) {
  const int64_t dim = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < dim; ++b) {
    double re = diag[b] * psi[2 * b];
    double im = diag[b] * psi[2 * b + 1];
    for (int i = 0; i < n; ++i) {
      const double c = half_omega[i];
      if (c != 0.0) {
        const int64_t p = b ^ ((int64_t)1 << i);
        re += c * psi[2 * p];
        im += c * psi[2 * p + 1];
      }
    }
    out[2 * b] = re;
    out[2 * b + 1] = im;
  }
}

/* Same arithmetic on the output range [b0, b1): a bounded sample of one H.psi
 * (each element still reads all of its N partners across the whole vector). */
void svref_matvec_range(int n, const double* psi, const double* diag, const double* half_omega, double* out,
                        int64_t b0, int64_t b1) {
#pragma omp parallel for schedule(static)
  for (int64_t b = b0; b < b1; ++b) {
    double re = diag[b] * psi[2 * b];
    double im = diag[b] * psi[2 * b + 1];
    for (int i = 0; i < n; ++i) {
      const double c = half_omega[i];
      if (c != 0.0) {
        const int64_t p = b ^ ((int64_t)1 << i);
        re += c * psi[2 * p];
        im += c * psi[2 * p + 1];
      }
    }
    out[2 * b] = re;
    out[2 * b + 1] = im;
  }
}

/* d[b] = -sum_i delta_i bit_i(b) + sum_{i<j} U_ij bit_i bit_j (row-major U, n x n). */
void svref_build_diagonal(int n, const double* deltas, const double* u, double* out) {
  const int64_t dim = (int64_t)1 << n;
  out[0] = 0.0;
  int64_t half = 1;
  for (int k = 0; k < n; ++k) {
    /* extending by qubit k: the bit_k = 1 half adds -delta_k + sum_{i<k} U_ik bit_i */
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < half; ++b) {
      double add = -deltas[k];
      for (int i = 0; i < k; ++i)
        if ((b >> i) & 1) add += u[(int64_t)i * n + k];
      out[half + b] = out[b] + add;
    }
    half <<= 1;
  }
  (void)dim;
}

void svref_fill(int64_t count, double* x, uint64_t seed) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

/* <x|y> = sum conj(x_b) y_b over n complex values (np.vdot, krylov.py:101,104). */
void svref_zdotc(int64_t n, const double* x, const double* y, double* out2) {
  double re = 0.0, im = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : re, im)
  for (int64_t b = 0; b < n; ++b) {
    const double xr = x[2 * b], xi = x[2 * b + 1], yr = y[2 * b], yi = y[2 * b + 1];
    re += xr * yr + xi * yi;
    im += xr * yi - xi * yr;
  }
  out2[0] = re;
  out2[1] = im;
}

/* y += (a_re + i a_im) x (the in-place form of w -= c v, krylov.py:102-104,119-121). */
void svref_zaxpy(int64_t n, double a_re, double a_im, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < n; ++b) {
    const double xr = x[2 * b], xi = x[2 * b + 1];
    y[2 * b] += a_re * xr - a_im * xi;
    y[2 * b + 1] += a_re * xi + a_im * xr;
  }
}

/* y = (a_re + i a_im) x; x may alias y (w / beta, krylov.py:98,119). */
void svref_zscal(int64_t n, double a_re, double a_im, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < n; ++b) {
    const double xr = x[2 * b], xi = x[2 * b + 1];
    y[2 * b] = a_re * xr - a_im * xi;
    y[2 * b + 1] = a_re * xi + a_im * xr;
  }
}

/* sum |x_b|^2 (np.linalg.norm squared, krylov.py:93,105). */
double svref_norm2(int64_t n, const double* x) {
  double s = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : s)
  for (int64_t b = 0; b < 2 * n; ++b) s += x[b] * x[b];
  return s;
}
