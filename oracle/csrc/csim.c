/* ORACLE — test infrastructure only (see oracle/__init__.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU legs may load this library; the product path never does.
 *
 * The gate application loop of oracle/statevector.py written out in plain C, with OpenMP over the
 * amplitude pairs of ONE gate (the gates are still applied one at a time, in list order, with no
 * fusion, blocking or reordering): for a one-qubit gate M on qubit k of an n-qubit state (qubit k
 * = bit n-1-k of the index),
 *     psi'[i0] = M[0][0] psi[i0] + M[0][1] psi[i1],   psi'[i1] = M[1][0] psi[i0] + M[1][1] psi[i1]
 * for every pair i0 = i with bit n-1-k clear, i1 = i0 | 2^(n-1-k)  (Supp. A Eq. 4);
 * CZ negates the amplitudes whose two bits are set.  The 2x2 matrices are NOT defined
 * here: the caller passes them from oracle/gates.py, so this file holds only the index mechanics.
 * Amplitudes are interleaved complex128 (re, im).
 */
#include <stdint.h>
#include <omp.h>

/* psi: 2^n interleaved complex doubles.  codes[g]: 1 = one-qubit gate (matrix mats[8g..8g+7] as
 * re/im of M00, M01, M10, M11), 4 = CZ on (q0[g], q1[g]).  threads <= 0: OpenMP default. */
int oracle_run_gates(double *psi, int n, int64_t ngates, const int32_t *codes, const int32_t *q0,
                     const int32_t *q1, const double *mats, int threads) {
  const int64_t N = (int64_t)1 << n;
  if (threads > 0) omp_set_num_threads(threads);
  for (int64_t g = 0; g < ngates; ++g) {
    if (codes[g] == 4) {
      const int64_t s0 = (int64_t)1 << (n - 1 - q0[g]), s1 = (int64_t)1 << (n - 1 - q1[g]);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < N; ++i)
        if ((i & s0) && (i & s1)) {
          psi[2 * i] = -psi[2 * i];
          psi[2 * i + 1] = -psi[2 * i + 1];
        }
    } else if (codes[g] == 1) {
      const double *M = mats + 8 * g;
      const int64_t s = (int64_t)1 << (n - 1 - q0[g]);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < N; ++i) {
        if (i & s) continue;
        const int64_t j = i | s;
        const double ar = psi[2 * i], ai = psi[2 * i + 1], br = psi[2 * j], bi = psi[2 * j + 1];
        psi[2 * i] = M[0] * ar - M[1] * ai + M[2] * br - M[3] * bi;
        psi[2 * i + 1] = M[0] * ai + M[1] * ar + M[2] * bi + M[3] * br;
        psi[2 * j] = M[4] * ar - M[5] * ai + M[6] * br - M[7] * bi;
        psi[2 * j + 1] = M[4] * ai + M[5] * ar + M[6] * bi + M[7] * br;
      }
    } else {
      return -1;
    }
  }
  return 0;
}

/* psi[i] = v for every i (a state of uniform amplitude, e.g. the caller's H^{(x)n}|0>) */
void oracle_fill(double *psi, int n, double re, double im, int threads) {
  const int64_t N = (int64_t)1 << n;
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    psi[2 * i] = re;
    psi[2 * i + 1] = im;
  }
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
