/* oracle/qk_oracle.h — TEST INFRASTRUCTURE ONLY (checker + CPU baseline); see qk_oracle.c. */
#ifndef QK_ORACLE_H_
#define QK_ORACLE_H_
#include <stdint.h>

typedef struct {
  double re, im;
} cplx_parts;

/* <0|U(x_i)^dag U(x_j)|0> for the RY + linear-CNOT feature map with L layers. */
cplx_parts qko_amplitude(int n, int L, const double* xi, const double* xj);

/* Amplitudes of pairs[k] = (p, q) -> (A[p], B[q]); A, B row-major [*, n]; pthreads. */
int qko_amplitudes(int n, int L, const double* A, const double* B, const int64_t* pairs,
                   int64_t n_pairs, double* out_re, double* out_im, int threads);

int qko_abi_version(void);
#endif
