/*
 * oracle/qk_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's quantum-kernel contraction, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm as the
 * CHECKER and the CPU baseline.  Nothing in the product package links or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/tnkernel):
 *   - the kernel circuit of a pair (circuit.py:121-157): U(x_j) = [RY(x_j) on every wire,
 *     CNOT(q, q+1) for q = 0..n-2] x L, followed by adjoint(U(x_i)) = reversed gates,
 *     negated angles, CNOT ladders in descending order;
 *   - RY(theta) = [[cos(theta/2), -sin(theta/2)], [sin(theta/2), cos(theta/2)]] as
 *     complex128 (gate_unitary, circuit.py:94-100), rebuilt per pair like rebind_operands
 *     (network.py:283-302);
 *   - the closed network of circuit_to_network (network.py:125-176): one operand per gate,
 *     (1,0) caps on both ends of every wire, CNOT data[out_c, out_t, in_c, in_t];
 *   - contraction to the scalar <0..0|U_i^dag U_j|0..0> (engine.py:52-108) along a
 *     wire-by-wire path.  Any valid path gives the same scalar (paths.py plan contract); the
 *     reference's greedy plan is not reproduced because only the value is observable.
 *     Every CNOT(q, q+1) is split into a COPY on the control and an XOR on the target joined
 *     by one extent-2 bond, so the cut between wires q and q+1 carries 2L such bonds
 *     (boundary state of 4^L complex entries); each wire is contracted into the boundary in
 *     the gate order of the circuit.  Unlike the GPU path this does NOT cancel C.C^dag, does
 *     not rotate the basis and works in complex128 for any L.
 *   - kernel value |amp|^2 ("probability") or |amp| ("magnitude") (statevector.py:62-70).
 *
 * Pinned by tests/golden/*.npz, produced by running the reference itself
 * (tests/golden/make_golden.py) and checked in tests/test_oracle.py.
 */
#include "qk_oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define MAX_LAYERS 8

/* Apply the 2x2 matrix m (row-major) to the wire value of every boundary slot. */
static void apply_wire(cplx* psi, int nk, const cplx m[4]) {
  for (int k = 0; k < nk; ++k) {
    cplx a = psi[2 * k], b = psi[2 * k + 1];
    psi[2 * k] = m[0] * a + m[1] * b;
    psi[2 * k + 1] = m[2] * a + m[3] * b;
  }
}

/* XOR target: wire value w -> w ^ k_bit (the CNOT control value carried by bond `bit`). */
static void apply_xor(cplx* psi, int nk, int bit) {
  for (int k = 0; k < nk; ++k) {
    if ((k >> bit) & 1) {
      cplx t = psi[2 * k];
      psi[2 * k] = psi[2 * k + 1];
      psi[2 * k + 1] = t;
    }
  }
}

/* Sum out bond `bit` (its value is consumed): slot bit -> 0. */
static void sum_bond(cplx* psi, int nk, int bit) {
  for (int k = 0; k < nk; ++k) {
    if ((k >> bit) & 1) {
      int k0 = k & ~(1 << bit);
      psi[2 * k0] += psi[2 * k];
      psi[2 * k0 + 1] += psi[2 * k + 1];
      psi[2 * k] = 0;
      psi[2 * k + 1] = 0;
    }
  }
}

/* COPY control into a free bond `bit`: the bond takes the wire value. */
static void copy_bond(cplx* psi, int nk, int bit) {
  for (int k = 0; k < nk; ++k) {
    if (((k >> bit) & 1) == 0) {
      int k1 = k | (1 << bit);
      psi[2 * k1 + 1] = psi[2 * k + 1]; /* wire = 1 -> bond = 1 */
      psi[2 * k + 1] = 0;               /* bond = 0 keeps wire = 0 only */
      psi[2 * k1] = 0;
    }
  }
}

/* Move bond `from` into the free bond `to` (slots with `to` set are all zero). */
static void move_bond(cplx* psi, int nk, int from, int to) {
  for (int k = 0; k < nk; ++k) {
    if (((k >> from) & 1) && !((k >> to) & 1)) {
      int k2 = (k & ~(1 << from)) | (1 << to);
      psi[2 * k2] = psi[2 * k];
      psi[2 * k2 + 1] = psi[2 * k + 1];
      psi[2 * k] = 0;
      psi[2 * k + 1] = 0;
    }
  }
}

static void ry(cplx m[4], double theta) {
  double c = cos(theta / 2), s = sin(theta / 2); /* circuit.py:98-100 */
  m[0] = c;
  m[1] = -s;
  m[2] = s;
  m[3] = c;
}

cplx_parts qko_amplitude(int n, int L, const double* xi, const double* xj) {
  cplx_parts out = {NAN, NAN};
  if (n < 1 || L < 1 || L > MAX_LAYERS) return out;
  const int nb = 2 * L;           /* boundary bonds: one per CNOT ladder */
  const int extra = nb;           /* scratch bond for COPY-before-XOR ladders */
  const int nk = 1 << (nb + 1);   /* boundary slots incl. scratch */
  cplx* beta = (cplx*)calloc((size_t)(1 << nb), sizeof(cplx));
  cplx* psi = (cplx*)calloc((size_t)nk * 2, sizeof(cplx));
  if (!beta || !psi) {
    free(beta);
    free(psi);
    return out;
  }
  beta[0] = 1.0;
  for (int q = 0; q < n; ++q) {
    const int has_in = q > 0, has_out = q < n - 1;
    cplx m[4];
    memset(psi, 0, sizeof(cplx) * (size_t)nk * 2);
    for (int k = 0; k < (1 << nb); ++k) psi[2 * k] = beta[k]; /* start cap |0> */
    /* U(x_j): per layer RY(x_j[q]) then ladder m=l (CNOT(q-1,q) before CNOT(q,q+1)) */
    for (int l = 0; l < L; ++l) {
      ry(m, xj[q]);
      apply_wire(psi, nk, m);
      if (has_in) {
        apply_xor(psi, nk, l);
        sum_bond(psi, nk, l);
      }
      if (has_out) copy_bond(psi, nk, l);
    }
    /* U(x_i)^dag: per layer, ladder m=L+l in descending order (CNOT(q,q+1) first) then
     * RY(-x_i[q]) */
    for (int l = 0; l < L; ++l) {
      const int b = L + l;
      if (has_in) {
        if (has_out) copy_bond(psi, nk, extra);
        apply_xor(psi, nk, b);
        sum_bond(psi, nk, b);
        if (has_out) move_bond(psi, nk, extra, b);
      } else if (has_out) {
        copy_bond(psi, nk, b);
      }
      ry(m, -xi[q]);
      apply_wire(psi, nk, m);
    }
    /* end cap <0| */
    for (int k = 0; k < (1 << nb); ++k) beta[k] = psi[2 * k];
  }
  cplx a = beta[0];
  free(beta);
  free(psi);
  out.re = creal(a);
  out.im = cimag(a);
  return out;
}

typedef struct {
  int n, L;
  const double* A;
  const double* B;
  const int64_t* pairs;
  int64_t begin, end;
  double* re;
  double* im;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  for (int64_t k = j->begin; k < j->end; ++k) {
    const int64_t p = j->pairs[2 * k], q = j->pairs[2 * k + 1];
    cplx_parts a = qko_amplitude(j->n, j->L, j->A + p * j->n, j->B + q * j->n);
    j->re[k] = a.re;
    if (j->im) j->im[k] = a.im;
  }
  return NULL;
}

int qko_amplitudes(int n, int L, const double* A, const double* B, const int64_t* pairs,
                   int64_t n_pairs, double* out_re, double* out_im, int threads) {
  if (n < 1 || L < 1 || L > MAX_LAYERS || n_pairs < 0) return 1;
  if (threads < 1) threads = 1;
  if (threads > 512) threads = 512;
  if ((int64_t)threads > n_pairs) threads = (int)(n_pairs > 0 ? n_pairs : 1);
  pthread_t tid[512];
  job_t jobs[512];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (job_t){n, L, A, B, pairs, n_pairs * t / threads, n_pairs * (t + 1) / threads,
                      out_re, out_im};
  }
  if (threads == 1) {
    worker(&jobs[0]);
    return 0;
  }
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  return 0;
}

int qko_abi_version(void) { return 1; }
