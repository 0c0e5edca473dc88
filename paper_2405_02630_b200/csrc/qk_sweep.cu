// qk_sweep.cu — sm_100a kernels of the QSVM quantum-kernel hot path.
//
//   gate_build_kernel : angles [N x n] -> per-(sample, qubit) rotation planes (HBM-bound)
//   sweep_kernel      : pair-tiled overlap contraction, bond state in registers (FP64-bound)
//   pairs_kernel      : same recurrence for an explicit pair list (contract_batch drop-in)
//   unpack_kernel     : packed tiles -> dense (symmetrised) kernel matrix
//   dfma_peak_kernel  : FP64 FMA issue-rate microbenchmark (roofline denominator check)
//
// The math (derivation in DESIGN.md §2).  For L = 2 the kernel circuit of a pair
// (circuit.py:151-157) is  U(x_i)^dag U(x_j) = R(-x_i) C^dag R(x_j - x_i) C R(x_j)  after the
// middle C C^dag cancels, so the amplitude is the overlap of two bond-2 MPS and reduces to a
// bond-4 transfer sweep along the qubit chain.  In the rotated basis
//     S+ = V00 + V11,  T+ = V01 + V10,  S- = V00 - V11,  T- = V01 - V10
// with full-angle per-sample values a = cos x, b = sin x and C = cos(x_j - x_i),
// D = sin(x_j - x_i), one qubit is (the 1/2 per qubit is folded into one exact power-of-two
// scale at the end):
//     S+' = (1 + C) S+ + (b_i + b_j) T+        T-' = (a_j - a_i) S+ - D T+
//     S-' = (a_i + a_j) S- + D T-              T+' = (b_i - b_j) T- - (1 - C) S-
// amp = (S+ + T+) 2^-n.  That is 16 FP64 instructions per pair-qubit (4 DMUL, 4 DADD,
// 8 DFMA) against 24 for the textbook (A_i^T V A_j) o RY(delta) form.
// For L = 1 the amplitude is prod_q cos((x_j - x_i)/2) from half-angle planes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>

#include "qk_internal.h"

namespace qk {

// Thread layout of a tile: kTX threads along j with kRJ j-samples each; along i, RI
// i-samples per thread (template parameter: RI = 4 -> 256 threads, RI = 2 -> 512 threads).
// RI = 1: 512 threads over a 32-row work item (every item a half tile, all 16 warps busy with
// 1 x 4 micro-tiles; short chains, where 64-row items leave too few waves).
constexpr int kTX = 16;                 // threads along j
constexpr int kRJ = kTile / kTX;        // j-samples per thread (4)
template <int RI>
struct Geo {
  static constexpr int kRI = RI;
  static constexpr int kRows = RI == 1 ? kTile / 2 : kTile;  // tile rows one item's threads span
  static constexpr int kTY = kRows / RI;           // threads along i
  static constexpr int kThreads = kTX * kTY;
  static constexpr int kWarps = kThreads / 32;
};
constexpr int kChunkElems = kChunk * kTile;            // double2 per block-chunk
constexpr uint32_t kChunkBytes = kChunkElems * 16;     // 16 KB
#ifndef QK_QUNROLL
#define QK_QUNROLL 8
#endif
// qubits unrolled per inner iteration (tuning knob; config-4 bench with RI = 2: 1 -> 1.175,
// 2 -> 1.212, 4 -> 1.222, 8 -> 1.233, 16 -> 1.215 G entries/s)
constexpr int kQUnroll = QK_QUNROLL;
constexpr size_t kSmemBytes =  // ring, barriers + release counters, epilogue stage
    size_t(kStages) * 2 * kChunkBytes + 2 * kStages * 8 +
    size_t(kTile) * (kTile + 1) * 8;

static_assert(kRJ * kTX == kTile, "tile mapping");

// ------------------------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copy (TMA engine, SASS UBLKCP)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef QK_SPIN_WAIT  // diagnostic: non-suspending test_wait spin instead of try_wait
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "QK_SPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra QK_SPIN_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "QK_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra QK_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// A warp's release of a ring stage it has finished reading: acq_rel, so every warp's reads of
// the stage happen-before the refill that the last releaser issues (which then orders the
// async-proxy write after them with fence.proxy.async).  Returns the previous count.
__device__ __forceinline__ int release_stage(int* counter) {
  int old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
               : "=r"(old)
               : "r"(smem_u32(counter))
               : "memory");
  return old;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Timeline instrumentation (diagnostic builds only: -DQK_TIMELINE, tools/timeline_probe.py):
// thread 0 of each CTA records %globaltimer at kernel entry, after the prologue, and per work
// item at its start (after the claim barrier), after its first stage landed, after the sweep
// and after the epilogue.  Read back with qk_timeline_read.
#ifdef QK_TIMELINE
#ifdef QK_TL_GLOBALTIMER
#define QK_TL_CLOCK() ([] { unsigned long long v; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v)); return v; }())
#else  // SM cycle counter (cheap; intra-CTA intervals), converted at the nominal clock
#define QK_TL_CLOCK() ((unsigned long long)clock64())
#endif
constexpr int kTLSlots = 256;  // per CTA: 2 + 4 per item (first 23 items), 96 + k: item k issued,
                               // 128 + k: item k's first stage already full at its start, 160 + k: released,
                               // 192 + k: warp 0 idle in item k
__device__ unsigned long long qk_tl_buf[1024 * kTLSlots];
__device__ __forceinline__ void tl_store(int slot, unsigned long long v) {
  if (slot < kTLSlots && blockIdx.x < 1024) qk_tl_buf[blockIdx.x * kTLSlots + slot] = v;
}
__device__ __forceinline__ void tl_mark(int slot) {
  if (threadIdx.x == 0 && slot < kTLSlots && blockIdx.x < 1024) {
    unsigned long long t;
    t = QK_TL_CLOCK();
    qk_tl_buf[blockIdx.x * kTLSlots + slot] = t;
  }
}
__device__ __forceinline__ void tl_mark_any(int slot) {  // any thread (e.g. a stage refill)
  if (slot < kTLSlots && blockIdx.x < 1024) {
    unsigned long long t;
    t = QK_TL_CLOCK();
    qk_tl_buf[blockIdx.x * kTLSlots + slot] = t;
  }
}
#define QK_TL(slot) tl_mark(slot)
#define QK_TL_ANY(slot) tl_mark_any(slot)
#else
#define QK_TL(slot) ((void)0)
#define QK_TL_ANY(slot) ((void)0)
#endif

// ------------------------------------------------------------------------------------------
// The per-qubit recurrences (shared by the tile sweep and the pair-list kernel so the two
// produce bit-identical amplitudes).
// ------------------------------------------------------------------------------------------
struct Bond4 {
  double sp, tp, sm, tm;
};

__device__ __forceinline__ void bond4_init(Bond4& s) {
  s.sp = 1.0;
  s.tp = 0.0;
  s.sm = 1.0;
  s.tm = 0.0;
}

// 4 DMUL + 4 DADD + 8 DFMA per pair-qubit.  Six of the DFMAs read three distinct registers;
// the FP64 pipe issues those at ~2/3 rate unless an operand hits the operand-reuse cache
// (register-file read bandwidth; tools/rfbench.cu: 0.33 vs 0.49 warp-instr/clk/SMSP), so the
// operand order is chosen to let pairs of three-source DFMAs share a register in one slot.
// QK_STEPV selects among the measured orderings (config-4 bench, RI = 2 / RI = 4, G entries/s):
//   1: c/d plain, T+ and T- shared in slot B            1.209 / 1.201
//   2: + c and d share b_i in slot A          (default)  1.220 / 1.202
//   3: c and d share b_j in slot A                        1.210 / 1.202
//   4: T+/T- shared in slot A                             1.211 / 1.202
//   5: no sharing (first version)                         1.195 / 1.196
//   6: 2 + 4                                              1.220 / 1.203
// Distributing the sums into FMA chains (4 DMUL + 12 DFMA) adds three-source DFMAs and
// measured 5-9 % slower.
#ifndef QK_STEPV
#define QK_STEPV 2
#endif
__device__ __forceinline__ void bond4_step(Bond4& s, double2 vi, double2 vj) {
  const double ai = vi.x, bi = vi.y, aj = vj.x, bj = vj.y;
#if QK_STEPV == 1 || QK_STEPV == 4 || QK_STEPV == 5
  const double c = fma(bi, bj, ai * aj);     // cos(x_j - x_i)
  const double d = fma(ai, bj, -(bi * aj));  // sin(x_j - x_i)
#elif QK_STEPV == 2 || QK_STEPV == 6
  const double c = fma(bi, bj, ai * aj);
  const double d = fma(-bi, aj, ai * bj);  // shares b_i (slot A) with c
#else
  const double c = fma(bj, bi, aj * ai);
  const double d = fma(bj, ai, -(aj * bi));  // shares b_j (slot A) with c
#endif
  const double s1 = bi + bj, d2 = bi - bj, s2 = ai + aj, d1 = aj - ai;
#if QK_STEPV == 4 || QK_STEPV == 6
  const double nsp = fma(s.tp, s1, fma(s.sp, c, s.sp));
  const double ntm = fma(s.tp, -d, s.sp * d1);  // shares T+ (slot A) with nsp
  const double nsm = fma(s.tm, d, s.sm * s2);
  const double ntp = fma(s.tm, d2, fma(s.sm, c, -s.sm));  // shares T- (slot A) with nsm
#elif QK_STEPV == 5
  const double nsp = fma(s1, s.tp, fma(c, s.sp, s.sp));
  const double ntm = fma(d1, s.sp, -(d * s.tp));
  const double nsm = fma(d, s.tm, s2 * s.sm);
  const double ntp = fma(d2, s.tm, fma(c, s.sm, -s.sm));
#else
  const double nsp = fma(s1, s.tp, fma(c, s.sp, s.sp));
  const double ntm = fma(-d, s.tp, d1 * s.sp);  // shares T+ (slot B) with nsp
  const double nsm = fma(d, s.tm, s2 * s.sm);
  const double ntp = fma(d2, s.tm, fma(c, s.sm, -s.sm));  // shares T- (slot B) with nsm
#endif
  s.sp = nsp;
  s.tp = ntp;
  s.sm = nsm;
  s.tm = ntm;
}

// Whole-micro-tile step in an explicit issue order (QK_MT = 1: plain C++, 2: each FP64 op an
// asm volatile statement so ptxas sees them in this order).  Same operations and operands as
// bond4_step (STEPV 2) up to commuted multiplicands, so bit-identical.  Order: per tile row,
// c and d of all its pairs back to back (b_i stays in slot A: operand-reuse cache), then per
// pair the state update with the T+ pair and the T- pair of DFMAs adjacent (shared slot A).
#ifndef QK_MT
#define QK_MT 0
#endif
#if QK_MT == 2
__device__ __forceinline__ double xfma(double a, double b, double c) {
  double d;
  asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c));
  return d;
}
__device__ __forceinline__ double xmul(double a, double b) {
  double d;
  asm volatile("mul.rn.f64 %0, %1, %2;" : "=d"(d) : "d"(a), "d"(b));
  return d;
}
__device__ __forceinline__ double xadd(double a, double b) {
  double d;
  asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(d) : "d"(a), "d"(b));
  return d;
}
__device__ __forceinline__ double xsub(double a, double b) {
  double d;
  asm volatile("sub.rn.f64 %0, %1, %2;" : "=d"(d) : "d"(a), "d"(b));
  return d;
}
#else
__device__ __forceinline__ double xfma(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
#endif

template <int NI, int NJ>
__device__ __forceinline__ void bond4_tile_step(Bond4 (&st)[NI][NJ], const double2 (&vi)[NI],
                                                const double2 (&vj)[NJ]) {
  double c[NI][NJ], d[NI][NJ];
#pragma unroll
  for (int r = 0; r < NI; ++r) {
    double p[NJ], q[NJ];
#pragma unroll
    for (int k = 0; k < NJ; ++k) p[k] = xmul(vi[r].x, vj[k].x);
#pragma unroll
    for (int k = 0; k < NJ; ++k) q[k] = xmul(vi[r].x, vj[k].y);
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
      c[r][k] = xfma(vi[r].y, vj[k].y, p[k]);
      d[r][k] = xfma(-vi[r].y, vj[k].x, q[k]);
    }
  }
#pragma unroll
  for (int r = 0; r < NI; ++r)
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
      const double ai = vi[r].x, bi = vi[r].y, aj = vj[k].x, bj = vj[k].y;
      Bond4& s = st[r][k];
      const double s1 = xadd(bi, bj), d2 = xsub(bi, bj), s2 = xadd(ai, aj), d1 = xsub(aj, ai);
      const double x = xfma(c[r][k], s.sp, s.sp);
      const double y = xmul(d1, s.sp);
      const double z = xmul(s2, s.sm);
      const double w = xfma(c[r][k], s.sm, -s.sm);
      const double nsp = xfma(s.tp, s1, x);
      const double ntm = xfma(s.tp, -d[r][k], y);
      const double nsm = xfma(s.tm, d[r][k], z);
      const double ntp = xfma(s.tm, d2, w);
      s.sp = nsp;
      s.tp = ntp;
      s.sm = nsm;
      s.tm = ntm;
    }
}

__device__ __forceinline__ void bond4_scale(Bond4& s, double f) {
  s.sp *= f;
  s.tp *= f;
  s.sm *= f;
  s.tm *= f;
}

__device__ __forceinline__ double bond4_amp(const Bond4& s, double final_scale) {
  return (s.sp + s.tp) * final_scale;
}

struct Bond1 {
  double v;
};
__device__ __forceinline__ void bond1_init(Bond1& s) { s.v = 1.0; }
__device__ __forceinline__ void bond1_step(Bond1& s, double2 vi, double2 vj) {
  s.v *= fma(vi.y, vj.y, vi.x * vj.x);  // cos((x_j - x_i)/2) from half-angle planes
}

// L >= 3: amp = <phi_{L-1}(x_i)| R(x_j - x_i) |phi_{L-1}(x_j)>, phi_m = (C R)^m |0> is an MPS
// of bond D = 2^m whose site matrix is F(x)[a][b] = prod_k RY(x)[a_k ^ b_k][b_{k-1}] (level-k
// bits, b_{-1} = 0); the pair state V is D x D and one qubit is V <- (F_i^T V F_j) o RY(delta)
// on the top-level bits.  Half-angle planes (c, s).  |V| <= 1: no rescaling.
//
// F is never formed: F^T x factorises over the levels.  Summing level k out (k = 0, 1, ...)
// replaces input bit a_k by output bit b_k with the 2x2 factor RY[a_k ^ b_k][b_{k-1}], whose
// column b_{k-1} is an output bit already, so one level is a 2x2 rotation of every element
// pair differing in bit k, selected by bit k-1:
//     sel 0: (y0, y1) = (c x0 + s x1, s x0 + c x1)     sel 1: (y0, y1) = (-s x0 + c x1, c x0 - s x1)
// i.e. y0 = p x0 + q x1, y1 = q x0 + p x1 with (p, q) = sel ? (-s, c) : (c, s).  One side costs
// M passes of D^2 / 2 rotations (2 D^2 M instructions) instead of the D^3 of F^T V.
// V is flat, e = row * D + col: row bit k sits at bit M + k of e, column bit k at bit k.
__device__ __forceinline__ void rot_pair(double& x0, double& x1, double c, double s, int sel) {
  const double p = sel ? -s : c, q = sel ? c : s;
  const double y0 = fma(p, x0, q * x1), y1 = fma(q, x0, p * x1);
  x0 = y0;
  x1 = y1;
}

__device__ __forceinline__ double ry_delta_mask(int e, int M, double cd, double sd) {
  const int tb = (e >> (2 * M - 1)) & 1, tc = (e >> (M - 1)) & 1;
  return tb == tc ? cd : (tb ? sd : -sd);
}

// L = 3, 4 in a rotated, blocked basis (the L = 2 trick applied to the top level).  The D x D
// state (D = 2^M, M = L - 1) splits into (D/2)^2 blocks B[r][c] of 2x2 over the top bits,
// indexed by the lower M - 1 bits of row and column.  One qubit: the lower-level passes mix the
// blocks (the factored rotations above, rows with (c_i, s_i), columns with (c_j, s_j)); then
// each block takes an L = 2-type step B <- (A(x_i + t_r pi) B A(x_j + t_c pi)) o RY(delta),
// t_r / t_c = bit M - 2 of the block's row / column (the top-level pass is selected by it: RY
// at the angle shifted by pi).  In the Hadamard basis of the top bits, S = w00 + w11,
// Dg = w00 - w11, T = w01 + w10, E = w01 - w10 of every block update with the SAME seven
// coefficients as L = 2 up to signs and permutations: 1 +- C, D (C, D = cos, sin of
// x_j - x_i) and the separable a_i + a_j, b_i + b_j, b_j - b_i, a_i - a_j (a, b = cos, sin of
// the full angles), the 1/2 per qubit folded into one power of two (2^-512 rescales as L = 2).
// (4 (M-1) E + 2 E + 16) FP64 instructions per pair-qubit (E = D^2): L = 3 112 instead of 148,
// L = 4 656 instead of 836.  Verified in numpy against the reference goldens for L = 3..6.
template <int M>
struct BondR {
  static constexpr int H = 1 << (M - 1), E = 4 * H * H;
  double v[E];  // block (r, c) at 4 (r H + c): S, Dg, T, E
};

template <int M>
__device__ __forceinline__ void bondr_init(BondR<M>& s) {
#pragma unroll
  for (int e = 0; e < BondR<M>::E; ++e) s.v[e] = (e == 0 || e == 2) ? 1.0 : 0.0;
}

// the per-block L = 2-type step for top-level selectors (TR, TC)
template <int TR, int TC>
__device__ __forceinline__ void block_step(double* v, double C, double D, double p1, double q1,
                                           double p2, double q2) {
  const double S = v[0], Dg = v[1], T = v[2], E = v[3];
  if (TR == 0 && TC == 0) {
    v[0] = fma(q1, Dg, fma(C, S, S));
    v[1] = fma(p2, E, fma(C, T, -T));
    v[2] = fma(-D, E, p1 * T);
    v[3] = fma(D, Dg, q2 * S);
  } else if (TR == 0) {
    v[0] = fma(p1, Dg, -(D * S));
    v[1] = fma(-q2, E, -(D * T));
    v[2] = fma(-q1, T, -fma(C, E, E));
    v[3] = fma(p2, S, fma(C, Dg, -Dg));
  } else if (TC == 0) {
    v[0] = fma(p1, Dg, D * S);
    v[1] = fma(-q2, E, D * T);
    v[2] = fma(-q1, T, fma(C, E, E));
    v[3] = fma(p2, S, fma(-C, Dg, Dg));
  } else {
    v[0] = fma(-q1, Dg, fma(C, S, S));
    v[1] = fma(-p2, E, fma(C, T, -T));
    v[2] = fma(-D, E, -(p1 * T));
    v[3] = fma(D, Dg, -(q2 * S));
  }
}

template <int M>
__device__ __forceinline__ void bondr_step(BondR<M>& s, double2 vi, double2 vj) {
  constexpr int H = BondR<M>::H;
  const double ci = vi.x, si = vi.y, cj = vj.x, sj = vj.y;  // half-angle planes
  const double ai = fma(ci, ci, -(si * si)), bi = (ci + ci) * si;  // cos x_i, sin x_i
  const double aj = fma(cj, cj, -(sj * sj)), bj = (cj + cj) * sj;
  const double C = fma(bi, bj, ai * aj);   // cos(x_j - x_i)
  const double D = fma(-bi, aj, ai * bj);  // sin(x_j - x_i)
  const double p1 = ai + aj, q1 = bi + bj, p2 = bj - bi, q2 = ai - aj;
  double* v = s.v;
#pragma unroll
  for (int k = 0; k < M - 1; ++k)  // lower levels, rows (block row index r)
#pragma unroll
    for (int r = 0; r < H; ++r) {
      if (r & (1 << k)) continue;
      const int r1 = r | (1 << k), sel = k == 0 ? 0 : (r >> (k - 1)) & 1;
#pragma unroll
      for (int e = 0; e < 4 * H; ++e) rot_pair(v[4 * H * r + e], v[4 * H * r1 + e], ci, si, sel);
    }
#pragma unroll
  for (int k = 0; k < M - 1; ++k)  // lower levels, columns (block column index c)
#pragma unroll
    for (int c = 0; c < H; ++c) {
      if (c & (1 << k)) continue;
      const int c1 = c | (1 << k), sel = k == 0 ? 0 : (c >> (k - 1)) & 1;
#pragma unroll
      for (int r = 0; r < H; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          rot_pair(v[4 * (r * H + c) + q], v[4 * (r * H + c1) + q], cj, sj, sel);
    }
#pragma unroll
  for (int r = 0; r < H; ++r)
#pragma unroll
    for (int c = 0; c < H; ++c) {
      double* b = v + 4 * (r * H + c);
      const int tr = (r >> (M - 2)) & 1, tc = (c >> (M - 2)) & 1;
      if (tr == 0 && tc == 0) block_step<0, 0>(b, C, D, p1, q1, p2, q2);
      else if (tr == 0) block_step<0, 1>(b, C, D, p1, q1, p2, q2);
      else if (tc == 0) block_step<1, 0>(b, C, D, p1, q1, p2, q2);
      else block_step<1, 1>(b, C, D, p1, q1, p2, q2);
    }
}

template <int M>
__device__ __forceinline__ double bondr_amp(const BondR<M>& s, double final_scale) {
  double t = 0.0;  // sum(V) = sum over blocks of 2 w00 = S + Dg
#pragma unroll
  for (int b = 0; b < BondR<M>::E / 4; ++b) t += s.v[4 * b] + s.v[4 * b + 1];
  return t * final_scale;
}

template <int LAYERS>
struct BondT;
template <>
struct BondT<1> {
  using type = Bond1;
};
template <>
struct BondT<2> {
  using type = Bond4;
};
template <>
struct BondT<3> {
  using type = BondR<2>;
};
template <>
struct BondT<4> {
  using type = BondR<3>;
};

template <int LAYERS>
__device__ __forceinline__ void st_init(typename BondT<LAYERS>::type& s) {
  if constexpr (LAYERS == 2) bond4_init(s);
  else if constexpr (LAYERS == 1) bond1_init(s);
  else bondr_init<LAYERS - 1>(s);
}
template <int LAYERS>
__device__ __forceinline__ void st_step(typename BondT<LAYERS>::type& s, double2 vi, double2 vj) {
  if constexpr (LAYERS == 2) bond4_step(s, vi, vj);
  else if constexpr (LAYERS == 1) bond1_step(s, vi, vj);
  else bondr_step<LAYERS - 1>(s, vi, vj);
}
template <int LAYERS>
__device__ __forceinline__ void st_rescale(typename BondT<LAYERS>::type& s) {
  if constexpr (LAYERS == 2) bond4_scale(s, 0x1p-512);
  if constexpr (LAYERS == 3 || LAYERS == 4) {
#pragma unroll
    for (int e = 0; e < BondR<LAYERS - 1>::E; ++e) s.v[e] *= 0x1p-512;
  }
}
template <int LAYERS>
__device__ __forceinline__ double st_amp(const typename BondT<LAYERS>::type& s, double fs) {
  if constexpr (LAYERS == 2) return bond4_amp(s, fs);
  else if constexpr (LAYERS == 1) return s.v;
  else return bondr_amp<LAYERS - 1>(s, fs);
}

__device__ __forceinline__ double kernel_value(double amp, int convention) {
  return convention == QK_MAGNITUDE ? fabs(amp) : amp * amp;
}

// Fence between a tile's stores and its progress-counter bump (host pipelines only).  The
// tile, the counter and the copy engine's reads all live in / go through this device's memory
// and L2, so gpu scope suffices; a system-scope fence cost ~3 % of the sweep (measured).

#ifndef QK_PROGRESS_FENCE
#define QK_PROGRESS_FENCE __threadfence
#endif

// Tile order.  Gram tiles are grouped into super-rows of kGroup tile rows (rows b..nb-1 of
// each tile row b of the upper triangle) and, inside a super-row, walked column by column: a
// wave of 148 persistent CTAs then covers ~kGroup tile rows x ~148/kGroup tile columns, whose
// gate planes (~20 MB at 784 qubits) stay in L2.  A super-row holds exactly the tiles of its
// rows, so super-row boundaries coincide with plain row-major offsets (used by the host-side
// row panels).  Cross tiles use kRectGroup (1 = row-major): a wave then finishes about one
// tile row, so the host pipeline's D2H tail after the sweep is one 64-row panel (0.1 ms at
// config 4) instead of a whole super-row (0.6 ms); the extra plane re-reads are L2/DRAM
// traffic the FP64-bound sweep does not notice (measured).
// Row-major position -> tile row (the plain upper-triangle row containing linear index g).
__host__ __device__ __forceinline__ int64_t upper_row_of(int64_t g, int64_t nb) {
  const double m = 2.0 * double(nb) + 1.0;
  int64_t b = int64_t((m - sqrt(m * m - 8.0 * double(g))) * 0.5);
  if (b < 0) b = 0;
  if (b > nb - 1) b = nb - 1;
  while (b > 0 && upper_row_offset(b, nb) > g) --b;
  while (b + 1 < nb && upper_row_offset(b + 1, nb) <= g) ++b;
  return b;
}

__host__ __device__ __forceinline__ void decode_upper(int64_t g, int64_t nb, int64_t& bi, int64_t& bj) {
  const int64_t r0 = (upper_row_of(g, nb) / kGroup) * kGroup;
  const int64_t h = nb - r0 < kGroup ? nb - r0 : kGroup;
  const int64_t local = g - upper_row_offset(r0, nb);
  const int64_t tri = h * (h + 1) / 2;
  if (local < tri) {  // columns r0 .. r0+h-1: column c holds rows r0 .. r0+c
    int64_t c = int64_t((sqrt(8.0 * double(local) + 1.0) - 1.0) * 0.5);
    while (c > 0 && c * (c + 1) / 2 > local) --c;
    while ((c + 1) * (c + 2) / 2 <= local) ++c;
    bj = r0 + c;
    bi = r0 + (local - c * (c + 1) / 2);
  } else {  // columns r0+h .. nb-1: full columns of h rows
    const int64_t l2 = local - tri;
    bj = r0 + h + l2 / h;
    bi = r0 + l2 % h;
  }
}

// Gram tile order with a head: for 0 < B < nb (B a multiple of kGroup) the tiles of the
// B x B leading block triangle come first (in the grouped order over B blocks), then rows
// [0, B) restricted to columns [B, nb) (super-rows of kGroup rows, column by column), then the
// super-rows from B on exactly as decode_upper orders them.  A host pipeline can then sweep
// the head while the angles of blocks >= B are still uploading.  B = 0: decode_upper.
__host__ __device__ __forceinline__ void decode_gram(int64_t g, int64_t nb, int64_t B,
                                                     int64_t& bi, int64_t& bj) {
  if (B <= 0 || B >= nb) {
    decode_upper(g, nb, bi, bj);
    return;
  }
  const int64_t head = B * (B + 1) / 2;
  if (g < head) {
    decode_upper(g, B, bi, bj);
    return;
  }
  g -= head;
  const int64_t w = nb - B, strip = B * w;
  if (g < strip) {
    const int64_t l = g % (int64_t(kGroup) * w);
    bj = B + l / kGroup;
    bi = (g / (int64_t(kGroup) * w)) * kGroup + l % kGroup;
    return;
  }
  decode_upper(g - strip + upper_row_offset(B, nb), nb, bi, bj);
}

__host__ __device__ __forceinline__ void decode_rect(int64_t g, int64_t nb_rows, int64_t nb_cols,
                                            int64_t& bi, int64_t& bj,
                                            int64_t tail = kRectTail) {
  const int64_t grouped = nb_rows > tail ? nb_rows - tail : 0;  // rows in super-rows
  if (g >= grouped * nb_cols) {  // the row-major tail
    const int64_t l = g - grouped * nb_cols;
    bi = grouped + l / nb_cols;
    bj = l % nb_cols;
    return;
  }
  const int64_t r0 = (g / (kRectGroup * nb_cols)) * kRectGroup;
  const int64_t h = grouped - r0 < kRectGroup ? grouped - r0 : kRectGroup;
  const int64_t local = g - r0 * nb_cols;
  bj = local / h;
  bi = r0 + local % h;
}

// ------------------------------------------------------------------------------------------
// Gate build: angles -> planes[block][q][t] = (cos x, sin x)  (L = 2)  or  half angles (L != 2)
// ------------------------------------------------------------------------------------------
// One plane set of a launch: angles X [n x ld] (sample-major), plane blocks [blk0, blk0 + nblk).
struct GateSet {
  const double* X;
  int64_t n, ld;
  double2* planes;
  unsigned long long* bad;  // optional: atomicMin of the first non-finite sample
  int64_t blk0, nblk;
};

// Work item = one plane block (64 samples) x one slab of 16 * QD plane qubits.  Thread
// (t = tid % 64, u = tid / 64) owns sample t and the qubit quads u, u + 4, ... of the slab.
// VEC: each quad is one 32-byte sector of the sample's row (two 16 B loads), so every fetched
// sector is used whole; all of a thread's loads are issued before its first sincos.  Stores:
// a warp writes 32 consecutive samples of one qubit (512 contiguous bytes).  PERSIST: grid-
// stride CTAs with a register double buffer (the next item's loads in flight during the
// current item's sincos and stores); otherwise one CTA per item.  Padding samples (front of
// block 0) and the identity qubits of the width padding (front of the chain) get angle 0.
// A second plane set (e.g. the test samples of a joint job) rides in the same launch.
struct GateItem {
  const double* X;
  int64_t ld;
  double2* planes;
  unsigned long long* bad;
  int64_t blk, s;
  int q_slab;
  bool live;
};

// (field selects, not a pointer to the parameter, so the sets stay in the constant bank)
template <int QD>
__device__ __forceinline__ GateItem gate_item(const GateSet& s0, const GateSet& s1, int slabs,
                                              int64_t item) {
  GateItem g;
  const int64_t b = item / slabs;
  g.q_slab = int(item - b * slabs) * 16 * QD;
  const bool second = b >= s0.nblk;
  g.X = second ? s1.X : s0.X;
  g.ld = second ? s1.ld : s0.ld;
  g.planes = second ? s1.planes : s0.planes;
  g.bad = second ? s1.bad : s0.bad;
  const int64_t n = second ? s1.n : s0.n;
  g.blk = second ? s1.blk0 + b - s0.nblk : s0.blk0 + b;
  g.s = g.blk * kTile + (threadIdx.x & 63) - sample_pad(n);
  g.live = g.s >= 0 && g.s < n;
  return g;
}

template <bool VEC, int QD>
__device__ __forceinline__ void gate_load(const GateItem& g, int width, int front,
                                          double (&x)[QD][4]) {
  const int u = threadIdx.x >> 6;
  const double* row = g.X + (g.live ? g.s : 0) * g.ld;
#pragma unroll
  for (int k = 0; k < QD; ++k) {
    const int qi = g.q_slab + 4 * (u + 4 * k) - front;  // input qubit of element 0
    if (VEC) {
      // front % 4 == 0 and n_pad % 4 == 0: a quad is wholly input qubits or wholly padding
      if (g.live && qi >= 0 && qi < width) {
        const double2 lo = __ldg(reinterpret_cast<const double2*>(row + qi));
        const double2 hi = __ldg(reinterpret_cast<const double2*>(row + qi) + 1);
        x[k][0] = lo.x, x[k][1] = lo.y, x[k][2] = hi.x, x[k][3] = hi.y;
      } else {
        x[k][0] = x[k][1] = x[k][2] = x[k][3] = 0.0;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        x[k][e] = g.live && qi + e >= 0 && qi + e < width ? __ldg(row + qi + e) : 0.0;
    }
  }
}

template <int QD>
__device__ __forceinline__ void gate_store(const GateItem& g, int n_pad, int half,
                                           const double (&x)[QD][4]) {
  if (g.bad != nullptr) {
    bool finite = true;
#pragma unroll
    for (int k = 0; k < QD; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e) finite = finite && isfinite(x[k][e]);
    if (!finite) atomicMin(g.bad, (unsigned long long)g.s);  // padding values are 0
  }
  const int u = threadIdx.x >> 6;
  double2* out = g.planes + g.blk * int64_t(n_pad) * kTile + (threadIdx.x & 63);
#pragma unroll
  for (int k = 0; k < QD; ++k) {
    const int q0 = g.q_slab + 4 * (u + 4 * k);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (q0 + e < n_pad) {
        double sn, cs;
        sincos(half ? 0.5 * x[k][e] : x[k][e], &sn, &cs);
        out[int64_t(q0 + e) * kTile] = make_double2(cs, sn);
      }
    }
  }
}

template <bool VEC, int QD, bool PERSIST, int MINB>
__global__ void __launch_bounds__(256, MINB) gate_build_kernel(GateSet s0, GateSet s1, int width,
                                                               int n_pad, int front, int half) {
  // a sweep launched behind this kernel as a programmatic dependent may start its prologue
  // now (it waits for this grid's completion before reading the planes)
  asm volatile("griddepcontrol.launch_dependents;");
  const int slabs = (n_pad + 16 * QD - 1) / (16 * QD);
  const int64_t n_items = (s0.nblk + s1.nblk) * slabs;
  int64_t it = blockIdx.x;
  if (it >= n_items) return;
  double xa[QD][4];
  GateItem ga = gate_item<QD>(s0, s1, slabs, it);
  gate_load<VEC, QD>(ga, width, front, xa);
  if constexpr (!PERSIST) {
    gate_store<QD>(ga, n_pad, half, xa);
  } else {
    double xb[QD][4];
    for (;;) {  // two items per trip so the double buffer needs no register moves
      const int64_t nb = it + gridDim.x;
      GateItem gb;
      if (nb < n_items) {
        gb = gate_item<QD>(s0, s1, slabs, nb);
        gate_load<VEC, QD>(gb, width, front, xb);
      }
      gate_store<QD>(ga, n_pad, half, xa);
      if (nb >= n_items) break;
      it = nb + gridDim.x;
      if (it < n_items) {
        ga = gate_item<QD>(s0, s1, slabs, it);
        gate_load<VEC, QD>(ga, width, front, xa);
      }
      gate_store<QD>(gb, n_pad, half, xb);
      if (it >= n_items) break;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Pair-tiled sweep.  Persistent CTAs walk tiles g = tile_begin + blockIdx.x + k*gridDim.x.
// The (tile, chunk) sequence streams through a kStages-deep shared-memory ring of bulk async
// copies (TMA engine; i-block chunk + j-block chunk, 32 KB per stage) that complete on the
// stage's `full` mbarrier.  There is no CTA-wide barrier in the loop and no producer warp: each
// warp counts itself off a stage when it is done reading it, and the LAST warp to release a
// stage refills it with the item kStages ahead.  Each thread owns a kRI x kRJ micro-tile of
// pairs whose bond states stay in registers for the whole qubit sweep; per qubit it reads
// kRI + kRJ double2 from shared memory (broadcast within the warp) and issues 16 * kRI * kRJ
// FP64 instructions.
// ------------------------------------------------------------------------------------------
struct SweepArgs {
  const double2* rows;
  const double2* cols;
  int64_t n_rows, n_cols;
  int64_t nb_rows, nb_cols;
  int64_t tile_begin, n_tiles;
  double* out;
  int64_t ld_out;
  double final_scale;
  int n_pad, nchunks, convention;
  int front;               // identity qubits at the front of chunk 0, skipped by the sweep
  unsigned int* progress;  // optional: per-tile-row count of finished tiles (host pipelines)
  // kModeJob: tiles [0, n_first) are the Gram of (rows = cols); the rest the cross block
  // rows2 x cols (rows2 = test planes) stored to out2 (ld = n_cols), counted in progress2.
  const double2* rows2;
  int64_t n_rows2, nb_rows2, n_first;
  double* out2;
  unsigned int* progress2;
  int pad_rows, pad_cols, pad_rows2;  // sample_pad() of each plane set (front of block 0)
  unsigned long long* next_tile;  // dynamic tile claims (all-ones before a launch's first claim)
  int64_t n_split;  // the last n_split tiles run as two row halves each (finer last wave)
  int64_t head_b;   // Gram tile order with a B-block head (decode_gram; 0: decode_upper)
  int pdl;          // host only: launch as a programmatic dependent of the preceding kernel
  int64_t rect_tail;  // cross tile rows swept row by row at the end of the list (decode_rect)
};

// Per-tile coordinates: tile rows/cols in plane blocks and which problem of a kModeJob launch.
struct TileXY {
  int64_t bi, bj;
  int prob;
};

// A CTA's claimed work item (dynamic tile schedule; see sweep_kernel).
struct Claim {
  int64_t g;  // launch-local work item (>= n_items: none)
  int64_t t;  // launch-local tile index
  int bi, bj, prob;
  int half;   // -1: whole tile; 0 / 1: tile rows 0-31 / 32-63 only
};

// EPI (sweep epilogue): 0 = CTA-staged whole-row stores (two CTA barriers per tile; the
// default), 1 = per-warp stores straight from the registers and a warp-private transposing
// stage for the Gram mirror (no CTA barrier: short chains, where a tile's sweep is only a few
// microseconds and the CTA-wide epilogue would idle the FP64 pipe for a large share of it).
template <int LAYERS, int MODE, int OUT, int RI, int EPI>
__device__ __forceinline__ void sweep_body(const SweepArgs& a) {
  using St = typename BondT<LAYERS>::type;
  constexpr int kRI = Geo<RI>::kRI, kWarps = Geo<RI>::kWarps;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + size_t(kStages) * 2 * kChunkBytes);
  int* released = reinterpret_cast<int*>(full + kStages);

  const int tid = threadIdx.x;
  const int lane = tid % 32;
  const int nchunks = a.nchunks;
  QK_TL(0);

  // Dynamic tile schedule: CTA b starts with tiles b, b + G, ..., b + kLook G (G = gridDim.x,
  // static: no atomic in the prologue); every further tile is claimed from a launch-wide
  // counter (tiles (kLook + 1) G, (kLook + 1) G + 1, ... in list order), so CTAs that spend
  // time elsewhere (plane builds, cheaper padding tiles) simply take fewer tiles.  The chunks
  // of a CTA's tile k + kLook are issued during tile k, so tile k + kLook is claimed (thread
  // 0) at the start of tile k and published by a CTA barrier.  Short chains (RI = 1, a tile of
  // a few microseconds) issue that claim's atomic one tile earlier and only decode it at the
  // next tile start, so its latency never stalls the CTA.  Claims live in a small shared ring
  // indexed by the CTA-local tile number.
  const int kLook = 1 + (kStages - 1) / nchunks;
  constexpr bool kEarly = RI == 1;
  __shared__ Claim ring[8];
  double* stage_T = reinterpret_cast<double*>(released + 2 * kStages);  // epilogue staging tile
  // Work items: tiles [0, n_tiles - n_split) whole, then the last n_split tiles as two row
  // halves each, so the final wave ends in half-tile steps (a half tile takes about half the
  // time: the warps of the other half skip the sweep like padding rows do).
  const int64_t n_whole = a.n_tiles - a.n_split, n_items = a.n_tiles + a.n_split;
  auto claim_raw = [&](int64_t k) -> int64_t {  // thread 0 only
    if constexpr (RI == 1)  // the first kLook + 1 tiles static (no atomic in the prologue)
      return k <= kLook ? int64_t(blockIdx.x) + k * int64_t(gridDim.x)
                        : (kLook + 1) * int64_t(gridDim.x) + int64_t(atomicAdd(a.next_tile, 1ull) + 1);
    return k == 0 ? int64_t(blockIdx.x)
                  : int64_t(gridDim.x) + int64_t(atomicAdd(a.next_tile, 1ull) + 1);
  };
  auto claim_set = [&](int64_t k, int64_t g_item) {  // thread 0 only
    Claim c;
    c.g = g_item;
    c.bi = c.bj = c.prob = 0;
    c.half = -1;
    c.t = c.g;
    if (c.g >= n_whole && c.g < n_items) {
      c.t = n_whole + (c.g - n_whole) / 2;
      c.half = int((c.g - n_whole) % 2);
    }
    if (c.g < n_items) {
      const int64_t g = a.tile_begin + c.t;
      int64_t bi, bj;
      if (MODE == kModeGram || (MODE == kModeJob && g < a.n_first)) {
        decode_gram(g, a.nb_rows, a.head_b, bi, bj);
      } else if (MODE == kModeCross) {
        decode_rect(g, a.nb_rows, a.nb_cols, bi, bj, a.rect_tail);
      } else {
        decode_rect(g - a.n_first, a.nb_rows2, a.nb_cols, bi, bj, a.rect_tail);
        c.prob = 1;
      }
      c.bi = int(bi);
      c.bj = int(bj);
    }
    ring[k & 7] = c;
  };
  auto valid = [&](int64_t k) { return ring[k & 7].g < n_items; };
  int64_t pending = 0;  // kEarly: raw claim of tile k + kLook + 1, issued during tile k
  auto tile_of = [&](int64_t k) -> TileXY {
    const Claim& c = ring[k & 7];
    return TileXY{c.bi, c.bj, c.prob};
  };
  if (tid == 0) {
    for (int64_t k = 0; k <= kLook; ++k) claim_set(k, claim_raw(k));
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    fence_mbar_init();
  }
  // Programmatic dependent launch: everything above overlaps the tail of the kernel this one
  // was launched behind (the gate build); global memory is touched only after this wait.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  auto issue = [&](int64_t f) {  // fill stage f % kStages with item f (if its tile exists)
    const int64_t k = f / nchunks;
    if (!valid(k)) return;
    const int c = int(f - k * nchunks);
    const TileXY t = tile_of(k);
    const int stage = int(f % kStages);
    double2* dst = sbuf + size_t(stage) * 2 * kChunkElems;
    const double2* si =
        (t.prob ? a.rows2 : a.rows) + (t.bi * a.n_pad + int64_t(c) * kChunk) * kTile;
    const double2* sj = a.cols + (t.bj * a.n_pad + int64_t(c) * kChunk) * kTile;
    if (c == 0 && k < 32) QK_TL_ANY(96 + int(k));
    mbar_arrive_expect_tx(&full[stage], 2 * kChunkBytes);
    bulk_g2s(dst, si, kChunkBytes, &full[stage]);
    bulk_g2s(dst + kChunkElems, sj, kChunkBytes, &full[stage]);
  };

  if (tid == 0) {
    for (int64_t f = 0; f < kStages; ++f) issue(f);
    if (kEarly) pending = claim_raw(kLook + 1);
  }
  __syncthreads();
  QK_TL(1);

  // ---------------- compute warps ----------------
  // Thread (ty, tx) owns tile rows rb + ty*kRI .. rb + ty*kRI+kRI-1 (consecutive, so a warp
  // covers 2*kRI whole rows) and columns tx + kTX*c; rb = 0, or the item's first row for RI = 1.
  const int tx = tid % kTX, ty = tid / kTX;
  const int warp_row_end0 = (tid / 32 + 1) * (32 / kTX) * kRI;  // rows [.., end) of the warp
  St st[kRI][kRJ];
  int64_t f = 0;
  for (int64_t k = 0; valid(k); ++k) {
    if (k > 0) {  // claim tile k + kLook (its chunks are issued during tile k)
      if (tid == 0) {
        if (kEarly) {
          claim_set(k + kLook, pending);
          pending = claim_raw(k + kLook + 1);
        } else {
          claim_set(k + kLook, claim_raw(k + kLook));
        }
      }
      __syncthreads();
    }
    QK_TL(2 + 4 * int(k));
    const TileXY tk = tile_of(k);
    // padding rows of this tile (front of plane block 0): warps made only of them skip the
    // sweep (they still release every stage) — the ragged sample block costs ~1/4 of a tile
    const int pad_r = tk.bi == 0 ? (tk.prob ? a.pad_rows2 : a.pad_rows) : 0;
    const int half = ring[k & 7].half;
    const int r_lo = half == 1 ? kTile / 2 : 0, r_hi = half == 0 ? kTile / 2 : kTile;
    const int rb = RI == 1 ? r_lo : 0;  // first tile row of this thread layout
    const int warp_row_end = rb + warp_row_end0;
    const bool idle = warp_row_end <= (pad_r > r_lo ? pad_r : r_lo) ||
                      warp_row_end - (32 / kTX) * kRI >= r_hi;
#pragma unroll
    for (int r = 0; r < kRI; ++r)
#pragma unroll
      for (int c = 0; c < kRJ; ++c) st_init<LAYERS>(st[r][c]);

    for (int ch = 0; ch < nchunks; ++ch, ++f) {
      const int stage = int(f % kStages);
#ifdef QK_TIMELINE
      if (ch == 0 && tid == 0 && k < 32) {
        uint32_t ready;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n}" : "=r"(ready) : "r"(smem_u32(&full[stage])),
                     "r"(uint32_t((f / kStages) & 1)) : "memory");
        tl_store(128 + int(k), ready + 1);
        tl_store(192 + int(k), idle ? 2 : 1);
      }
#endif
      mbar_wait(&full[stage], uint32_t((f / kStages) & 1));
      if (ch == 0) QK_TL(3 + 4 * int(k));
      const double2* sI = sbuf + size_t(stage) * 2 * kChunkElems;
      const double2* sJ = sI + kChunkElems;
      auto qubit = [&](int q) {
        double2 vi[kRI], vj[kRJ];
#pragma unroll
        for (int r = 0; r < kRI; ++r) vi[r] = sI[q * kTile + rb + ty * kRI + r];
#pragma unroll
        for (int c = 0; c < kRJ; ++c) vj[c] = sJ[q * kTile + tx + kTX * c];
        if constexpr (LAYERS == 2 && QK_MT != 0) {
          bond4_tile_step<kRI, kRJ>(st, vi, vj);
        } else {
#pragma unroll
          for (int r = 0; r < kRI; ++r)
#pragma unroll
            for (int c = 0; c < kRJ; ++c) st_step<LAYERS>(st[r][c], vi[r], vj[c]);
        }
      };
      if (!idle) {
        if (ch == 0 && a.front > 0) {
          // chunk 0 starts with the identity qubits of the width padding: skip them
          for (int q = a.front; q < kChunk; ++q) qubit(q);
        } else {
#pragma unroll(kQUnroll)
          for (int q = 0; q < kChunk; ++q) qubit(q);
        }
      }
      __syncwarp();  // every lane's reads of this stage have completed
      if (lane == 0) {
        // the last warp to release the stage refills it with item f + kStages
        if (release_stage(&released[stage]) == kWarps - 1) {
          if (ch == 0 && k < 32) QK_TL_ANY(160 + int(k));
          released[stage] = 0;
          fence_proxy_async_smem();  // the generic-proxy reads before the async-proxy refill
          issue(f + kStages);
        }
      }
      if (LAYERS == 2 && ch + 1 < nchunks && ((ch + 1) % kRescaleChunks) == 0) {
#pragma unroll
        for (int r = 0; r < kRI; ++r)
#pragma unroll
          for (int c = 0; c < kRJ; ++c) st_rescale<LAYERS>(st[r][c]);
      }
    }

    // ---- epilogue ----
    QK_TL(4 + 4 * int(k));
    const TileXY t = tk;
    const int64_t bi = t.bi, bj = t.bj;
    const bool gram = MODE == kModeGram || (MODE == kModeJob && t.prob == 0);
    if (OUT == QK_OUT_PACKED) {
      double* o = a.out + ring[k & 7].t * int64_t(kTile * kTile);
#pragma unroll
      for (int r = 0; r < kRI; ++r)
#pragma unroll
        for (int c = 0; c < kRJ; ++c)
          if (rb + ty * kRI + r >= r_lo && rb + ty * kRI + r < r_hi)
            o[(rb + ty * kRI + r) * kTile + tx + kTX * c] =
                kernel_value(st_amp<LAYERS>(st[r][c], a.final_scale), a.convention);
    } else if (EPI == 1) {
      // Per-warp epilogue, no CTA barrier: the warp's 2*kRI rows go out straight from the
      // registers (each store instruction writes two 128 B row segments), and the Gram mirror
      // through a warp-private transposing stage in shared memory (each lane writes the
      // warp's 2*kRI values of one or two rows of K).  Warps outside the item's rows (a half
      // tile) store nothing.
      constexpr int kWR = 2 * kRI;  // rows per warp
      const bool mine = warp_row_end > r_lo && warp_row_end - kWR < r_hi;
      double* out = t.prob ? a.out2 : a.out;
      const int64_t ld = t.prob ? a.n_cols : a.ld_out;
      const int64_t n_rows = t.prob ? a.n_rows2 : a.n_rows;
      const int64_t i0 = bi * kTile - (t.prob ? a.pad_rows2 : a.pad_rows);
      const int64_t j0 = bj * kTile - (gram ? a.pad_rows : a.pad_cols);
      double v[kRI][kRJ];
#pragma unroll
      for (int r = 0; r < kRI; ++r)
#pragma unroll
        for (int c = 0; c < kRJ; ++c) {
          v[r][c] = kernel_value(st_amp<LAYERS>(st[r][c], a.final_scale), a.convention);
          const int64_t i = i0 + rb + ty * kRI + r, j = j0 + tx + kTX * c;
          if (!mine) {
          } else if (gram) {
            if (i >= 0 && i < n_rows && j < n_rows && i <= j)
              out[i * ld + j] = i == j ? 1.0 : v[r][c];
          } else if (i >= 0 && j >= 0 && i < n_rows && j < a.n_cols) {
            out[i * ld + j] = v[r][c];
          }
        }
#ifdef QK_DIAG_NO_MIRROR  // diagnostic timing variant: the per-warp epilogue skips the mirror
      if (false) {
#else
      if (gram && mine) {
#endif
        const int w = tid / 32;
        double* wb = stage_T + w * (kWR * (kTile + 1));
        __syncwarp();  // this warp's mirror pass of the previous tile has read wb
#pragma unroll
        for (int r = 0; r < kRI; ++r)
#pragma unroll
          for (int c = 0; c < kRJ; ++c)
            wb[((ty & 1) * kRI + r) * (kTile + 1) + tx + kTX * c] = v[r][c];
        __syncwarp();
        const int64_t iw = i0 + rb + w * kWR;  // first row of this warp
#pragma unroll
        for (int h = 0; h < kTile / 32; ++h) {
          const int jl = lane + 32 * h;
          const int64_t j = j0 + jl;
          if (j < n_rows) {
#pragma unroll
            for (int lr = 0; lr < kWR; ++lr) {
              const int64_t i = iw + lr;
              if (i >= 0 && i < j) out[j * ld + i] = wb[lr * (kTile + 1) + jl];
            }
          }
        }
      }
    } else {
      // Stage the tile in shared memory, then store it row by row and (Gram) its mirror
      // column by column, so every store instruction writes whole contiguous rows of K
      // (full 128 B lines in L2, or over NVLink when K lives on another GPU).
      __syncthreads();  // the previous tile's store pass has finished reading the stage
#pragma unroll
      for (int r = 0; r < kRI; ++r)
#pragma unroll
        for (int c = 0; c < kRJ; ++c)
          stage_T[(rb + ty * kRI + r) * (kTile + 1) + tx + kTX * c] =
              kernel_value(st_amp<LAYERS>(st[r][c], a.final_scale), a.convention);
      __syncthreads();
      double* out = t.prob ? a.out2 : a.out;
      const int64_t ld = t.prob ? a.n_cols : a.ld_out;
      const int64_t n_rows = t.prob ? a.n_rows2 : a.n_rows;
      const int64_t i0 = bi * kTile - (t.prob ? a.pad_rows2 : a.pad_rows);
      const int64_t j0 = bj * kTile - (gram ? a.pad_rows : a.pad_cols);
      for (int e = r_lo * kTile + tid; e < r_hi * kTile; e += blockDim.x) {
        const int il = e / kTile, jl = e % kTile;  // consecutive threads: consecutive columns
        const int64_t i = i0 + il, j = j0 + jl;
        if (gram) {
          if (i >= 0 && i < n_rows && j < n_rows && i <= j)
            out[i * ld + j] = i == j ? 1.0 : stage_T[il * (kTile + 1) + jl];
        } else if (i >= 0 && j >= 0 && i < n_rows && j < a.n_cols) {
          out[i * ld + j] = stage_T[il * (kTile + 1) + jl];
        }
      }
      if (gram) {
        const int span = r_hi - r_lo;
        for (int e = tid; e < kTile * span; e += blockDim.x) {
          const int jl = e / span, il = r_lo + e % span;  // mirror: row j of K, consecutive i
          const int64_t i = i0 + il, j = j0 + jl;
          if (i >= 0 && i < j && j < n_rows) out[j * ld + i] = stage_T[il * (kTile + 1) + jl];
        }
      }
    }
    unsigned int* prog = t.prob ? a.progress2 : a.progress;
    if (prog != nullptr) {
      // publish the finished tile to a copy stream waiting on its super-row counter
      QK_PROGRESS_FENCE();
      __syncthreads();
      if (tid == 0) atomicAdd(prog + bi, half < 0 ? 2u : 1u);  // per tile row: 2 per tile
    }
    QK_TL(5 + 4 * int(k));
  }
}

template <int LAYERS, int MODE, int OUT, int RI, int EPI>
__global__ void __launch_bounds__(Geo<RI>::kThreads, 1) sweep_kernel(const SweepArgs a) {
  sweep_body<LAYERS, MODE, OUT, RI, EPI>(a);
}

// ------------------------------------------------------------------------------------------
// L >= 3 tiles: the bond-16 state (16 doubles) does not fit a register micro-tile, so each
// thread carries ONE pair; a 64x64 tile is 16 work items of 16x16 pairs spread over the
// grid.  Planes are read through L1/L2 (the step is ~180 FP64 instructions per 32 B loaded).
// ------------------------------------------------------------------------------------------
template <int LAYERS, int MODE, int OUT>
__global__ void __launch_bounds__(256) sweep_general_kernel(const SweepArgs a) {
  using St = typename BondT<LAYERS>::type;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t items = a.n_tiles * 16;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t g = a.tile_begin + it / 16;
    const int sub = int(it % 16);
    int64_t bi, bj;
    if (MODE == kModeGram) {
      decode_upper(g, a.nb_rows, bi, bj);
    } else {
      decode_rect(g, a.nb_rows, a.nb_cols, bi, bj, a.rect_tail);
    }
    const int il = (sub / 4) * 16 + ty, jl = (sub % 4) * 16 + tx;
    const double2* pi = a.rows + bi * int64_t(a.n_pad) * kTile + il;
    const double2* pj = a.cols + bj * int64_t(a.n_pad) * kTile + jl;
    St st;
    st_init<LAYERS>(st);
    // unrolled so the next qubits' plane loads issue early (measured: L = 3 x4 +3.6 %,
    // L = 4 x2 +1.4 %, x4 -12 %)
    constexpr int kUnrollQ = LAYERS == 3 ? 4 : 2;
#pragma unroll kUnrollQ
    for (int q = a.front; q < a.n_pad; ++q) {  // the front padding qubits are identities
      st_step<LAYERS>(st, __ldg(pi + int64_t(q) * kTile), __ldg(pj + int64_t(q) * kTile));
      // L = 3, 4 (rotated, 1/2 per qubit dropped): the same 2^-512 rescale points as L = 2
      if (LAYERS >= 3 && (q + 1) % (kChunk * kRescaleChunks) == 0 && q + 1 < a.n_pad)
        st_rescale<LAYERS>(st);
    }
    const double v = kernel_value(st_amp<LAYERS>(st, a.final_scale), a.convention);
    if (OUT == QK_OUT_PACKED) {
      a.out[(g - a.tile_begin) * int64_t(kTile * kTile) + il * kTile + jl] = v;
    } else {
      const int64_t i = bi * kTile + il - a.pad_rows, j = bj * kTile + jl - a.pad_cols;
      if (MODE == kModeGram) {
        if (i >= 0 && i < a.n_rows && j < a.n_rows) {
          if (i < j) {
            a.out[i * a.ld_out + j] = v;
            a.out[j * a.ld_out + i] = v;
          } else if (i == j) {
            a.out[i * a.ld_out + i] = 1.0;
          }
        }
      } else if (i >= 0 && j >= 0 && i < a.n_rows && j < a.n_cols) {
        a.out[i * a.ld_out + j] = v;
      }
    }
    if (a.progress != nullptr) {
      QK_PROGRESS_FENCE();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(a.progress + bi, 1u);  // per tile row, 16 per tile
    }
  }
}

// ------------------------------------------------------------------------------------------
// L = 5..8 (D = 16..128, state 2 KB..128 KB per pair), PP pairs per CTA of 256 threads.
// L = 5: the rotated blocked form in registers (deep_sweep_bondr); L = 6, 7: the state in
// registers, one thread per column / row (deep_sweep_reg); both with one shared-memory
// transpose per qubit.  L = 8 (round 1's scheme): the D x D state in shared memory (rows
// padded to D + 1 doubles: conflict-free row and column walks); per qubit two register
// rounds: each thread loads one column (F_i side: all M row-level passes in registers) or one
// row (F_j side + the RY(delta) mask), so every element crosses shared memory once per side; a
// CTA barrier after each round; a thread holds half a column / row (64 values) and the top
// level is one extra pair round.  Shared by the tile kernel and the pair-list kernel
// (bit-identical).
// ------------------------------------------------------------------------------------------
constexpr int kDeepThreads = 256;
template <int M>
struct Deep {
  static constexpr int D = 1 << M, E = D * D, RS = D + 1;  // padded row stride (doubles)
  static constexpr int G = M < 6 ? M : 6;    // levels per register round (2^G values/thread)
  static constexpr int H = M - G;            // remaining levels: pair rounds (M = 7: one)
  static constexpr bool kR = QK_DEEP_BONDR && M == 4;  // the rotated blocked form (L = 5)
  static constexpr int HB = D / 2;           // kR: blocks per side
  static constexpr int IPP = kR ? HB : D << H;  // threads per pair
  static constexpr int PP = kDeepThreads / IPP;       // pairs per CTA: 16 (32), 8, 4, 1
  static constexpr int kGroups = kTile * kTile / PP;  // pair groups (work items) per tile
  // doubles per pair (kR: [component][block row][block column], rows padded, slots offset by
  // 8 doubles mod 16 so the two pairs of a half-warp use disjoint banks)
  static constexpr int kSlot = kR ? 4 * HB * (HB + 1) + 8 : D * RS;
  static constexpr size_t kSmem = size_t(PP) * kSlot * sizeof(double);
};

static_assert(progress_unit(5) == Deep<4>::kGroups && progress_unit(6) == Deep<5>::kGroups &&
                  progress_unit(7) == Deep<6>::kGroups && progress_unit(8) == Deep<7>::kGroups,
              "host progress unit = deep pair groups per tile");

__device__ __forceinline__ int insert0(int w, int p) {
  return ((w >> p) << (p + 1)) | (w & ((1 << p) - 1));
}

// One side of one qubit for this thread's column (COLS = false: F_i^T on the row index) or
// row (COLS = true: F_j on the column index, then the RY(delta) mask when H = 0).
template <int M, bool COLS>
__device__ __forceinline__ void deep_reg_round(double* V, double c, double s, double cd,
                                               double sd) {
  using Dp = Deep<M>;
  constexpr int D = Dp::D, RS = Dp::RS, G = Dp::G, N = 1 << G;
  const int w = threadIdx.x % Dp::IPP;
  const int lo = w % D, hi = w / D;  // lo: the fixed column (row side) or row (column side)
  double* base = V + (threadIdx.x / Dp::IPP) * Dp::kSlot + (COLS ? lo * RS : lo);
  constexpr int step = COLS ? 1 : RS;
  double x[N];
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = base[((hi << G) | k) * step];
#pragma unroll
  for (int k = 0; k < G; ++k)
#pragma unroll
    for (int e = 0; e < N; ++e) {
      if (e & (1 << k)) continue;
      rot_pair(x[e], x[e | (1 << k)], c, s, k == 0 ? 0 : (e >> (k - 1)) & 1);
    }
  if (COLS && Dp::H == 0) {  // top row bit = bit M-1 of lo, top column bit = bit M-1 of k
    const bool tb = (lo >> (M - 1)) & 1;
    const double m0 = tb ? sd : cd, m1 = tb ? cd : -sd;
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] *= ((k >> (M - 1)) & 1) ? m1 : m0;
  }
#pragma unroll
  for (int k = 0; k < N; ++k) base[((hi << G) | k) * step] = x[k];
}

// The top level (bit G of the side) as element-pair rotations, L = 8 only.
template <int M, bool COLS>
__device__ __forceinline__ void deep_pair_round(double* V, double c, double s, double cd,
                                                double sd) {
  using Dp = Deep<M>;
  constexpr int D = Dp::D, RS = Dp::RS, p0 = (COLS ? 0 : M) + Dp::G;
  for (int w = threadIdx.x; w < Dp::PP * (Dp::E / 2); w += kDeepThreads) {
    double* v = V + (w / (Dp::E / 2)) * Dp::kSlot;
    const int e0 = insert0(w % (Dp::E / 2), p0), e1 = e0 | (1 << p0);
    const int a0 = (e0 >> M) * RS + (e0 & (D - 1)), a1 = (e1 >> M) * RS + (e1 & (D - 1));
    double x0 = v[a0], x1 = v[a1];
    rot_pair(x0, x1, c, s, (e0 >> (p0 - 1)) & 1);
    if (COLS) {
      x0 *= ry_delta_mask(e0, M, cd, sd);
      x1 *= ry_delta_mask(e1, M, cd, sd);
    }
    v[a0] = x0;
    v[a1] = x1;
  }
}

// L = 6, 7 (and L = 5 with QK_DEEP_BONDR=0; one thread per column of a pair's D x D state):
// the state stays in registers for the whole sweep.  Layout A: thread t holds column t (x[r] = V[r][t]), so the
// F_i^T levels (on the row index) are register-local; layout B: thread t holds row t
// (x[c] = V[t][c]) for the F_j levels.  The row and column passes of one qubit commute, so
// even qubits run rows -> transpose -> columns -> mask and odd ones columns -> transpose ->
// rows -> mask: ONE transpose through the pair's shared-memory slot per qubit (each element
// written and read once: half the shared-memory traffic of two register rounds), synchronised
// only among the pair's D threads (a warp or, at D = 64, a named barrier) instead of the CTA.
#ifndef QK_DEEP_REG
#define QK_DEEP_REG 1
#endif
template <int M>
__device__ __forceinline__ void pair_sync() {
  if constexpr ((1 << M) <= 32) {
    __syncwarp();  // the pair's threads lie in one warp (and every warp runs the same loop)
  } else {
    const int id = 1 + int(threadIdx.x) / (1 << M);  // named barrier of the pair's 2 warps
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(1 << M) : "memory");
  }
}

// All M levels of one side on this thread's D values.  The previous qubit's RY(delta) mask is
// folded into level 0 (a pair differing in bit 0 shares its top bit, hence its mask factor):
// m0 / m1 scale the elements whose register top bit is 0 / 1.
template <int M>
__device__ __forceinline__ void deep_levels(double (&x)[1 << M], double c, double s, double m0,
                                            double m1) {
  constexpr int D = 1 << M;
  const double c0 = c * m0, s0 = s * m0, c1 = c * m1, s1 = s * m1;
#pragma unroll
  for (int e = 0; e < D; e += 2) {
    const bool top = (e >> (M - 1)) & 1;
    rot_pair(x[e], x[e + 1], top ? c1 : c0, top ? s1 : s0, 0);
  }
#pragma unroll
  for (int k = 1; k < M; ++k)
#pragma unroll
    for (int e = 0; e < D; ++e) {
      if (e & (1 << k)) continue;
      rot_pair(x[e], x[e | (1 << k)], c, s, (e >> (k - 1)) & 1);
    }
}

// The RY(delta) mask factors of this thread's two element groups (register top bit 0 / 1);
// ROW_OWNER: thread t holds row t (layout B), else column t (layout A).
template <int M, bool ROW_OWNER>
__device__ __forceinline__ void deep_mask_factors(int t, double cd, double sd, double& m0,
                                                  double& m1) {
  const bool mine = (t >> (M - 1)) & 1;
  // element top bits (tb: row, tc: column) = (mine, g) for a row owner, (g, mine) otherwise
  auto f = [&](bool g) {
    const bool tb = ROW_OWNER ? mine : g, tc = ROW_OWNER ? g : mine;
    return tb == tc ? cd : (tb ? sd : -sd);
  };
  m0 = f(false);
  m1 = f(true);
}

template <int M, bool TO_ROWS>  // A -> B (TO_ROWS) or B -> A through the pair's slot v
__device__ __forceinline__ void deep_transpose(double* v, double (&x)[1 << M], int t) {
  constexpr int D = 1 << M, RS = D + 1;
  pair_sync<M>();  // the previous transpose's reads of v are done
#pragma unroll
  for (int e = 0; e < D; ++e) v[TO_ROWS ? e * RS + t : t * RS + e] = x[e];
  pair_sync<M>();
#pragma unroll
  for (int e = 0; e < D; ++e) x[e] = v[TO_ROWS ? t * RS + e : e * RS + t];
}

template <int M>
__device__ __forceinline__ void deep_sweep_reg(double* V, double* red, const double2* pi,
                                               const double2* pj, int q_begin, int q_end) {
  using Dp = Deep<M>;
  constexpr int D = Dp::D;
  const int t = threadIdx.x % D;
  double* v = V + (threadIdx.x / D) * Dp::kSlot;
  double x[D];
#pragma unroll
  for (int e = 0; e < D; ++e) x[e] = 0.0;
  if (t == 0) x[0] = 1.0;  // V = e_00, layout A
  // the mask of each qubit is deferred into the next qubit's first level (m0 / m1: pending
  // factors of the current layout's two element groups)
  double m0 = 1.0, m1 = 1.0;
  int q = q_begin;
  for (; q + 1 < q_end; q += 2) {
    {  // even: layout A in, B out
      const double2 vi = __ldg(pi + int64_t(q) * kTile), vj = __ldg(pj + int64_t(q) * kTile);
      const double cd = fma(vi.y, vj.y, vi.x * vj.x), sd = fma(vi.x, vj.y, -(vi.y * vj.x));
      deep_levels<M>(x, vi.x, vi.y, m0, m1);
      deep_transpose<M, true>(v, x, t);
      deep_levels<M>(x, vj.x, vj.y, 1.0, 1.0);
      deep_mask_factors<M, true>(t, cd, sd, m0, m1);
    }
    {  // odd: layout B in, A out
      const double2 vi = __ldg(pi + int64_t(q + 1) * kTile),
                    vj = __ldg(pj + int64_t(q + 1) * kTile);
      const double cd = fma(vi.y, vj.y, vi.x * vj.x), sd = fma(vi.x, vj.y, -(vi.y * vj.x));
      deep_levels<M>(x, vj.x, vj.y, m0, m1);
      deep_transpose<M, false>(v, x, t);
      deep_levels<M>(x, vi.x, vi.y, 1.0, 1.0);
      deep_mask_factors<M, false>(t, cd, sd, m0, m1);
    }
  }
  if (q < q_end) {  // a last even qubit
    const double2 vi = __ldg(pi + int64_t(q) * kTile), vj = __ldg(pj + int64_t(q) * kTile);
    const double cd = fma(vi.y, vj.y, vi.x * vj.x), sd = fma(vi.x, vj.y, -(vi.y * vj.x));
    deep_levels<M>(x, vi.x, vi.y, m0, m1);
    deep_transpose<M, true>(v, x, t);
    deep_levels<M>(x, vj.x, vj.y, 1.0, 1.0);
    deep_mask_factors<M, true>(t, cd, sd, m0, m1);
  }
#pragma unroll
  for (int e = 0; e < D; ++e) x[e] *= ((e >> (M - 1)) & 1) ? m1 : m0;  // the last pending mask
  // amp = sum(V): each thread its D values in order, then the pair's D partial sums in order
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < D; ++e) acc += x[e];
  __syncthreads();
  red[threadIdx.x] = acc;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int k = 0; k < D; ++k) s += red[threadIdx.x + k];
    red[threadIdx.x] = s;  // only this thread touches its group's first entry now
  }
  __syncthreads();
}

// L = 5 in the rotated blocked form of L = 3, 4 (bondr_step) over registers of HB = 8 threads
// per pair: thread t holds block column t (layout A: x[4 r + q], the lower row levels are
// local) or block row t (layout B: x[4 c + q], the lower column levels), the two layouts
// alternating by qubit as in deep_sweep_reg (one transpose per qubit).  The per-block
// L = 2-type step depends on the top-level selectors (TR, TC) = bit M-2 of the block's row and
// column; one of them is a thread bit, so each thread forms the step's eight coefficients for
// both values of the other (all four variants are 2-term combinations of (S, Dg) and (T, E)).
struct BCoef {
  double a0, b0, a1, b1, a2, b2, a3, b3;
};

__device__ __forceinline__ BCoef bondr_coef(bool tr, bool tc, double C, double D, double p1,
                                            double q1, double p2, double q2) {
  const double opc = 1.0 + C, cm1 = C - 1.0;
  BCoef k;
  if (tr == tc) {  // (0, 0) / (1, 1)
    k.a0 = opc, k.b0 = tr ? -q1 : q1, k.a1 = cm1, k.b1 = tr ? -p2 : p2;
    k.a2 = tr ? -p1 : p1, k.b2 = -D, k.a3 = tr ? -q2 : q2, k.b3 = D;
  } else {  // (0, 1) / (1, 0)
    k.a0 = tr ? D : -D, k.b0 = p1, k.a1 = tr ? D : -D, k.b1 = -q2;
    k.a2 = -q1, k.b2 = tr ? opc : -opc, k.a3 = p2, k.b3 = tr ? -cm1 : cm1;
  }
  return k;
}

__device__ __forceinline__ void bondr_block(double* v, const BCoef& k) {
  const double S = v[0], Dg = v[1], T = v[2], E = v[3];
  v[0] = fma(k.b0, Dg, k.a0 * S);
  v[1] = fma(k.b1, E, k.a1 * T);
  v[2] = fma(k.b2, E, k.a2 * T);
  v[3] = fma(k.b3, Dg, k.a3 * S);
}

// Per-pair thread geometry of the blocked form: HB block columns (layout A) / rows (B), one
// thread each, holding the column's / row's NB = HB blocks (4 components each).  (Splitting a
// column over two lanes for L = 6, with the top lower level as a lane exchange, measured 12 %
// slower than the column-per-thread form: 0.69 vs 0.78 M entries/s at 784 qubits.)
template <int M>
struct BondRGeo {
  static constexpr int HB = 1 << (M - 1), NB = HB, N = 4 * NB;
};

// The lower levels (k = 0 .. M-2) on the owned block index, register-local.
template <int M>
__device__ __forceinline__ void bondr_lower(double (&x)[BondRGeo<M>::N], double c, double s) {
  using G = BondRGeo<M>;
#pragma unroll
  for (int k = 0; k < M - 1; ++k)
#pragma unroll
    for (int b = 0; b < G::NB; ++b) {
      if (b & (1 << k)) continue;
      const int b1 = b | (1 << k), sel = k == 0 ? 0 : (b >> (k - 1)) & 1;
#pragma unroll
      for (int q = 0; q < 4; ++q) rot_pair(x[4 * b + q], x[4 * b1 + q], c, s, sel);
    }
}

template <int M, bool TO_ROWS>  // A -> B (TO_ROWS) or B -> A through the pair's slot v
__device__ __forceinline__ void bondr_transpose(double* v, double (&x)[BondRGeo<M>::N], int o) {
  using G = BondRGeo<M>;
  constexpr int RS = G::HB + 1, QS = G::HB * RS;
  __syncwarp();  // the previous transpose's reads of v are done
#pragma unroll
  for (int b = 0; b < G::NB; ++b)
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q * QS + (TO_ROWS ? b * RS + o : o * RS + b)] = x[4 * b + q];
  __syncwarp();
#pragma unroll
  for (int b = 0; b < G::NB; ++b)
#pragma unroll
    for (int q = 0; q < 4; ++q) x[4 * b + q] = v[q * QS + (TO_ROWS ? o * RS + b : b * RS + o)];
}

template <int M>
__device__ __forceinline__ void deep_sweep_bondr(double* V, double* red, const double2* pi,
                                                 const double2* pj, int q_begin, int q_end,
                                                 double final_scale) {
  using Dp = Deep<M>;
  using G = BondRGeo<M>;
  constexpr int HB = G::HB, NB = G::NB, N = G::N, TPP = HB;
  static_assert(TPP <= 32, "a pair within one warp");
  const int o = threadIdx.x % TPP;  // the block column (A) / row (B) this thread owns
  double* v = V + (threadIdx.x / TPP) * Dp::kSlot;
  const bool obit = (o >> (M - 2)) & 1;  // selector bit of this thread's owned row (B) / col (A)
  double x[N];
#pragma unroll
  for (int e = 0; e < N; ++e) x[e] = 0.0;
  if (o == 0) x[0] = x[2] = 1.0;  // block (0, 0) as bondr_init, layout A
  auto qubit = [&](int q, bool even) {
    const double2 vi = __ldg(pi + int64_t(q) * kTile), vj = __ldg(pj + int64_t(q) * kTile);
    const double ci = vi.x, si = vi.y, cj = vj.x, sj = vj.y;
    const double ai = fma(ci, ci, -(si * si)), bi = (ci + ci) * si;
    const double aj = fma(cj, cj, -(sj * sj)), bj = (cj + cj) * sj;
    const double C = fma(bi, bj, ai * aj), D = fma(-bi, aj, ai * bj);
    const double p1 = ai + aj, q1 = bi + bj, p2 = bj - bi, q2 = ai - aj;
    // the selector of the dimension this thread holds NB blocks of: bit M-2 of the block index
    auto held_bit = [&](int b) { return ((b >> (M - 2)) & 1) != 0; };
    if (even) {  // A: rows, transpose, B: columns, blocks (o, b): TR = obit
      bondr_lower<M>(x, ci, si);
      bondr_transpose<M, true>(v, x, o);
      bondr_lower<M>(x, cj, sj);
      const BCoef k0 = bondr_coef(obit, false, C, D, p1, q1, p2, q2);
      const BCoef k1 = bondr_coef(obit, true, C, D, p1, q1, p2, q2);
#pragma unroll
      for (int b = 0; b < NB; ++b) bondr_block(x + 4 * b, held_bit(b) ? k1 : k0);
    } else {  // B: columns, transpose, A: rows, blocks (b, o): TC = obit
      bondr_lower<M>(x, cj, sj);
      bondr_transpose<M, false>(v, x, o);
      bondr_lower<M>(x, ci, si);
      const BCoef k0 = bondr_coef(false, obit, C, D, p1, q1, p2, q2);
      const BCoef k1 = bondr_coef(true, obit, C, D, p1, q1, p2, q2);
#pragma unroll
      for (int b = 0; b < NB; ++b) bondr_block(x + 4 * b, held_bit(b) ? k1 : k0);
    }
    if ((q + 1) % (kChunk * kRescaleChunks) == 0 && q + 1 < q_end) {  // as the L = 3, 4 sweep
#pragma unroll
      for (int e = 0; e < N; ++e) x[e] *= 0x1p-512;
    }
  };
  int q = q_begin;
  for (; q + 1 < q_end; q += 2) {
    qubit(q, true);
    qubit(q + 1, false);
  }
  if (q < q_end) qubit(q, true);
  // amp = sum over blocks of (S + Dg) (bondr_amp): each thread its blocks in order, then the
  // pair's TPP partial sums in order
  double acc = 0.0;
#pragma unroll
  for (int b = 0; b < NB; ++b) acc += x[4 * b] + x[4 * b + 1];
  __syncthreads();
  red[threadIdx.x] = acc;
  __syncthreads();
  if (o == 0) {
    double sum = 0.0;
    for (int k = 0; k < TPP; ++k) sum += red[threadIdx.x + k];
    red[threadIdx.x] = sum * final_scale;
  }
  __syncthreads();
}

// Sweeps the PP pairs whose plane columns (qubit 0) are pi / pj for this thread's slot;
// leaves amp of slot s in red[s * IPP].  Starts and ends with a barrier.
template <int M>
__device__ __forceinline__ void deep_sweep(double* V, double* red, const double2* pi,
                                           const double2* pj, int q_begin, int q_end,
                                           double final_scale) {
  using Dp = Deep<M>;
  if constexpr (Dp::kR) {
    __syncthreads();
    deep_sweep_bondr<M>(V, red, pi, pj, q_begin, q_end, final_scale);
  } else if constexpr (QK_DEEP_REG && Dp::H == 0) {
    __syncthreads();
    deep_sweep_reg<M>(V, red, pi, pj, q_begin, q_end);
  } else {
    for (int e = threadIdx.x; e < Dp::PP * Dp::kSlot; e += kDeepThreads)
      V[e] = (e % Dp::kSlot) == 0 ? 1.0 : 0.0;
    __syncthreads();
    for (int q = q_begin; q < q_end; ++q) {
      const double2 vi = __ldg(pi + int64_t(q) * kTile), vj = __ldg(pj + int64_t(q) * kTile);
      const double cd = fma(vi.y, vj.y, vi.x * vj.x);   // cos((x_j - x_i)/2)
      const double sd = fma(vi.x, vj.y, -(vi.y * vj.x));  // sin((x_j - x_i)/2)
      deep_reg_round<M, false>(V, vi.x, vi.y, cd, sd);
      __syncthreads();
      if constexpr (Dp::H > 0) {
        deep_pair_round<M, false>(V, vi.x, vi.y, cd, sd);
        __syncthreads();
      }
      deep_reg_round<M, true>(V, vj.x, vj.y, cd, sd);
      __syncthreads();
      if constexpr (Dp::H > 0) {
        deep_pair_round<M, true>(V, vj.x, vj.y, cd, sd);
        __syncthreads();
      }
    }
    // amp = sum(V) per slot (padding entries are zero): IPP threads per slot, fixed order
    const int w = threadIdx.x % Dp::IPP;
    const double* v = V + (threadIdx.x / Dp::IPP) * Dp::kSlot;
    double acc = 0.0;
    for (int e = w; e < Dp::kSlot; e += Dp::IPP) acc += v[e];
    red[threadIdx.x] = acc;
    __syncthreads();
    if (w == 0) {
      double t = 0.0;
      for (int k = 0; k < Dp::IPP; ++k) t += red[threadIdx.x + k];
      red[threadIdx.x] = t;  // only this thread touches its group's first entry now
    }
    __syncthreads();
  }
}

template <int M, int MODE, int OUT>
__global__ void __launch_bounds__(kDeepThreads) sweep_deep_kernel(const SweepArgs a) {
  extern __shared__ double V[];
  __shared__ double red[kDeepThreads];
  constexpr int PP = Deep<M>::PP, G = Deep<M>::kGroups, TPS = Deep<M>::IPP;
  const int my_slot = threadIdx.x / TPS;
  const int64_t items = a.n_tiles * G;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t g = a.tile_begin + it / G;
    const int grp = int(it % G);
    int64_t bi, bj;
    if (MODE == kModeGram) {
      decode_upper(g, a.nb_rows, bi, bj);
    } else {
      decode_rect(g, a.nb_rows, a.nb_cols, bi, bj, a.rect_tail);
    }
    // does any pair of the group need computing?  (uniform: every thread evaluates all)
    bool any = false;
#pragma unroll
    for (int sl = 0; sl < PP; ++sl) {
      const int pl = grp * PP + sl;
      const int64_t i = bi * kTile + pl / kTile - a.pad_rows, j = bj * kTile + pl % kTile - a.pad_cols;
      any |= MODE == kModeGram ? (i >= 0 && i < j && j < a.n_rows)
                               : (i >= 0 && j >= 0 && i < a.n_rows && j < a.n_cols);
    }
    const int pl = grp * PP + my_slot, il = pl / kTile, jl = pl % kTile;
    if (any) {
      deep_sweep<M>(V, red, a.rows + bi * int64_t(a.n_pad) * kTile + il,
                    a.cols + bj * int64_t(a.n_pad) * kTile + jl, a.front, a.n_pad,
                    a.final_scale);
    }
    if (threadIdx.x % TPS == 0) {
      const int64_t i = bi * kTile + il - a.pad_rows, j = bj * kTile + jl - a.pad_cols;
      const bool need = MODE == kModeGram ? (i >= 0 && i < j && j < a.n_rows)
                                          : (i >= 0 && j >= 0 && i < a.n_rows && j < a.n_cols);
      const double v = need ? kernel_value(red[threadIdx.x], a.convention) : 0.0;
      if (OUT == QK_OUT_PACKED) {
        a.out[(g - a.tile_begin) * int64_t(kTile * kTile) + pl] = v;
      } else if (MODE == kModeGram) {
        if (need) {
          a.out[i * a.ld_out + j] = v;
          a.out[j * a.ld_out + i] = v;
        } else if (i == j && i >= 0 && i < a.n_rows) {
          a.out[i * a.ld_out + i] = 1.0;
        }
      } else if (need) {
        a.out[i * a.ld_out + j] = v;
      }
    }
    __syncthreads();  // red and V are reused by the next item
    if (a.progress != nullptr) {
      if (threadIdx.x % TPS == 0) QK_PROGRESS_FENCE();
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(a.progress + bi, 1u);  // G per tile
    }
  }
}

template <int M>
__global__ void __launch_bounds__(kDeepThreads) pairs_deep_kernel(
    const double2* __restrict__ A, int64_t n_a, const double2* __restrict__ B, int64_t n_b,
    const int64_t* __restrict__ pairs, int64_t n_pairs, double* __restrict__ amp, int n_pad,
    int front, int value, double final_scale) {
  extern __shared__ double V[];
  __shared__ double red[kDeepThreads];
  constexpr int PP = Deep<M>::PP, TPS = Deep<M>::IPP;
  const int my_slot = threadIdx.x / TPS;
  const int64_t k = int64_t(blockIdx.x) * PP + my_slot;
  int64_t p = 0, q = 0;
  bool ok = false;
  if (k < n_pairs) {
    p = pairs[2 * k];
    q = pairs[2 * k + 1];
    ok = p >= 0 && p < n_a && q >= 0 && q < n_b;
  }
  if (!ok) p = q = 0;  // sweep a valid column; the result is discarded
  const int64_t sp = p + sample_pad(n_a), sq = q + sample_pad(n_b);  // plane slots
  deep_sweep<M>(V, red, A + (sp / kTile) * int64_t(n_pad) * kTile + (sp % kTile),
                B + (sq / kTile) * int64_t(n_pad) * kTile + (sq % kTile), front, n_pad,
                final_scale);
  if (threadIdx.x % TPS == 0 && k < n_pairs)
    amp[k] = !ok ? __longlong_as_double(0x7ff8000000000000LL)
                 : value < 0 ? red[threadIdx.x] : kernel_value(red[threadIdx.x], value);
}

// ------------------------------------------------------------------------------------------
// Pair-list kernel: one pair per thread, planes read straight from global/L2.
// ------------------------------------------------------------------------------------------
template <int LAYERS>
__global__ void __launch_bounds__(128) pairs_kernel(const double2* __restrict__ A, int64_t n_a,
                                                    const double2* __restrict__ B, int64_t n_b,
                                                    const int64_t* __restrict__ pairs,
                                                    int64_t n_pairs, double* __restrict__ amp,
                                                    int n_pad, int nchunks, int front,
                                                    double final_scale, int value) {
  using St = typename BondT<LAYERS>::type;
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n_pairs) return;
  const int64_t p = pairs[2 * k], q = pairs[2 * k + 1];
  if (p < 0 || p >= n_a || q < 0 || q >= n_b) {
    amp[k] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  const int64_t sp = p + sample_pad(n_a), sq = q + sample_pad(n_b);  // plane slots
  const double2* a = A + (sp / kTile) * int64_t(n_pad) * kTile + (sp % kTile);
  const double2* b = B + (sq / kTile) * int64_t(n_pad) * kTile + (sq % kTile);
  St s;
  st_init<LAYERS>(s);
  for (int ch = 0; ch < nchunks; ++ch) {
#pragma unroll 4
    for (int qq = ch == 0 ? front : 0; qq < kChunk; ++qq) {  // front padding: identities
      const int64_t off = int64_t(ch * kChunk + qq) * kTile;
      st_step<LAYERS>(s, __ldg(a + off), __ldg(b + off));
    }
    if (LAYERS >= 2 && ch + 1 < nchunks && ((ch + 1) % kRescaleChunks) == 0)
      st_rescale<LAYERS>(s);
  }
  const double v = st_amp<LAYERS>(s, final_scale);
  amp[k] = value < 0 ? v : kernel_value(v, value);  // value: -1 amplitude, else convention
}

// ------------------------------------------------------------------------------------------
// Unpack packed tiles (multi-rank gather output) into the dense kernel matrix.
// ------------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(256) unpack_kernel(const double* __restrict__ packed,
                                                     int64_t n_rows, int64_t n_cols,
                                                     int64_t nb_rows, int64_t nb_cols,
                                                     int64_t tile_begin, double* __restrict__ K,
                                                     int64_t ld) {
  const int64_t g = tile_begin + blockIdx.x;
  int64_t bi, bj;
  if (MODE == kModeGram) {
    decode_upper(g, nb_rows, bi, bj);
  } else {
    decode_rect(g, nb_rows, nb_cols, bi, bj);
  }
  const double* src = packed + int64_t(blockIdx.x) * kTile * kTile;
  const int pr = sample_pad(n_rows), pc = sample_pad(n_cols);
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int il = e / kTile, jl = e % kTile;
    const int64_t i = bi * kTile + il - pr, j = bj * kTile + jl - pc;
    const double v = src[e];
    if (MODE == kModeGram) {
      if (i >= 0 && i < n_rows && j < n_rows) {
        if (i < j) {
          K[i * ld + j] = v;
          K[j * ld + i] = v;
        } else if (i == j) {
          K[i * ld + i] = 1.0;
        }
      }
    } else if (i >= 0 && j >= 0 && i < n_rows && j < n_cols) {
      K[i * ld + j] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------
// FP64 FMA issue-rate microbenchmark: 8 independent DFMA chains per thread.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  const double m = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;  // keep the chains alive
}

// ------------------------------------------------------------------------------------------
// Launchers
// ------------------------------------------------------------------------------------------
static qk_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return QK_OK;
  return set_error(QK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  if ((sms = cache[dev].load(std::memory_order_relaxed)) > 0) return sms;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  cache[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

// Resident CTAs per SM of a kernel with `smem` bytes of dynamic shared memory, after opting it
// in to that much shared memory — once per (kernel, device): the attribute call and the
// occupancy query cost microseconds of host time, which small jobs notice.
template <class Kern>
static qk_status resident_ctas(Kern kern, int threads, size_t smem, int* per_sm) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_status(e, "cudaGetDevice");
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), dev, threads, smem);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *per_sm = it->second;
    return QK_OK;
  }
  if (smem > 48 * 1024)
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem)))
      return cuda_status(e, "smem attribute");
  int n = 0;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem))
    return cuda_status(e, "occupancy");
  *per_sm = n < 1 ? 1 : n;
  cache.emplace(key, *per_sm);
  return QK_OK;
}

// Plane sets s0 (and s1 when s1.nblk > 0) in one launch.
static qk_status launch_gate_sets(const Plan& p, GateSet s0, GateSet s1, cudaStream_t st) {
  const int64_t nb = s0.nblk + s1.nblk;
  if (nb <= 0) return QK_OK;
  auto al32 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 31u) == 0; };
  const bool vec = p.front_pad % 4 == 0 && s0.ld % 4 == 0 && al32(s0.X) &&
                   (s1.nblk == 0 || (s1.ld % 4 == 0 && al32(s1.X)));
  const int half = p.layers == 2 ? 0 : 1;
  // QK_GATE_VARIANT (tuning; ncu, 10,000 x 784, B200): 0 = 2 quads per thread, one CTA per
  // 32-qubit item (default: 35.0 us, 5.39 TB/s algorithmic); 1 = 4 quads, 64-qubit items
  // (38.3 us); 2 = 2 quads, persistent double-buffered (43 us); 3 = 2 quads, 6 resident CTAs
  // per SM; 4 = 1 quad, 16-qubit items
  static const int variant = [] {
    const char* v = getenv("QK_GATE_VARIANT");
    return v == nullptr ? 0 : v[0] - '0';
  }();
  auto launch = [&](auto kern, int qd, bool persist) -> qk_status {
    const int64_t items = nb * ((p.width_padded + 16 * qd - 1) / (16 * qd));
    int64_t grid = items;
    if (persist) {
      int per_sm = 0;
      if (qk_status s = resident_ctas(kern, 256, 0, &per_sm)) return s;
      const int sms = sm_count();
      if (sms <= 0) return set_error(QK_ERR_CUDA, "no CUDA device");
      grid = std::min<int64_t>(items, int64_t(sms) * per_sm);
    }
    kern<<<unsigned(grid), 256, 0, st>>>(s0, s1, p.width, p.width_padded, p.front_pad, half);
    return QK_OK;
  };
  qk_status ls;
  switch (variant) {
    case 1:
      ls = vec ? launch(gate_build_kernel<true, 4, false, 1>, 4, false)
               : launch(gate_build_kernel<false, 4, false, 1>, 4, false);
      break;
    case 2:
      ls = vec ? launch(gate_build_kernel<true, 2, true, 4>, 2, true)
               : launch(gate_build_kernel<false, 2, true, 4>, 2, true);
      break;
    case 3:
      ls = vec ? launch(gate_build_kernel<true, 2, false, 6>, 2, false)
               : launch(gate_build_kernel<false, 2, false, 6>, 2, false);
      break;
    case 4:
      ls = vec ? launch(gate_build_kernel<true, 1, false, 1>, 1, false)
               : launch(gate_build_kernel<false, 1, false, 1>, 1, false);
      break;
    default:
      ls = vec ? launch(gate_build_kernel<true, 2, false, 1>, 2, false)
               : launch(gate_build_kernel<false, 2, false, 1>, 2, false);
  }
  if (ls != QK_OK) return ls;
  return cuda_status(cudaGetLastError(), "gate_build launch");
}

static GateSet gate_set(const double* X, int64_t n, int64_t ld, void* planes, uint64_t* bad,
                        int64_t blk_begin, int64_t blk_end) {
  if (blk_end < 0 || blk_end > blocks_for(n)) blk_end = blocks_for(n);
  GateSet g{X, n, ld, static_cast<double2*>(planes),
            reinterpret_cast<unsigned long long*>(bad), blk_begin,
            n == 0 ? 0 : std::max<int64_t>(0, blk_end - blk_begin)};
  return g;
}

qk_status launch_gate_build(const Plan& p, const double* d_angles, int64_t n, int64_t ld,
                            void* d_planes, uint64_t* d_bad, void* stream, int64_t blk_begin,
                            int64_t blk_end) {
  if (n == 0) return QK_OK;
  return launch_gate_sets(p, gate_set(d_angles, n, ld, d_planes, d_bad, blk_begin, blk_end),
                          GateSet{}, static_cast<cudaStream_t>(stream));
}

qk_status launch_gate_build2(const Plan& p, const double* d_a, int64_t n_a, void* d_planes_a,
                             uint64_t* d_bad_a, const double* d_b, int64_t n_b,
                             void* d_planes_b, uint64_t* d_bad_b, void* stream,
                             int64_t blk_begin_a) {
  return launch_gate_sets(p, gate_set(d_a, n_a, p.width, d_planes_a, d_bad_a, blk_begin_a, -1),
                          gate_set(d_b, n_b, p.width, d_planes_b, d_bad_b, 0, -1),
                          static_cast<cudaStream_t>(stream));
}

// Per-launch tile-claim counters (the dynamic schedule): a ring of reset 8-byte slots per
// device, one per launch, so concurrent launches on different streams never share one.  A
// launch captured into a CUDA graph gets its own stream-ordered allocation instead (a graph
// memory node, allocated and freed around the kernel on every replay), so a replay never
// shares a counter with a later ring launch.  *owned: the caller frees it after the launch.
qk_status acquire_tile_counter(void* stream, unsigned long long** out, bool* owned) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  constexpr int kSlots = 4096;
  static unsigned long long* pool[64] = {};
  static std::mutex mu;
  static std::atomic<uint64_t> seq{0};
  *owned = false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaError_t e = cudaStreamIsCapturing(st, &cap)) return cuda_status(e, "capture query");
  if (cap == cudaStreamCaptureStatusActive) {
    if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), sizeof(unsigned long long), st))
      return cuda_status(e, "captured tile counter");
    *owned = true;
  } else {
    int dev = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return cuda_status(e, "cudaGetDevice");
    if (dev < 0 || dev >= 64) return set_error(QK_ERR_CUDA, "device index out of range");
    {
      std::lock_guard<std::mutex> g(mu);
      if (pool[dev] == nullptr)
        if (cudaError_t e = cudaMalloc(&pool[dev], kSlots * sizeof(unsigned long long)))
          return cuda_status(e, "tile counter allocation");
    }
    *out = pool[dev] + (seq.fetch_add(1) % kSlots);
  }
  // all-ones: a claim adds one and wraps to 0 (one memset value for a job's whole state)
  return cuda_status(cudaMemsetAsync(*out, 0xFF, sizeof(unsigned long long), st),
                     "tile counter reset");
}

// Short chains (width_padded <= kShortChain): per-warp epilogue (EPI = 1), and a job of only a
// few waves runs every tile as two row halves (finer dynamic balance over the 148 SMs).
// QK_SHORT_CHAIN overrides the threshold (0: never).
static int short_chain_limit() {
  static const int v = [] {
    const char* e = getenv("QK_SHORT_CHAIN");
    return e == nullptr ? 64 : atoi(e);
  }();
  return v;
}

template <int LAYERS, int MODE, int OUT, int RI, int EPI>
static qk_status launch_sweep_ri(SweepArgs a, cudaStream_t st) {
  bool owned = false;  // a.next_tile preset: the caller reset it earlier in stream order
  if (a.next_tile == nullptr)
    if (qk_status s = acquire_tile_counter(st, &a.next_tile, &owned)) return s;
  struct Release {  // a captured counter is freed after the launch, on the same stream
    unsigned long long* p;
    cudaStream_t st;
    bool on;
    ~Release() {
      if (on) cudaFreeAsync(p, st);
    }
  } release{a.next_tile, st, owned};
  auto kern = sweep_kernel<LAYERS, MODE, OUT, RI, EPI>;
  constexpr int threads = Geo<RI>::kThreads;
  int per_sm = 0;
  if (qk_status s = resident_ctas(kern, threads, kSmemBytes, &per_sm)) return s;
  const int sms = sm_count();
  if (sms <= 0) return set_error(QK_ERR_CUDA, "no CUDA device");
  int64_t grid = int64_t(sms) * per_sm;
  // the last wave runs as half tiles; short-chain jobs of a few waves: every tile
  static const int split_mode = [] {  // QK_HALF_TILES: 0 off, 1 on
    const char* v = getenv("QK_HALF_TILES");
    return v == nullptr ? 1 : v[0] - '0';
  }();
  const bool split = split_mode == 1;
  static const double split_waves = [] {  // QK_SPLIT_WAVES: tail tiles split, in grids (tuning)
    const char* v = getenv("QK_SPLIT_WAVES");
    return v == nullptr ? -1.0 : atof(v);
  }();
  if (RI == 1)  // 32-row layout: every item is a half tile
    a.n_split = a.n_tiles;
  else if (!split)
    a.n_split = 0;
  else if (split_waves >= 0)
    a.n_split = std::min<int64_t>(a.n_tiles, int64_t(split_waves * grid));
  else
    a.n_split = (EPI == 1 && a.n_tiles <= 4 * grid) ? a.n_tiles : std::min<int64_t>(a.n_tiles, grid);
  if (grid > a.n_tiles + a.n_split) grid = a.n_tiles + a.n_split;
  if (!a.pdl) {
    kern<<<unsigned(grid), threads, kSmemBytes, st>>>(a);
    return cuda_status(cudaGetLastError(), "sweep launch");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_status(cudaLaunchKernelEx(&cfg, kern, a), "sweep launch (programmatic)");
}

// Micro-tile rows per thread: 2 (512 threads, 2x4 micro-tiles, 16 warps/SM) or 4 (256
// threads, 4x4 micro-tiles).  Measured (784 qubits, one B200): L = 2 RI 2 1.206 vs RI 4
// 1.171 G entries/s; L = 1 (3 FP64 instructions per pair-qubit, so the shared-memory loads
// per pair matter) RI 2 4.18 vs RI 4 5.49 G entries/s.  QK_SWEEP_RI=2/4 overrides.
static int sweep_ri(int layers) {
  static int forced = [] {
    const char* v = getenv("QK_SWEEP_RI");
    return v == nullptr ? 0 : (v[0] == '4' ? 4 : 2);
  }();
  if (forced) return forced;
  return layers == 1 ? 4 : 2;
}

// Short chains at L = 2 run 32-row items with all 16 warps busy (RI = 1) unless
// QK_SHORT_RI1=0 (then 64-row items, half of them split, with RI = 2).
static bool short_ri1() {
  static const bool v = [] {
    const char* e = getenv("QK_SHORT_RI1");
    return e == nullptr || e[0] != '0';
  }();
  return v;
}

template <int LAYERS, int MODE, int OUT>
static qk_status launch_sweep_t(const SweepArgs& a, cudaStream_t st) {
  const bool short_chain = OUT == QK_OUT_DENSE && a.n_pad <= short_chain_limit();
  if constexpr (LAYERS == 2 && OUT == QK_OUT_DENSE)
    if (short_chain && short_ri1()) return launch_sweep_ri<LAYERS, MODE, OUT, 1, 1>(a, st);
  if (sweep_ri(LAYERS) == 2)
    return short_chain ? launch_sweep_ri<LAYERS, MODE, OUT, 2, 1>(a, st)
                       : launch_sweep_ri<LAYERS, MODE, OUT, 2, 0>(a, st);
  return short_chain ? launch_sweep_ri<LAYERS, MODE, OUT, 4, 1>(a, st)
                     : launch_sweep_ri<LAYERS, MODE, OUT, 4, 0>(a, st);
}

template <int LAYERS, int MODE, int OUT>
static qk_status launch_general(const SweepArgs& a, cudaStream_t st) {
  auto kern = sweep_general_kernel<LAYERS, MODE, OUT>;
  int per_sm = 0;
  if (qk_status s = resident_ctas(kern, 256, 0, &per_sm)) return s;
  const int sms = sm_count();
  if (sms <= 0) return set_error(QK_ERR_CUDA, "no CUDA device");
  int64_t grid = int64_t(sms) * per_sm;
  if (grid > a.n_tiles * 16) grid = a.n_tiles * 16;
  kern<<<unsigned(grid), 256, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "general sweep launch");
}

template <int M, int MODE, int OUT>
static qk_status launch_deep(const SweepArgs& a, cudaStream_t st) {
  auto kern = sweep_deep_kernel<M, MODE, OUT>;
  constexpr size_t smem = Deep<M>::kSmem;
  int per_sm = 0;
  if (qk_status s = resident_ctas(kern, kDeepThreads, smem, &per_sm)) return s;
  const int sms = sm_count();
  if (sms <= 0) return set_error(QK_ERR_CUDA, "no CUDA device");
  int64_t grid = int64_t(sms) * per_sm;
  const int64_t items = a.n_tiles * Deep<M>::kGroups;
  if (grid > items) grid = items;
  kern<<<unsigned(grid), kDeepThreads, smem, st>>>(a);
  return cuda_status(cudaGetLastError(), "deep sweep launch");
}

template <int M>
static qk_status launch_deep_t(const SweepArgs& a, int mode, bool packed, cudaStream_t st) {
  if (mode == kModeGram)
    return packed ? launch_deep<M, kModeGram, QK_OUT_PACKED>(a, st)
                  : launch_deep<M, kModeGram, QK_OUT_DENSE>(a, st);
  return packed ? launch_deep<M, kModeCross, QK_OUT_PACKED>(a, st)
                : launch_deep<M, kModeCross, QK_OUT_DENSE>(a, st);
}

template <int M>
static qk_status launch_pairs_deep(const Plan& p, const void* d_a, int64_t n_a, const void* d_b,
                                   int64_t n_b, const int64_t* d_pairs, int64_t n_pairs,
                                   double* d_amp, int value, cudaStream_t st) {
  auto kern = pairs_deep_kernel<M>;
  constexpr size_t smem = Deep<M>::kSmem;
  int per_sm = 0;
  if (qk_status s = resident_ctas(kern, kDeepThreads, smem, &per_sm)) return s;
  const int64_t grid = (n_pairs + Deep<M>::PP - 1) / Deep<M>::PP;
  kern<<<unsigned(grid), kDeepThreads, smem, st>>>(
      static_cast<const double2*>(d_a), n_a, static_cast<const double2*>(d_b), n_b, d_pairs,
      n_pairs, d_amp, p.width_padded, p.front_pad, value, p.final_scale);
  return cuda_status(cudaGetLastError(), "deep pairs launch");
}

qk_status launch_sweep(const Plan& p, int mode, const void* d_rows, int64_t n_rows,
                       const void* d_cols, int64_t n_cols, int64_t tile_begin, int64_t tile_end,
                       double* d_out, int64_t ld_out, int out_mode, void* stream,
                       unsigned int* d_progress, int64_t head_b, unsigned long long* counter,
                       bool pdl, int64_t rect_tail) {
  if (tile_end <= tile_begin) return QK_OK;
  if (head_b != 0 && (p.layers > 2 || head_b % kGroup != 0))
    return set_error(QK_ERR_VALUE, "Gram head order needs layers <= 2 and a multiple of 8");
  SweepArgs a{};
  a.next_tile = counter;
  a.pdl = pdl ? 1 : 0;
  a.rect_tail = rect_tail < 0 ? kRectTail : rect_tail;
  if (mode == kModeGram) a.head_b = head_b;
  a.progress = d_progress;
  a.rows = static_cast<const double2*>(d_rows);
  a.cols = static_cast<const double2*>(d_cols);
  a.n_rows = n_rows;
  a.n_cols = n_cols;
  a.nb_rows = blocks_for(n_rows);
  a.nb_cols = blocks_for(n_cols);
  a.tile_begin = tile_begin;
  a.n_tiles = tile_end - tile_begin;
  a.out = d_out;
  a.ld_out = ld_out;
  a.final_scale = p.final_scale;
  a.n_pad = p.width_padded;
  a.nchunks = p.width_padded / kChunk;
  a.front = p.front_pad;
  a.convention = p.convention;
  a.pad_rows = sample_pad(n_rows);
  a.pad_cols = sample_pad(n_cols);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool packed = out_mode == QK_OUT_PACKED;
  if (p.layers == 2) {
    if (mode == kModeGram)
      return packed ? launch_sweep_t<2, kModeGram, QK_OUT_PACKED>(a, st)
                    : launch_sweep_t<2, kModeGram, QK_OUT_DENSE>(a, st);
    return packed ? launch_sweep_t<2, kModeCross, QK_OUT_PACKED>(a, st)
                  : launch_sweep_t<2, kModeCross, QK_OUT_DENSE>(a, st);
  }
  if (p.layers == 1) {
    if (mode == kModeGram)
      return packed ? launch_sweep_t<1, kModeGram, QK_OUT_PACKED>(a, st)
                    : launch_sweep_t<1, kModeGram, QK_OUT_DENSE>(a, st);
    return packed ? launch_sweep_t<1, kModeCross, QK_OUT_PACKED>(a, st)
                  : launch_sweep_t<1, kModeCross, QK_OUT_DENSE>(a, st);
  }
  switch (p.layers) {
    case 5: return launch_deep_t<4>(a, mode, packed, st);
    case 6: return launch_deep_t<5>(a, mode, packed, st);
    case 7: return launch_deep_t<6>(a, mode, packed, st);
    case 8: return launch_deep_t<7>(a, mode, packed, st);
    default: break;
  }
  if (p.layers == 4) {
    if (mode == kModeGram)
      return packed ? launch_general<4, kModeGram, QK_OUT_PACKED>(a, st)
                    : launch_general<4, kModeGram, QK_OUT_DENSE>(a, st);
    return packed ? launch_general<4, kModeCross, QK_OUT_PACKED>(a, st)
                  : launch_general<4, kModeCross, QK_OUT_DENSE>(a, st);
  }
  if (mode == kModeGram)
    return packed ? launch_general<3, kModeGram, QK_OUT_PACKED>(a, st)
                  : launch_general<3, kModeGram, QK_OUT_DENSE>(a, st);
  return packed ? launch_general<3, kModeCross, QK_OUT_PACKED>(a, st)
                : launch_general<3, kModeCross, QK_OUT_DENSE>(a, st);
}

qk_status launch_job(const Plan& p, const void* d_train, int64_t n_train, const void* d_test,
                     int64_t n_test, int64_t tile_begin, int64_t tile_end, double* d_K_train,
                     double* d_K_cross, void* stream, unsigned int* d_prog_train,
                     unsigned int* d_prog_cross, int64_t head_b, unsigned long long* counter,
                     bool pdl, int64_t rect_tail) {
  if (tile_end <= tile_begin) return QK_OK;
  if (head_b != 0 && (p.layers > 2 || head_b % kGroup != 0))
    return set_error(QK_ERR_VALUE, "Gram head order needs layers <= 2 and a multiple of 8");
  const int64_t nbt = blocks_for(n_train);
  const int64_t n_gram = nbt * (nbt + 1) / 2;
  if (p.layers >= 3 || n_test == 0 || tile_end <= n_gram || tile_begin >= n_gram) {
    // one problem only (or the one-pair-per-thread L >= 3 kernel): plain launches
    // (the caller's counter and programmatic launch go to the Gram launch, or to the cross
    // launch when the range holds no Gram tile)
    const bool gram_first = tile_begin < std::min(tile_end, n_gram);
    if (qk_status s = launch_sweep(p, kModeGram, d_train, n_train, d_train, n_train, tile_begin,
                                   std::min(tile_end, n_gram), d_K_train, n_train,
                                   QK_OUT_DENSE, stream, d_prog_train, head_b, counter, pdl))
      return s;
    if (n_test == 0 || tile_end <= n_gram) return QK_OK;
    return launch_sweep(p, kModeCross, d_test, n_test, d_train, n_train,
                        std::max(tile_begin, n_gram) - n_gram, tile_end - n_gram, d_K_cross,
                        n_train, QK_OUT_DENSE, stream, d_prog_cross, 0,
                        gram_first ? nullptr : counter, !gram_first && pdl, rect_tail);
  }
  SweepArgs a{};
  a.next_tile = counter;
  a.pdl = pdl ? 1 : 0;
  a.rect_tail = rect_tail < 0 ? kRectTail : rect_tail;
  a.head_b = head_b;
  a.rows = static_cast<const double2*>(d_train);
  a.cols = static_cast<const double2*>(d_train);
  a.n_rows = n_train;
  a.n_cols = n_train;
  a.nb_rows = nbt;
  a.nb_cols = nbt;
  a.tile_begin = tile_begin;
  a.n_tiles = tile_end - tile_begin;
  a.out = d_K_train;
  a.ld_out = n_train;
  a.final_scale = p.final_scale;
  a.n_pad = p.width_padded;
  a.nchunks = p.width_padded / kChunk;
  a.front = p.front_pad;
  a.convention = p.convention;
  a.progress = d_prog_train;
  a.rows2 = static_cast<const double2*>(d_test);
  a.n_rows2 = n_test;
  a.nb_rows2 = blocks_for(n_test);
  a.n_first = n_gram;
  a.out2 = d_K_cross;
  a.progress2 = d_prog_cross;
  a.pad_rows = a.pad_cols = sample_pad(n_train);
  a.pad_rows2 = sample_pad(n_test);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.layers == 2) return launch_sweep_t<2, kModeJob, QK_OUT_DENSE>(a, st);
  return launch_sweep_t<1, kModeJob, QK_OUT_DENSE>(a, st);
}

qk_status launch_unpack(const Plan& p, int mode, const double* d_packed, int64_t n_rows,
                        int64_t n_cols, int64_t tile_begin, int64_t tile_end, double* d_K,
                        int64_t ld, void* stream) {
  (void)p;
  if (tile_end <= tile_begin) return QK_OK;
  const int64_t nt = tile_end - tile_begin;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (mode == kModeGram)
    unpack_kernel<kModeGram><<<unsigned(nt), 256, 0, st>>>(
        d_packed, n_rows, n_rows, blocks_for(n_rows), blocks_for(n_rows), tile_begin, d_K, ld);
  else
    unpack_kernel<kModeCross><<<unsigned(nt), 256, 0, st>>>(
        d_packed, n_rows, n_cols, blocks_for(n_rows), blocks_for(n_cols), tile_begin, d_K, ld);
  return cuda_status(cudaGetLastError(), "unpack launch");
}

qk_status launch_pairs(const Plan& p, const void* d_a, int64_t n_a, const void* d_b, int64_t n_b,
                       const int64_t* d_pairs, int64_t n_pairs, double* d_amp, void* stream,
                       bool kernel_values) {
  const int value = kernel_values ? p.convention : -1;
  if (n_pairs == 0) return QK_OK;
  const unsigned grid = unsigned((n_pairs + 127) / 128);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nchunks = p.width_padded / kChunk;
  switch (p.layers) {
    case 5: return launch_pairs_deep<4>(p, d_a, n_a, d_b, n_b, d_pairs, n_pairs, d_amp, value, st);
    case 6: return launch_pairs_deep<5>(p, d_a, n_a, d_b, n_b, d_pairs, n_pairs, d_amp, value, st);
    case 7: return launch_pairs_deep<6>(p, d_a, n_a, d_b, n_b, d_pairs, n_pairs, d_amp, value, st);
    case 8: return launch_pairs_deep<7>(p, d_a, n_a, d_b, n_b, d_pairs, n_pairs, d_amp, value, st);
    default: break;
  }
  if (p.layers == 2)
    pairs_kernel<2><<<grid, 128, 0, st>>>(static_cast<const double2*>(d_a), n_a,
                                          static_cast<const double2*>(d_b), n_b, d_pairs,
                                          n_pairs, d_amp, p.width_padded, nchunks, p.front_pad,
                                          p.final_scale, value);
  else if (p.layers == 3)
    pairs_kernel<3><<<grid, 128, 0, st>>>(static_cast<const double2*>(d_a), n_a,
                                          static_cast<const double2*>(d_b), n_b, d_pairs,
                                          n_pairs, d_amp, p.width_padded, nchunks, p.front_pad,
                                          p.final_scale, value);
  else if (p.layers == 4)
    pairs_kernel<4><<<grid, 128, 0, st>>>(static_cast<const double2*>(d_a), n_a,
                                          static_cast<const double2*>(d_b), n_b, d_pairs,
                                          n_pairs, d_amp, p.width_padded, nchunks, p.front_pad,
                                          p.final_scale, value);
  else
    pairs_kernel<1><<<grid, 128, 0, st>>>(static_cast<const double2*>(d_a), n_a,
                                          static_cast<const double2*>(d_b), n_b, d_pairs,
                                          n_pairs, d_amp, p.width_padded, nchunks, p.front_pad,
                                          p.final_scale, value);
  return cuda_status(cudaGetLastError(), "pairs launch");
}

qk_status launch_dfma_peak(double* out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sms = sm_count();
  if (sms <= 0) return set_error(QK_ERR_CUDA, "no CUDA device");
  double* d_sink = nullptr;
  if (cudaError_t e = cudaMalloc(&d_sink, sizeof(double))) return cuda_status(e, "dfma malloc");
  const int blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_peak_kernel<<<blocks, 256, 0, st>>>(d_sink, 64);  // warm-up
  cudaEventRecord(e0, st);
  dfma_peak_kernel<<<blocks, 256, 0, st>>>(d_sink, iters);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_sink);
  if (e != cudaSuccess) return cuda_status(e, "dfma run");
  const double flops = double(blocks) * 256 * iters * 16 * 8 * 2;
  *out = flops / (double(ms) * 1e-3);
  return QK_OK;
}

}  // namespace qk

#ifdef QK_TIMELINE
extern "C" int qk_timeline_read(unsigned long long* host, int n_ctas, int clear) {
  const size_t bytes = size_t(n_ctas) * qk::kTLSlots * sizeof(unsigned long long);
  if (cudaMemcpyFromSymbol(host, qk::qk_tl_buf, bytes) != cudaSuccess) return 5;
  if (clear) {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, qk::qk_tl_buf);
    cudaMemset(p, 0, sizeof(unsigned long long) * 1024 * qk::kTLSlots);
  }
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 5;
}
#endif
