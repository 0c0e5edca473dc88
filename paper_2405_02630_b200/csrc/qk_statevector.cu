// qk_statevector.cu — dense state-vector ground truth on the device.
//
// Restates the reference's brute-force simulator (statevector.py:17-70) for the kernel circuit
// of a pair (compose_kernel_circuit, circuit.py:150-157: build_feature_map(x_j), then the
// adjoint of build_feature_map(x_i)): every gate applied in the reference's order to |0..0>,
// little-endian (qubit q = bit q of the state index, statevector.py:3-4).  It is independent of
// the sweep's closed form — no cancellation, no rotated basis — and exists to check the sweep
// beyond the reference's 24-qubit guard.
//
// All gates of the family are real (RY and CNOT, circuit.py:94-108), so the complex128 state of
// the reference has an exactly-zero imaginary part throughout and a real fp64 state carries the
// same numbers.  Each RY update is rn(rn(m00*a) + rn(m01*b)) with no FMA contraction — the
// reference's complex multiply-add on zero imaginary parts — and the gate coefficients are the
// host libm's cos/sin of parameter/2 (what math.cos/math.sin return), so the amplitudes are
// bit-identical to the reference's simulate() on the same host image.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "qk_internal.h"

namespace qk {
namespace {

constexpr int kSvMaxWidth = 40;        // index arithmetic limit; memory is the caller's
constexpr int kSvSmemMaxWidth = 13;    // batched pairs: 2^13 doubles = 64 KB of shared memory

// RY(theta) on `qubit`: [[c, -s], [s, c]] on each amplitude pair differing in that bit
// (statevector.py:17-24).
__global__ void sv_ry_kernel(double* __restrict__ st, int64_t half, int qubit, double c,
                             double s) {
  const int64_t lo_mask = (int64_t(1) << qubit) - 1;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < half;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = ((t & ~lo_mask) << 1) | (t & lo_mask);
    const int64_t i1 = i0 | (int64_t(1) << qubit);
    const double a = st[i0], b = st[i1];
    st[i0] = __dadd_rn(__dmul_rn(c, a), __dmul_rn(-s, b));
    st[i1] = __dadd_rn(__dmul_rn(s, a), __dmul_rn(c, b));
  }
}

// CNOT(control, target): swap the amplitudes with control = 1 and target = 0 / 1
// (statevector.py:27-38).
__global__ void sv_cnot_kernel(double* __restrict__ st, int64_t quarter, int control,
                               int target) {
  const int lo = control < target ? control : target, hi = control < target ? target : control;
  const int64_t m_lo = (int64_t(1) << lo) - 1, m_hi = (int64_t(1) << hi) - 1;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < quarter;
       t += int64_t(gridDim.x) * blockDim.x) {
    // insert zero bits at positions lo and hi
    int64_t x = ((t & ~m_lo) << 1) | (t & m_lo);
    x = ((x & ~m_hi) << 1) | (x & m_hi);
    const int64_t i0 = x | (int64_t(1) << control);  // control 1, target 0
    const int64_t i1 = i0 | (int64_t(1) << target);  // control 1, target 1
    const double v = st[i0];
    st[i0] = st[i1];
    st[i1] = v;
  }
}

__global__ void sv_zero_kernel(double* __restrict__ st, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x)
    st[t] = t == 0 ? 1.0 : 0.0;
}

// One gate of the pair circuit: kind 0 = RY (c, s), 1 = CNOT (q, q + 1).
struct SvGate {
  int kind, q;
  double c, s;
};

// The pair circuit's gate list in the reference's order (circuit.py:121-157): per layer RY on
// every wire then the CNOT chain, for x_j; then the adjoint for x_i — reversed order, negated
// angles.  Coefficients are cos/sin(parameter / 2) exactly as gate_unitary computes them.
std::vector<SvGate> pair_circuit(int width, int layers, const double* xi, const double* xj) {
  std::vector<SvGate> g;
  g.reserve(size_t(2) * layers * (2 * width - 1));
  for (int l = 0; l < layers; ++l) {
    for (int q = 0; q < width; ++q) g.push_back({0, q, std::cos(xj[q] / 2), std::sin(xj[q] / 2)});
    for (int q = 0; q + 1 < width; ++q) g.push_back({1, q, 0.0, 0.0});
  }
  for (int l = 0; l < layers; ++l) {
    for (int q = width - 2; q >= 0; --q) g.push_back({1, q, 0.0, 0.0});
    for (int q = width - 1; q >= 0; --q) {
      const double p = -xi[q];
      g.push_back({0, q, std::cos(p / 2), std::sin(p / 2)});
    }
  }
  return g;
}

// Batched small widths: one CTA per pair, the whole state in shared memory, the gate
// coefficients of both samples precomputed on the host (per sample and qubit: cos/sin of x/2
// for the feature map of x_j, of -x/2 for the adjoint of x_i).
__global__ void __launch_bounds__(256) sv_pairs_kernel(int width, int layers,
                                                       const double4* __restrict__ coef_a,
                                                       const double4* __restrict__ coef_b,
                                                       const int64_t* __restrict__ pairs,
                                                       int64_t n_pairs, double* __restrict__ amp) {
  extern __shared__ double sv[];
  const int64_t dim = int64_t(1) << width;
  for (int64_t p = blockIdx.x; p < n_pairs; p += gridDim.x) {
    const double4* ci = coef_a + pairs[2 * p] * width;      // row sample: the adjoint
    const double4* cj = coef_b + pairs[2 * p + 1] * width;  // column sample: the feature map
    for (int64_t t = threadIdx.x; t < dim; t += blockDim.x) sv[t] = t == 0 ? 1.0 : 0.0;
    __syncthreads();
    auto ry = [&](int q, double c, double s) {
      const int64_t lo_mask = (int64_t(1) << q) - 1;
      for (int64_t t = threadIdx.x; t < dim / 2; t += blockDim.x) {
        const int64_t i0 = ((t & ~lo_mask) << 1) | (t & lo_mask);
        const int64_t i1 = i0 | (int64_t(1) << q);
        const double a = sv[i0], b = sv[i1];
        sv[i0] = __dadd_rn(__dmul_rn(c, a), __dmul_rn(-s, b));
        sv[i1] = __dadd_rn(__dmul_rn(s, a), __dmul_rn(c, b));
      }
      __syncthreads();
    };
    auto cnot = [&](int q) {  // control q, target q + 1
      const int64_t m_lo = (int64_t(1) << q) - 1;
      for (int64_t t = threadIdx.x; t < dim / 4; t += blockDim.x) {
        int64_t x = ((t & ~m_lo) << 2) | (t & m_lo);  // zero bits at q and q + 1
        const int64_t i0 = x | (int64_t(1) << q);
        const int64_t i1 = i0 | (int64_t(1) << (q + 1));
        const double v = sv[i0];
        sv[i0] = sv[i1];
        sv[i1] = v;
      }
      __syncthreads();
    };
    for (int l = 0; l < layers; ++l) {
      for (int q = 0; q < width; ++q) ry(q, cj[q].x, cj[q].y);
      for (int q = 0; q + 1 < width; ++q) cnot(q);
    }
    for (int l = 0; l < layers; ++l) {
      for (int q = width - 2; q >= 0; --q) cnot(q);
      for (int q = width - 1; q >= 0; --q) ry(q, ci[q].z, ci[q].w);
    }
    if (threadIdx.x == 0) amp[p] = sv[0];
    __syncthreads();
  }
}

qk_status sv_check(int32_t width, int32_t layers, int max_width) {
  if (width < 1) return set_error(QK_ERR_VALUE, "width must be >= 1");
  if (layers < 1) return set_error(QK_ERR_VALUE, "layers must be >= 1");
  if (width > max_width)
    return set_error(QK_ERR_CAPACITY, "state vector for " + std::to_string(width) +
                                          " qubits exceeds the " + std::to_string(max_width) +
                                          "-qubit guard");
  return QK_OK;
}

qk_status sv_finite(const double* x, int64_t count) {
  for (int64_t k = 0; k < count; ++k)
    if (!std::isfinite(x[k])) return set_error(QK_ERR_REBIND, "feature angles must be finite");
  return QK_OK;
}

qk_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return QK_OK;
  return set_error(QK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace
}  // namespace qk

using namespace qk;

extern "C" {

size_t qk_statevector_bytes(int32_t width) {
  if (width < 1 || width > kSvMaxWidth) return 0;
  return (size_t(1) << width) * sizeof(double);
}

qk_status qk_statevector_amplitude(int32_t width, int32_t layers, const double* x_i,
                                   const double* x_j, double* d_state, double* out_amp,
                                   void* stream) {
  if (qk_status s = sv_check(width, layers, kSvMaxWidth)) return s;
  if (x_i == nullptr || x_j == nullptr || d_state == nullptr || out_amp == nullptr)
    return set_error(QK_ERR_VALUE, "NULL argument");
  if (qk_status s = sv_finite(x_i, width)) return s;
  if (qk_status s = sv_finite(x_j, width)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t dim = int64_t(1) << width;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto grid = [&](int64_t work) {
    return int(std::min<int64_t>((work + 255) / 256, int64_t(sms) * 8));
  };
  sv_zero_kernel<<<grid(dim), 256, 0, st>>>(d_state, dim);
  for (const SvGate& g : pair_circuit(width, layers, x_i, x_j)) {
    if (g.kind == 0)
      sv_ry_kernel<<<grid(dim / 2), 256, 0, st>>>(d_state, dim / 2, g.q, g.c, g.s);
    else
      sv_cnot_kernel<<<grid(dim / 4), 256, 0, st>>>(d_state, dim / 4, g.q, g.q + 1);
  }
  if (qk_status s = cuda_status(cudaGetLastError(), "statevector launch")) return s;
  if (qk_status s = cuda_status(cudaMemcpyAsync(out_amp, d_state, sizeof(double),
                                                cudaMemcpyDeviceToHost, st),
                                "statevector D2H"))
    return s;
  return cuda_status(cudaStreamSynchronize(st), "statevector");
}

qk_status qk_statevector_pairs(int32_t width, int32_t layers, const double* h_a, int64_t n_a,
                               const double* h_b, int64_t n_b, const int64_t* h_pairs,
                               int64_t n_pairs, double* h_amp) {
  if (qk_status s = sv_check(width, layers, kSvSmemMaxWidth)) return s;
  if (n_a < 0 || n_b < 0 || n_pairs < 0) return set_error(QK_ERR_VALUE, "negative size");
  if (n_pairs == 0) return QK_OK;
  if (!h_a || !h_b || !h_pairs || !h_amp) return set_error(QK_ERR_VALUE, "NULL host buffer");
  for (int64_t p = 0; p < n_pairs; ++p)
    if (h_pairs[2 * p] < 0 || h_pairs[2 * p] >= n_a || h_pairs[2 * p + 1] < 0 ||
        h_pairs[2 * p + 1] >= n_b)
      return set_error(QK_ERR_VALUE, "pair " + std::to_string(p) + " indexes outside the sets");
  if (qk_status s = sv_finite(h_a, n_a * width)) return s;
  if (qk_status s = sv_finite(h_b, n_b * width)) return s;
  // (cos, sin) of x/2 (feature map) and of -x/2 (adjoint), host libm as gate_unitary
  auto coef = [&](const double* x, int64_t n) {
    std::vector<double> c(size_t(n) * width * 4);
    for (int64_t k = 0; k < n * width; ++k) {
      const double p = -x[k];
      c[4 * k + 0] = std::cos(x[k] / 2);
      c[4 * k + 1] = std::sin(x[k] / 2);
      c[4 * k + 2] = std::cos(p / 2);
      c[4 * k + 3] = std::sin(p / 2);
    }
    return c;
  };
  const std::vector<double> ca = coef(h_a, n_a), cb = coef(h_b, n_b);
  void *d_ca = nullptr, *d_cb = nullptr, *d_pairs = nullptr, *d_amp = nullptr;
  cudaError_t e = cudaMalloc(&d_ca, std::max<size_t>(ca.size(), 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_cb, std::max<size_t>(cb.size(), 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_pairs, size_t(n_pairs) * 16);
  if (e == cudaSuccess) e = cudaMalloc(&d_amp, size_t(n_pairs) * 8);
  if (e == cudaSuccess) e = cudaMemcpy(d_ca, ca.data(), ca.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_cb, cb.data(), cb.size() * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(d_pairs, h_pairs, size_t(n_pairs) * 16, cudaMemcpyHostToDevice);
  const size_t smem = (size_t(1) << width) * sizeof(double);
  if (e == cudaSuccess && smem > 48 * 1024)
    e = cudaFuncSetAttribute(sv_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
  if (e == cudaSuccess) {
    const int blocks = int(std::min<int64_t>(n_pairs, 148 * 16));
    sv_pairs_kernel<<<blocks, 256, smem>>>(width, layers, static_cast<const double4*>(d_ca),
                                           static_cast<const double4*>(d_cb),
                                           static_cast<const int64_t*>(d_pairs), n_pairs,
                                           static_cast<double*>(d_amp));
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpy(h_amp, d_amp, size_t(n_pairs) * 8, cudaMemcpyDeviceToHost);
  cudaFree(d_ca);
  cudaFree(d_cb);
  cudaFree(d_pairs);
  cudaFree(d_amp);
  return cuda_status(e, "statevector pairs");
}

}  // extern "C"
