// qk_api.cu — C-ABI entry points of libqk: argument validation, launches, and the
// host-buffer pipelines behind compute_kernel_matrix / compute_cross_kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "qk_internal.h"

using namespace qk;

namespace {

qk_status cuda_err(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return QK_OK;
  cudaGetLastError();  // clear sticky-free errors
  return set_error(QK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Per-device workspace for the host-buffer entry points: device buffers grow monotonically,
// one non-blocking stream.  Guarded by a mutex: the host entry points are synchronous.
struct Workspace {
  std::mutex mu;
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t cap[4] = {0, 0, 0, 0};
  uint64_t* bad = nullptr;  // [2]: non-finite sample sentinels (rows, cols)

  qk_status ensure(int slot, size_t bytes) {
    if (cap[slot] >= bytes) return QK_OK;
    if (buf[slot]) cudaFree(buf[slot]);
    buf[slot] = nullptr;
    cap[slot] = 0;
    if (bytes == 0) return QK_OK;
    if (cudaError_t e = cudaMalloc(&buf[slot], bytes)) {
      return set_error(QK_ERR_CAPACITY, std::string("device allocation of ") +
                                            std::to_string(bytes) + " bytes failed: " +
                                            cudaGetErrorString(e));
    }
    cap[slot] = bytes;
    return QK_OK;
  }
};

Workspace g_ws[64];

qk_status workspace_for_current(Workspace** out, std::unique_lock<std::mutex>& lock) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_err(e, "cudaGetDevice");
  int count = 0;
  if (cudaError_t e = cudaGetDeviceCount(&count)) return cuda_err(e, "cudaGetDeviceCount");
  if (count == 0) return set_error(QK_ERR_CUDA, "no CUDA device");
  if (dev < 0 || dev >= 64) return set_error(QK_ERR_CUDA, "device index out of range");
  Workspace* w = &g_ws[dev];
  lock = std::unique_lock<std::mutex>(w->mu);
  if (w->device < 0) {
    if (cudaError_t e = cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking))
      return cuda_err(e, "stream create");
    if (cudaError_t e = cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking))
      return cuda_err(e, "stream create");
    if (cudaError_t e = cudaMalloc(&w->bad, 2 * sizeof(uint64_t))) return cuda_err(e, "malloc");
    w->device = dev;
  }
  *out = w;
  return QK_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Reads the non-finite sentinels written by the gate build (after the stream synced) and
// turns a hit into the reference's RebindError (network.py:295-296).
qk_status check_bad(const uint64_t* d_bad, int count, const char* const* names) {
  uint64_t h[2] = {UINT64_MAX, UINT64_MAX};
  if (cudaError_t e = cudaMemcpy(h, d_bad, count * sizeof(uint64_t), cudaMemcpyDeviceToHost))
    return cuda_err(e, "read non-finite sentinel");
  for (int k = 0; k < count; ++k)
    if (h[k] != UINT64_MAX)
      return set_error(QK_ERR_REBIND, std::string("feature angles must be finite (") + names[k] +
                                          " sample " + std::to_string(h[k]) + ")");
  return QK_OK;
}

}  // namespace

extern "C" {

qk_status qk_gate_build(const qk_plan* plan, const double* d_angles, int64_t n_samples,
                        int64_t ld, void* d_planes, uint64_t* d_bad_sample, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (n_samples < 0) return set_error(QK_ERR_VALUE, "n_samples must be >= 0");
  if (n_samples == 0) return QK_OK;
  if (ld < p->width)
    return set_error(QK_ERR_REBIND, "feature vectors of length " + std::to_string(ld) +
                                        " do not match width " + std::to_string(p->width));
  if (d_angles == nullptr || d_planes == nullptr)
    return set_error(QK_ERR_VALUE, "NULL device buffer");
  if (!aligned16(d_planes)) return set_error(QK_ERR_VALUE, "planes must be 16-byte aligned");
  return launch_gate_build(*p, d_angles, n_samples, ld, d_planes, d_bad_sample, stream);
}

qk_status qk_gram_tiles(const qk_plan* plan, const void* d_planes, int64_t n_samples,
                        int64_t tile_begin, int64_t tile_end, double* d_out, int32_t out_mode,
                        void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  const int64_t nt = qk_gram_tile_count(plan, n_samples);
  if (n_samples < 0 || tile_begin < 0 || tile_end < tile_begin || tile_end > nt)
    return set_error(QK_ERR_VALUE, "tile range [" + std::to_string(tile_begin) + ", " +
                                       std::to_string(tile_end) + ") outside [0, " +
                                       std::to_string(nt) + ")");
  if (out_mode != QK_OUT_DENSE && out_mode != QK_OUT_PACKED)
    return set_error(QK_ERR_VALUE, "unknown out_mode");
  if (tile_end == tile_begin) return QK_OK;
  if (d_planes == nullptr || d_out == nullptr) return set_error(QK_ERR_VALUE, "NULL buffer");
  if (!aligned16(d_planes)) return set_error(QK_ERR_VALUE, "planes must be 16-byte aligned");
  return launch_sweep(*p, kModeGram, d_planes, n_samples, d_planes, n_samples, tile_begin,
                      tile_end, d_out, n_samples, out_mode, stream);
}

qk_status qk_unpack_gram(const qk_plan* plan, const double* d_packed, int64_t n_samples,
                         int64_t tile_begin, int64_t tile_end, double* d_K, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  const int64_t nt = qk_gram_tile_count(plan, n_samples);
  if (tile_begin < 0 || tile_end < tile_begin || tile_end > nt)
    return set_error(QK_ERR_VALUE, "tile range outside the Gram tile list");
  if (tile_end == tile_begin) return QK_OK;
  if (d_packed == nullptr || d_K == nullptr) return set_error(QK_ERR_VALUE, "NULL buffer");
  return launch_unpack(*p, kModeGram, d_packed, n_samples, n_samples, tile_begin, tile_end, d_K,
                       n_samples, stream);
}

qk_status qk_cross_tiles(const qk_plan* plan, const void* d_planes_rows, int64_t n_rows,
                         const void* d_planes_cols, int64_t n_cols, int64_t tile_begin,
                         int64_t tile_end, double* d_out, int64_t ld_out, int32_t out_mode,
                         void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  const int64_t nt = qk_cross_tile_count(plan, n_rows, n_cols);
  if (n_rows < 0 || n_cols < 0 || tile_begin < 0 || tile_end < tile_begin || tile_end > nt)
    return set_error(QK_ERR_VALUE, "tile range outside the cross tile list");
  if (out_mode != QK_OUT_DENSE && out_mode != QK_OUT_PACKED)
    return set_error(QK_ERR_VALUE, "unknown out_mode");
  if (out_mode == QK_OUT_DENSE && ld_out < n_cols)
    return set_error(QK_ERR_VALUE, "ld_out < n_cols");
  if (tile_end == tile_begin) return QK_OK;
  if (!d_planes_rows || !d_planes_cols || !d_out) return set_error(QK_ERR_VALUE, "NULL buffer");
  if (!aligned16(d_planes_rows) || !aligned16(d_planes_cols))
    return set_error(QK_ERR_VALUE, "planes must be 16-byte aligned");
  return launch_sweep(*p, kModeCross, d_planes_rows, n_rows, d_planes_cols, n_cols, tile_begin,
                      tile_end, d_out, ld_out, out_mode, stream);
}

qk_status qk_unpack_cross(const qk_plan* plan, const double* d_packed, int64_t n_rows,
                          int64_t n_cols, int64_t tile_begin, int64_t tile_end, double* d_K,
                          int64_t ld, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  const int64_t nt = qk_cross_tile_count(plan, n_rows, n_cols);
  if (tile_begin < 0 || tile_end < tile_begin || tile_end > nt)
    return set_error(QK_ERR_VALUE, "tile range outside the cross tile list");
  if (ld < n_cols) return set_error(QK_ERR_VALUE, "ld < n_cols");
  if (tile_end == tile_begin) return QK_OK;
  if (d_packed == nullptr || d_K == nullptr) return set_error(QK_ERR_VALUE, "NULL buffer");
  return launch_unpack(*p, kModeCross, d_packed, n_rows, n_cols, tile_begin, tile_end, d_K, ld,
                       stream);
}

qk_status qk_pair_amplitudes(const qk_plan* plan, const void* d_planes_a, int64_t n_a,
                             const void* d_planes_b, int64_t n_b, const int64_t* d_pairs,
                             int64_t n_pairs, double* d_amp, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (n_pairs < 0 || n_a < 0 || n_b < 0) return set_error(QK_ERR_VALUE, "negative size");
  if (n_pairs == 0) return QK_OK;
  if (!d_planes_a || !d_planes_b || !d_pairs || !d_amp)
    return set_error(QK_ERR_VALUE, "NULL buffer");
  return launch_pairs(*p, d_planes_a, n_a, d_planes_b, n_b, d_pairs, n_pairs, d_amp, stream);
}

qk_status qk_dfma_peak(double* out_flops_per_s, void* stream) {
  if (out_flops_per_s == nullptr) return set_error(QK_ERR_VALUE, "NULL output");
  return launch_dfma_peak(out_flops_per_s, stream);
}

// ---- host-buffer pipelines -------------------------------------------------------------
// Inputs are copied H2D (pinned buffers DMA directly; pageable ones go through the driver's
// staging), the sweep runs on the workspace stream, and the result is copied back.  The
// Gram is produced in row panels so each panel's D2H overlaps the next panel's sweep.

qk_status qk_kernel_matrix_host(const qk_plan* plan, const double* h_angles, int64_t n_samples,
                                double* h_K) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (n_samples < 0) return set_error(QK_ERR_VALUE, "n_samples must be >= 0");
  if (n_samples == 0) return QK_OK;
  if (!h_angles || !h_K) return set_error(QK_ERR_VALUE, "NULL host buffer");
  Workspace* w;
  std::unique_lock<std::mutex> lock;
  if (qk_status s = workspace_for_current(&w, lock)) return s;
  const int64_t N = n_samples;
  const size_t xb = size_t(N) * p->width * sizeof(double);
  const size_t pb = qk_planes_bytes(plan, N);
  const size_t kb = size_t(N) * size_t(N) * sizeof(double);
  if (qk_status s = w->ensure(0, xb)) return s;
  if (qk_status s = w->ensure(1, pb)) return s;
  if (qk_status s = w->ensure(2, kb)) return s;
  double* dX = static_cast<double*>(w->buf[0]);
  double* dK = static_cast<double*>(w->buf[2]);
  cudaStream_t st = w->stream;
  if (cudaError_t e = cudaMemcpyAsync(dX, h_angles, xb, cudaMemcpyHostToDevice, st))
    return cuda_err(e, "H2D angles");
  if (cudaError_t e = cudaMemsetAsync(w->bad, 0xFF, sizeof(uint64_t), st))
    return cuda_err(e, "sentinel reset");
  if (qk_status s = launch_gate_build(*p, dX, N, p->width, w->buf[1], w->bad, st)) return s;

  // Row panels of whole tile rows; panel k's rows are final once panels 0..k have run
  // (row i's lower part is the mirror of earlier tile rows).
  const int64_t nb = blocks_for(N);
  const int64_t nt = nb * (nb + 1) / 2;
  const bool pinned = is_pinned(h_K);
  const int64_t panels = pinned ? std::min<int64_t>(nb, 8) : 1;
  auto row_off = [nb](int64_t r) { return r * nb - r * (r - 1) / 2; };
  std::vector<cudaEvent_t> evs;
  int64_t r0 = 0;
  for (int64_t k = 0; k < panels; ++k) {
    // split tile rows so each panel carries ~equal tile counts
    int64_t r1 = r0;
    const int64_t target = (nt * (k + 1)) / panels;
    while (r1 < nb && row_off(r1 + 1) <= target) ++r1;
    if (k == panels - 1) r1 = nb;
    if (r1 <= r0) continue;
    if (qk_status s = launch_sweep(*p, kModeGram, w->buf[1], N, w->buf[1], N, row_off(r0),
                                   row_off(r1), dK, N, QK_OUT_DENSE, st))
      return s;
    const int64_t i0 = r0 * kTile, i1 = std::min<int64_t>(r1 * kTile, N);
    if (pinned) {
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, st);
      cudaStreamWaitEvent(w->copy_stream, ev, 0);
      evs.push_back(ev);
      if (cudaError_t e = cudaMemcpyAsync(h_K + i0 * N, dK + i0 * N,
                                          size_t(i1 - i0) * N * sizeof(double),
                                          cudaMemcpyDeviceToHost, w->copy_stream))
        return cuda_err(e, "D2H kernel panel");
    }
    r0 = r1;
  }
  cudaError_t e = cudaSuccess;
  if (!pinned) e = cudaMemcpyAsync(h_K, dK, kb, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(w->copy_stream);
  for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
  if (e != cudaSuccess) return cuda_err(e, "kernel matrix pipeline");
  static const char* const names[1] = {"train"};
  return check_bad(w->bad, 1, names);
}

qk_status qk_cross_kernel_host(const qk_plan* plan, const double* h_rows, int64_t n_rows,
                               const double* h_cols, int64_t n_cols, double* h_K) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (n_rows < 0 || n_cols < 0) return set_error(QK_ERR_VALUE, "negative size");
  if (n_rows == 0 || n_cols == 0) return QK_OK;
  if (!h_rows || !h_cols || !h_K) return set_error(QK_ERR_VALUE, "NULL host buffer");
  Workspace* w;
  std::unique_lock<std::mutex> lock;
  if (qk_status s = workspace_for_current(&w, lock)) return s;
  const size_t xrb = size_t(n_rows) * p->width * sizeof(double);
  const size_t xcb = size_t(n_cols) * p->width * sizeof(double);
  const size_t prb = qk_planes_bytes(plan, n_rows);
  const size_t pcb = qk_planes_bytes(plan, n_cols);
  const size_t kb = size_t(n_rows) * size_t(n_cols) * sizeof(double);
  if (qk_status s = w->ensure(0, xrb + xcb)) return s;
  if (qk_status s = w->ensure(1, prb + pcb)) return s;
  if (qk_status s = w->ensure(2, kb)) return s;
  double* dXr = static_cast<double*>(w->buf[0]);
  double* dXc = dXr + size_t(n_rows) * p->width;
  char* dPr = static_cast<char*>(w->buf[1]);
  char* dPc = dPr + prb;
  double* dK = static_cast<double*>(w->buf[2]);
  cudaStream_t st = w->stream;
  cudaError_t e = cudaMemcpyAsync(dXr, h_rows, xrb, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dXc, h_cols, xcb, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_err(e, "H2D angles");
  if ((e = cudaMemsetAsync(w->bad, 0xFF, 2 * sizeof(uint64_t), st)) != cudaSuccess)
    return cuda_err(e, "sentinel reset");
  if (qk_status s = launch_gate_build(*p, dXr, n_rows, p->width, dPr, w->bad, st)) return s;
  if (qk_status s = launch_gate_build(*p, dXc, n_cols, p->width, dPc, w->bad + 1, st)) return s;
  const int64_t nbr = blocks_for(n_rows), nbc = blocks_for(n_cols);
  const bool pinned = is_pinned(h_K);
  const int64_t panels = pinned ? std::min<int64_t>(nbr, 8) : 1;
  std::vector<cudaEvent_t> evs;
  int64_t r0 = 0;
  for (int64_t k = 0; k < panels; ++k) {
    const int64_t r1 = (k == panels - 1) ? nbr : (nbr * (k + 1)) / panels;
    if (r1 <= r0) continue;
    if (qk_status s = launch_sweep(*p, kModeCross, dPr, n_rows, dPc, n_cols, r0 * nbc, r1 * nbc,
                                   dK, n_cols, QK_OUT_DENSE, st))
      return s;
    if (pinned) {
      const int64_t i0 = r0 * kTile, i1 = std::min<int64_t>(r1 * kTile, n_rows);
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, st);
      cudaStreamWaitEvent(w->copy_stream, ev, 0);
      evs.push_back(ev);
      e = cudaMemcpyAsync(h_K + i0 * n_cols, dK + i0 * n_cols,
                          size_t(i1 - i0) * n_cols * sizeof(double), cudaMemcpyDeviceToHost,
                          w->copy_stream);
      if (e != cudaSuccess) return cuda_err(e, "D2H cross panel");
    }
    r0 = r1;
  }
  if (!pinned) e = cudaMemcpyAsync(h_K, dK, kb, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(w->copy_stream);
  for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
  if (e != cudaSuccess) return cuda_err(e, "cross kernel pipeline");
  static const char* const names[2] = {"test", "train"};
  return check_bad(w->bad, 2, names);
}

}  // extern "C"
