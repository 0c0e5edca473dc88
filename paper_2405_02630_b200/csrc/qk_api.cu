// qk_api.cu — C-ABI entry points of libqk: argument validation, launches, and the
// host-buffer pipelines behind compute_kernel_matrix / compute_cross_kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
  cudaStream_t h2d_stream = nullptr;  // the rest's upload + sweep of the head-first pipeline
  // angles, planes, K, progress counters
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t cap[4] = {0, 0, 0, 0};
  uint64_t* bad = nullptr;  // [2]: non-finite sample sentinels (rows, cols)
  void* stage[2] = {nullptr, nullptr};  // pinned staging for pageable host buffers
  size_t stage_cap = 0;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  void* in_stage = nullptr;  // pinned copy of pageable angle arrays (head-first upload)
  size_t in_stage_cap = 0;

  qk_status ensure_in_stage(size_t bytes) {
    if (in_stage_cap >= bytes) return QK_OK;
    if (in_stage) cudaFreeHost(in_stage);
    in_stage = nullptr;
    in_stage_cap = 0;
    if (cudaError_t e = cudaHostAlloc(&in_stage, bytes, cudaHostAllocDefault))
      return set_error(QK_ERR_CAPACITY, std::string("pinned input staging allocation failed: ") +
                                            cudaGetErrorString(e));
    in_stage_cap = bytes;
    return QK_OK;
  }

  qk_status ensure_stage(size_t bytes) {
    if (stage_cap >= bytes) return QK_OK;
    for (int k = 0; k < 2; ++k) {
      if (stage[k]) cudaFreeHost(stage[k]);
      stage[k] = nullptr;
    }
    stage_cap = 0;
    for (int k = 0; k < 2; ++k) {
      if (cudaError_t e = cudaHostAlloc(&stage[k], bytes, cudaHostAllocDefault))
        return set_error(QK_ERR_CAPACITY, std::string("pinned staging allocation failed: ") +
                                              cudaGetErrorString(e));
      if (!stage_ev[k]) cudaEventCreateWithFlags(&stage_ev[k], cudaEventDisableTiming);
    }
    stage_cap = bytes;
    return QK_OK;
  }

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
    if (cudaError_t e = cudaStreamCreateWithFlags(&w->h2d_stream, cudaStreamNonBlocking))
      return cuda_err(e, "stream create");
    if (cudaError_t e = cudaMalloc(&w->bad, 2 * sizeof(uint64_t))) return cuda_err(e, "malloc");
    w->device = dev;
  }
  *out = w;
  return QK_OK;
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


// Small persistent pool for host-side memcpy between pageable user buffers and the pinned
// staging buffers (parallel copies also parallelise first-touch page faults).
class CopyPool {
 public:
  CopyPool() {
    unsigned n = std::thread::hardware_concurrency();
    n = std::max(1u, std::min(16u, n));
    for (unsigned k = 0; k < n; ++k) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // copies n bytes src -> dst in parallel; blocks until done
  void copy(void* dst, const void* src, size_t n) { run(dst, src, n); }
  // writes one byte of every 4 KB page of [dst, dst + n) in parallel: a fresh (never touched)
  // pageable output buffer takes its page faults here, while the GPU is busy, instead of
  // inside the drain copies that trail the sweep
  void touch(void* dst, size_t n) { run(dst, nullptr, n); }

 private:
  // Copies with non-temporal (streaming) stores: the destination lines go to DRAM instead of
  // sitting dirty in the host's last-level cache.  For the pinned input stage this matters on
  // the GPU side: a DMA read of cache-resident dirty lines ran at ~25 GB/s instead of ~55
  // (measured: the config-4 rest upload took 2.8-3.3 ms instead of 1.3 whenever nothing else
  // had pushed the staged angles out of the 60 MB L3); for the user's output buffers it also
  // skips the read-for-ownership of every destination line.
  static void stream_copy(char* d, const char* s, size_t n) {
    size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
    if (head > n) head = n;
    std::memcpy(d, s, head);
    d += head, s += head, n -= head;
    const size_t v = n / 64;
    for (size_t k = 0; k < v; ++k, d += 64, s += 64) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
      const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
    }
    std::memcpy(d, s, n - v * 64);
    _mm_sfence();
  }
  static void work(char* d, const char* sp, size_t lo, size_t hi) {
    if (sp != nullptr) {
      stream_copy(d + lo, sp + lo, hi - lo);
      return;
    }
    for (size_t o = (lo + 4095) & ~size_t(4095); o < hi; o += 4096)
      *reinterpret_cast<volatile char*>(d + o) = 0;
  }
  void run(void* dst, const void* src, size_t n) {
    const size_t parts = std::min<size_t>(workers_.size(), std::max<size_t>(1, n >> 20));
    if (parts <= 1) {
      work(static_cast<char*>(dst), static_cast<const char*>(src), 0, n);
      return;
    }
    std::lock_guard<std::mutex> one_caller(call_mu_);
    std::unique_lock<std::mutex> g(mu_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    n_ = n;
    parts_ = parts;
    next_ = 0;
    done_ = 0;
    ++gen_;
    cv_.notify_all();
    done_cv_.wait(g, [this] { return done_ == parts_; });
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> g(mu_);
    for (;;) {
      cv_.wait(g, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      while (next_ < parts_) {
        const size_t k = next_++;
        const size_t lo = n_ * k / parts_, hi = n_ * (k + 1) / parts_;
        char* d = dst_;
        const char* sp = src_;
        g.unlock();
        work(d, sp, lo, hi);
        g.lock();
        if (++done_ == parts_) done_cv_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  bool stop_ = false;
  uint64_t gen_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0, parts_ = 0, next_ = 0, done_ = 0;
};

CopyPool& copy_pool() {
  static CopyPool pool;
  return pool;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Host -> device on w->stream: pinned sources DMA directly; pageable ones go through the
// pinned staging pair (parallel memcpy into one slot while the other is in flight).
qk_status upload(Workspace* w, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return QK_OK;
  if (is_pinned(src))
    return cuda_err(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, w->stream), "H2D");
  const size_t chunk = size_t(64) << 20;
  if (qk_status s = w->ensure_stage(chunk)) return s;
  size_t k = 0;
  for (size_t off = 0; off < bytes; off += chunk, ++k) {
    const int slot = int(k & 1);
    const size_t n = std::min(chunk, bytes - off);
    cudaEventSynchronize(w->stage_ev[slot]);  // the slot's previous DMA (any call) is done
    copy_pool().copy(w->stage[slot], static_cast<const char*>(src) + off, n);
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, w->stage[slot], n,
                                    cudaMemcpyHostToDevice, w->stream);
    if (e != cudaSuccess) return cuda_err(e, "H2D staged");
    cudaEventRecord(w->stage_ev[slot], w->stream);
  }
  return QK_OK;
}

}  // namespace

extern "C" {

qk_status qk_set_device(int32_t device) {
  return cuda_err(cudaSetDevice(device), "cudaSetDevice");
}

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

qk_status qk_job_run(const qk_plan* plan, const double* d_train, int64_t n_train,
                     const double* d_test, int64_t n_test, void* d_planes_train,
                     void* d_planes_test, uint64_t* d_state, int64_t tile_begin,
                     int64_t tile_end, double* d_K_train, double* d_K_cross, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  const int64_t nt = qk_job_tile_count(plan, n_train, n_test);
  if (n_train < 0 || n_test < 0 || tile_begin < 0 || tile_end < tile_begin || tile_end > nt)
    return set_error(QK_ERR_VALUE, "tile range outside the job tile list");
  if (n_train == 0) return QK_OK;
  if (!d_train || !d_planes_train || !d_state || !d_K_train ||
      (n_test > 0 && (!d_test || !d_planes_test || !d_K_cross)))
    return set_error(QK_ERR_VALUE, "NULL buffer");
  if (!aligned16(d_planes_train) || (n_test > 0 && !aligned16(d_planes_test)))
    return set_error(QK_ERR_VALUE, "planes must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // sentinels and the sweep's claim counter (all-ones = no claim yet) in one memset, ahead
  // of the gate build, so the sweep can follow the gate build as a programmatic dependent
  // launch (its prologue overlaps the build's tail)
  if (cudaError_t e = cudaMemsetAsync(d_state, 0xFF, QK_JOB_STATE_WORDS * sizeof(uint64_t), st))
    return cuda_err(e, "job state reset");
  if (qk_status s = launch_gate_build2(*p, d_train, n_train, d_planes_train, d_state, d_test,
                                       n_test, d_planes_test, d_state + 1, st))
    return s;
  if (tile_end == tile_begin) return QK_OK;
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(d_state + 2);
  return launch_job(*p, d_planes_train, n_train, d_planes_test, n_test, tile_begin, tile_end,
                    d_K_train, d_K_cross, st, nullptr, nullptr, 0, ctr, true);
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

qk_status qk_pair_kernel_values(const qk_plan* plan, const void* d_planes_a, int64_t n_a,
                                const void* d_planes_b, int64_t n_b, const int64_t* d_pairs,
                                int64_t n_pairs, double* d_K, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (n_pairs < 0 || n_a < 0 || n_b < 0) return set_error(QK_ERR_VALUE, "negative size");
  if (n_pairs == 0) return QK_OK;
  if (!d_planes_a || !d_planes_b || !d_pairs || !d_K) return set_error(QK_ERR_VALUE, "NULL buffer");
  return launch_pairs(*p, d_planes_a, n_a, d_planes_b, n_b, d_pairs, n_pairs, d_K, stream, true);
}

qk_status qk_dfma_peak(double* out_flops_per_s, void* stream) {
  if (out_flops_per_s == nullptr) return set_error(QK_ERR_VALUE, "NULL output");
  return launch_dfma_peak(out_flops_per_s, stream);
}

// ---- host-buffer pipelines -------------------------------------------------------------
// H2D of the angles, gate build, ONE persistent sweep launch over every tile, and the D2H of
// the result overlapped with the sweep: the kernel counts finished tiles per tile row and a
// copy stream waits on the counters (cuStreamWaitValue32) of a row panel before copying it
// out.  A Gram row is final once its own and all earlier tile rows are done (its lower part
// mirrors earlier tile rows), and the waits are queued in row order.  Without stream memory
// operations the D2H follows the sweep.

}  // extern "C"

namespace {

typedef int (*StreamWaitValue32Fn)(cudaStream_t, uintptr_t, uint32_t, unsigned int);
typedef int (*StreamBatchMemOpFn)(cudaStream_t, unsigned int, CUstreamBatchMemOpParams*,
                                  unsigned int);

// cuStreamBatchMemOp: a drain panel's row-counter waits as ONE stream command (measured: eight
// separate cuStreamWaitValue32 per Gram super-row cost ~15-20 us of copy-stream time per panel).
StreamBatchMemOpFn stream_batch_mem_op() {
  static StreamBatchMemOpFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    const char* v = getenv("QK_BATCH_WAITS");  // tuning: 0 = one command per wait
    if ((v != nullptr && v[0] == '0') ||
        cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return StreamBatchMemOpFn(nullptr);
    }
    return reinterpret_cast<StreamBatchMemOpFn>(p);
  }();
  return fn;
}

// Waits on `cs` until counter[r] >= expect(r) for every r in [r0, r1) (GEQ); 0 on success.
template <class Expect>
int wait_rows(StreamWaitValue32Fn wait, cudaStream_t cs, const unsigned int* counter, int64_t r0,
              int64_t r1, Expect expect) {
  StreamBatchMemOpFn batch = stream_batch_mem_op();
  if (batch != nullptr && r1 - r0 > 1) {
    CUstreamBatchMemOpParams ops[16];
    for (int64_t r = r0; r < r1;) {
      const int n = int(std::min<int64_t>(16, r1 - r));
      for (int k = 0; k < n; ++k) {
        std::memset(&ops[k], 0, sizeof(ops[k]));
        ops[k].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
        ops[k].waitValue.address = CUdeviceptr(reinterpret_cast<uintptr_t>(counter + r + k));
        ops[k].waitValue.value = expect(r + k);
        ops[k].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
      }
      if (batch(cs, unsigned(n), ops, 0) != 0) return 1;
      r += n;
    }
    return 0;
  }
  for (int64_t r = r0; r < r1; ++r)
    if (wait(cs, reinterpret_cast<uintptr_t>(counter + r), expect(r), 0x0) != 0) return 1;
  return 0;
}

StreamWaitValue32Fn stream_wait_value32() {
  static StreamWaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return StreamWaitValue32Fn(nullptr);
    }
    return reinterpret_cast<StreamWaitValue32Fn>(p);
  }();
  return fn;
}

// Head-first overlap of the input upload (pinned inputs, L = 2, the default host pipeline;
// QK_HEAD_SPLIT=0 turns it off): the angles of the first B plane blocks go up and are
// gate-built, the sweep runs the B x B Gram head (decode_gram orders it first) while the rest
// of the angles upload on the h2d stream, then the rest is gate-built and swept.  B is the
// smallest multiple of kGroup whose head keeps the GPU busy for as long as the remaining
// upload takes (estimates: ~0.6 us per tile per qubit on 148 SMs, ~50 GB/s of H2D from pinned
// buffers; ~35 GB/s for pageable ones, which the host copy pool stages into pinned memory
// chunk by chunk, each chunk's DMA overlapping the next chunk's staging).
bool head_split_enabled(const Plan& p) {
  const char* v = getenv("QK_HEAD_SPLIT");
  return !(v != nullptr && v[0] == '0') && p.layers == 2;
}

int64_t choose_head(const Plan& p, int64_t n_train, int64_t n_test, double bw_bytes_per_ms) {
  if (!head_split_enabled(p)) return 0;
  const int64_t nb = blocks_for(n_train), pad = sample_pad(n_train);
  const double tile_ms = 6e-4 * p.width;
  for (int64_t B = kGroup; B + kGroup <= nb; B += kGroup) {
    const int64_t s1 = std::min<int64_t>(n_train, B * kTile - pad);
    const double rest_ms = double((n_train - s1) + n_test) * p.width * 8 / bw_bytes_per_ms;
    const double head_ms = double(B * (B + 1) / 2) / 148.0 * tile_ms;
    if (rest_ms < 0.05) return 0;  // nothing worth hiding
    if (head_ms >= rest_ms) return B;
  }
  return 0;
}

// Cross tile order of a host-pipeline sweep: grouped super-rows (kRectTail row-major tail rows)
// when the result drains into pinned memory; fully row-major when it drains into pageable
// memory, whose host-side copies (~12 GB/s) must start on each tile row as it finishes to keep
// pace with the sweep (grouped rows finish 8 at a time: config 4's pageable call measured
// 57.1 -> 58.2 ms with them).  The order only changes which tiles share L2, not the results.
static int64_t rect_tail_for(const void* h_out) { return is_pinned(h_out) ? -1 : INT64_MAX; }

// One row-major result matrix a sweep launch fills and the copy stream drains to the host.
struct DrainTarget {
  double* d_K;
  double* h_K;
  int64_t n_rows, n_cols;
  int mode;              // kModeGram or kModeCross: how tiles map onto super-rows
  unsigned int* d_prog;  // per-tile-row finished-tile counters (set by run_and_drain)
};

// Resets the progress counters, runs `launch` (which must pass targets[k].d_prog to the
// sweep) on w->stream, and copies each target's row panels (1 or kGroup tile rows) to the host
// on w->copy_stream as soon as their counters are complete — targets in order, panels in
// row order, matching the order in which the persistent sweep finishes tiles.
// QK_TRACE=1: timestamps of the host pipelines' phases on stderr (diagnostics only).
struct Trace {
  cudaEvent_t ev[6] = {};
  bool on = false;
  explicit Trace(cudaStream_t st) {
    const char* v = getenv("QK_TRACE");
    on = v != nullptr && v[0] == '1';
    if (!on) return;
    for (auto& e : ev) cudaEventCreate(&e);
    mark(0, st);
  }
  void mark(int k, cudaStream_t st) {
    if (on) cudaEventRecord(ev[k], st);
  }
  // named device event (ms after ev[0] on the device) and host timestamp (ms after the trace
  // started on the host), printed on a second line
  void point(const char* name, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    pts.push_back({name, e});
  }
  void host(const char* name) {
    if (on)
      hpts.push_back({name, std::chrono::duration<double, std::milli>(
                                std::chrono::steady_clock::now() - t0).count()});
  }
  ~Trace() {
    if (!on) return;
    cudaEventSynchronize(ev[5]);
    float t[5];
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]);
    fprintf(stderr, "qk_trace h2d %.3f gate %.3f sweep %.3f tail %.3f host %.3f ms\n", t[0],
            t[1], t[2], t[3], t[4]);
    if (!pts.empty() || !hpts.empty()) {
      fprintf(stderr, "qk_trace2");
      for (auto& p : pts) {
        float ms = 0;
        cudaEventSynchronize(p.second);
        cudaEventElapsedTime(&ms, ev[0], p.second);
        fprintf(stderr, " dev:%s=%.3f", p.first, ms);
        cudaEventDestroy(p.second);
      }
      for (auto& h : hpts) fprintf(stderr, " host:%s=%.3f", h.first, h.second);
      fprintf(stderr, "\n");
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
  std::vector<std::pair<const char*, cudaEvent_t>> pts;
  std::vector<std::pair<const char*, double>> hpts;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
};

template <class Launch>
qk_status run_and_drain(Workspace* w, const Plan& p, DrainTarget* tg, int n_targets,
                        Launch&& launch, Trace* trace = nullptr) {
  StreamWaitValue32Fn wait = stream_wait_value32();
  int64_t n_rows_total = 0;  // one counter per tile row
  bool all_pinned = true;
  for (int k = 0; k < n_targets; ++k) {
    n_rows_total += blocks_for(tg[k].n_rows);
    all_pinned = all_pinned && is_pinned(tg[k].h_K);
  }
  // panel height in tile rows: pinned outputs drain per tile row (small tail); pageable ones
  // per super-row so each staged copy-pool pass moves a few tens of MB
  const int64_t panel_rows = all_pinned ? 1 : kGroup;
  size_t panel_bytes = 0;
  for (int k = 0; k < n_targets; ++k)
    panel_bytes = std::max(panel_bytes, size_t(panel_rows) * kTile * tg[k].n_cols * 8);
  if (!all_pinned)
    if (qk_status s = w->ensure_stage(panel_bytes)) return s;
  if (wait != nullptr) {
    if (qk_status s = w->ensure(3, size_t(n_rows_total) * sizeof(unsigned int))) return s;
    unsigned int* base = static_cast<unsigned int*>(w->buf[3]);
    if (cudaError_t e = cudaMemsetAsync(base, 0, size_t(n_rows_total) * 4, w->stream))
      return cuda_err(e, "progress reset");
    for (int k = 0; k < n_targets; ++k) {
      tg[k].d_prog = base;
      base += blocks_for(tg[k].n_rows);
    }
  } else {
    for (int k = 0; k < n_targets; ++k) tg[k].d_prog = nullptr;
  }
  // the copy stream may start waiting on the counters once they are reset (NOT once the
  // sweep finished: the event is recorded before the launch)
  cudaEvent_t reset;
  cudaEventCreateWithFlags(&reset, cudaEventDisableTiming);
  cudaEventRecord(reset, w->stream);
  if (trace) trace->mark(2, w->stream);
  if (qk_status s = launch()) {
    cudaEventDestroy(reset);
    return s;
  }
  if (!all_pinned) {  // pageable outputs: take their page faults while the sweep runs
    cudaStreamQuery(w->stream);
    for (int k = 0; k < n_targets; ++k)
      if (!is_pinned(tg[k].h_K))
        copy_pool().touch(tg[k].h_K, size_t(tg[k].n_rows) * tg[k].n_cols * sizeof(double));
  }
  if (trace) trace->mark(3, w->stream);
  if (trace) trace->host("touched");
  cudaStream_t cs = w->copy_stream;
  if (!all_pinned) {  // the staging slots may still feed the H2D of the inputs
    for (int k = 0; k < 2; ++k)
      if (w->stage_ev[k]) cudaStreamWaitEvent(cs, w->stage_ev[k], 0);
  }
  if (wait != nullptr) {
    cudaStreamWaitEvent(cs, reset, 0);
  } else {
    cudaEvent_t fin;  // no stream memory ops: drain after the sweep
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(fin, w->stream);
    cudaStreamWaitEvent(cs, fin, 0);
    cudaEventDestroy(fin);
  }
  cudaStreamQuery(w->stream);  // flush the launch to the device before host-blocking work
  // flat list of panels (target, tile rows [r0, r1)), in the order the sweep finishes them:
  // panel_rows tile rows each, except that the LAST target's final kGroup tile rows go out one
  // tile row at a time, so the copy that trails the sweep is one 64-row panel
  struct Panel {
    int k;
    int64_t r0, r1;
  };
  std::vector<Panel> panels;
  for (int k = 0; k < n_targets; ++k) {
    const int64_t nbr = blocks_for(tg[k].n_rows);
    const int64_t fine_from = k == n_targets - 1 ? std::max<int64_t>(0, nbr - kGroup) : nbr;
    for (int64_t r0 = 0; r0 < nbr;) {
      const int64_t step = r0 >= fine_from ? 1 : panel_rows;
      const int64_t r1 = std::min(std::min(r0 + step, nbr), r0 < fine_from ? fine_from : nbr);
      panels.push_back({k, r0, r1});
      r0 = r1;
    }
  }
  const uint32_t unit = progress_unit(p.layers);
  auto rows_of = [&](const Panel& pn, int64_t& i0, int64_t& i1) {
    // sample rows of the panel (the front padding of block 0 is not a sample)
    const int64_t pad = sample_pad(tg[pn.k].n_rows);
    i0 = std::max<int64_t>(0, pn.r0 * kTile - pad);
    i1 = std::min<int64_t>(pn.r1 * kTile - pad, tg[pn.k].n_rows);
  };
  auto enqueue = [&](size_t idx, void* dst) -> cudaError_t {
    const Panel& pn = panels[idx];
    const DrainTarget& t = tg[pn.k];
    if (t.d_prog != nullptr) {  // every tile row of the panel is complete
      const int64_t nbr = blocks_for(t.n_rows), nbc = blocks_for(t.n_cols);
      if (wait_rows(wait, cs, t.d_prog, pn.r0, pn.r1, [&](int64_t r) {
            return unit * uint32_t(t.mode == kModeGram ? nbr - r : nbc);
          }) != 0)
        return cudaErrorNotSupported;
    }
    int64_t i0, i1;
    rows_of(pn, i0, i1);
    return cudaMemcpyAsync(dst, t.d_K + i0 * t.n_cols,
                           size_t(i1 - i0) * t.n_cols * sizeof(double), cudaMemcpyDeviceToHost,
                           cs);
  };
  cudaError_t e = cudaSuccess;
  const size_t np = panels.size();
  if (all_pinned) {
    // Straight into the user's pinned matrix.  Cross targets: one 64-row panel per tile row.
    // Gram targets: per super-row R (tile rows r0..r1-1, which the grouped tile order finishes
    // together), its rows from column block r0 on, and the strip of all LATER rows in column
    // blocks r0..r1-1 (mirrors of R's tiles).  Each step then ships data in proportion to the
    // tiles it waited for, so the D2H keeps pace with the sweep to the end instead of piling
    // up behind the short last tile rows (whole row panels: ~1.4 ms tail at 10,000 samples).
    for (int k = 0; k < n_targets && e == cudaSuccess; ++k) {
      const DrainTarget& t = tg[k];
      const int64_t nbr = blocks_for(t.n_rows);
      const int64_t pad_r = sample_pad(t.n_rows), pad_c = sample_pad(t.n_cols);
      auto row_lo = [&](int64_t b) {
        return std::min(std::max<int64_t>(b * kTile - pad_r, 0), t.n_rows);
      };
      auto col_lo = [&](int64_t b) {
        return std::min(std::max<int64_t>(b * kTile - pad_c, 0), t.n_cols);
      };
      auto copy = [&](int64_t i0, int64_t i1, int64_t c0, int64_t c1) -> cudaError_t {
        if (i1 <= i0 || c1 <= c0) return cudaSuccess;
        const size_t pitch = size_t(t.n_cols) * sizeof(double);
        return cudaMemcpy2DAsync(t.h_K + i0 * t.n_cols + c0, pitch, t.d_K + i0 * t.n_cols + c0,
                                 pitch, size_t(c1 - c0) * sizeof(double), size_t(i1 - i0),
                                 cudaMemcpyDeviceToHost, cs);
      };
      const bool gram = t.mode == kModeGram;
      // cross panels: whole tile rows, but at least ~2 MB per copy (small jobs: a 64-row
      // copy of a narrow matrix is latency-bound)
      const int64_t row_bytes = kTile * t.n_cols * int64_t(sizeof(double));
      const int64_t step = gram ? kGroup : std::max<int64_t>(1, ((2 << 20) + row_bytes - 1) /
                                                                    row_bytes);
      for (int64_t r0 = 0; r0 < nbr && e == cudaSuccess; r0 += step) {
        const int64_t r1 = std::min(r0 + step, nbr);
        if (t.d_prog != nullptr && wait_rows(wait, cs, t.d_prog, r0, r1, [&](int64_t q) {
              return unit * uint32_t(gram ? nbr - q : blocks_for(t.n_cols));
            }) != 0)
          e = cudaErrorNotSupported;
        if (e != cudaSuccess) break;
        static const char* const kReady[2][4] = {{"g0_ready", "g1_ready", "g2_ready", "g3_ready"},
                                                 {"x0_ready", "x1_ready", "x2_ready", "x3_ready"}};
        static const char* const kCopied[2][4] = {{"g0_copied", "g1_copied", "g2_copied",
                                                   "g3_copied"},
                                                  {"x0_copied", "x1_copied", "x2_copied",
                                                   "x3_copied"}};
        const int64_t pi = r0 / step;  // first and last panels of each target traced
        const int ti = pi < 2 ? int(pi) : (r1 == nbr ? 3 : (r1 + step >= nbr ? 2 : -1));
        if (trace && ti >= 0) trace->point(kReady[gram ? 0 : 1][ti], cs);
        if (!gram || t.d_prog == nullptr) {
          e = copy(row_lo(r0), row_lo(r1), 0, t.n_cols);
        } else {
          e = copy(row_lo(r0), row_lo(r1), col_lo(r0), t.n_cols);
          if (e == cudaSuccess) e = copy(row_lo(r1), t.n_rows, col_lo(r0), col_lo(r1));
        }
        if (trace && ti >= 0) trace->point(kCopied[gram ? 0 : 1][ti], cs);
      }
    }
  } else {
    // two pinned slots: DMA panel idx+2 while the pool copies panel idx into the user buffer
    for (size_t idx = 0; idx < std::min<size_t>(2, np) && e == cudaSuccess; ++idx) {
      e = enqueue(idx, w->stage[idx & 1]);
      if (e == cudaSuccess) e = cudaEventRecord(w->stage_ev[idx & 1], cs);
    }
    static const char* const kLanded[4] = {"p-4_landed", "p-3_landed", "p-2_landed",
                                           "p-1_landed"};
    static const char* const kCopied[4] = {"p-4_copied", "p-3_copied", "p-2_copied",
                                           "p-1_copied"};
    for (size_t idx = 0; idx < np && e == cudaSuccess; ++idx) {
      const int slot = int(idx & 1);
      e = cudaEventSynchronize(w->stage_ev[slot]);
      if (e != cudaSuccess) break;
      const int last = int(np - 1 - idx);  // trace the last four panels (host side)
      if (trace && last < 4) trace->host(kLanded[3 - last]);
      const DrainTarget& t = tg[panels[idx].k];
      int64_t i0, i1;
      rows_of(panels[idx], i0, i1);
      copy_pool().copy(t.h_K + i0 * t.n_cols, w->stage[slot],
                       size_t(i1 - i0) * t.n_cols * sizeof(double));
      if (trace && last < 4) trace->host(kCopied[3 - last]);
      if (idx + 2 < np) {
        e = enqueue(idx + 2, w->stage[slot]);
        if (e == cudaSuccess) e = cudaEventRecord(w->stage_ev[slot], cs);
      }
    }
  }
  if (trace) trace->mark(4, cs);
  if (trace) trace->host("drain_enqueued");
  cudaError_t e2 = cudaStreamSynchronize(w->stream);
  cudaError_t e3 = cudaStreamSynchronize(cs);
  if (trace) trace->mark(5, cs);
  cudaEventDestroy(reset);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = e3;
  return cuda_err(e, "sweep/D2H pipeline");
}

}  // namespace

extern "C" {

qk_status qk_kernel_matrix_host(const qk_plan* plan, const double* h_angles, int64_t n_samples,
                                double* h_K) {
  // the train Gram alone is the joint pipeline without a test set (same drain, same head-first
  // upload overlap for pinned inputs)
  if (n_samples < 0) return set_error(QK_ERR_VALUE, "n_samples must be >= 0");
  return qk_kernel_matrices_host(plan, h_angles, n_samples, nullptr, 0, h_K, nullptr);
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
  if (qk_status s = w->ensure(0, xrb + xcb)) return s;
  if (qk_status s = w->ensure(1, prb + pcb)) return s;
  if (qk_status s = w->ensure(2, size_t(n_rows) * size_t(n_cols) * sizeof(double))) return s;
  double* dXr = static_cast<double*>(w->buf[0]);
  double* dXc = dXr + size_t(n_rows) * p->width;
  char* dPr = static_cast<char*>(w->buf[1]);
  char* dPc = dPr + prb;
  cudaStream_t st = w->stream;
  Trace trace(st);
  if (qk_status s = upload(w, dXr, h_rows, xrb)) return s;
  if (qk_status s = upload(w, dXc, h_cols, xcb)) return s;
  trace.mark(1, st);
  if (cudaError_t e = cudaMemsetAsync(w->bad, 0xFF, 2 * sizeof(uint64_t), st))
    return cuda_err(e, "sentinel reset");
  if (qk_status s = launch_gate_build2(*p, dXr, n_rows, dPr, w->bad, dXc, n_cols, dPc,
                                       w->bad + 1, st))
    return s;
  DrainTarget tg[1] = {
      {static_cast<double*>(w->buf[2]), h_K, n_rows, n_cols, kModeCross, nullptr}};
  if (qk_status s = run_and_drain(w, *p, tg, 1, [&] {
        return launch_sweep(*p, kModeCross, dPr, n_rows, dPc, n_cols, 0,
                            qk_cross_tile_count(plan, n_rows, n_cols), tg[0].d_K, n_cols,
                            QK_OUT_DENSE, w->stream, tg[0].d_prog, 0, nullptr, false,
                            rect_tail_for(h_K));
      }, &trace))
    return s;
  static const char* const names[2] = {"test", "train"};
  return check_bad(w->bad, 2, names);
}

qk_status qk_kernel_matrices_host(const qk_plan* plan, const double* h_train, int64_t n_train,
                                  const double* h_test, int64_t n_test, double* h_K_train,
                                  double* h_K_cross) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (n_train < 0 || n_test < 0) return set_error(QK_ERR_VALUE, "negative size");
  if (n_train == 0) return QK_OK;
  if (!h_train || !h_K_train || (n_test > 0 && (!h_test || !h_K_cross)))
    return set_error(QK_ERR_VALUE, "NULL host buffer");
  Workspace* w;
  std::unique_lock<std::mutex> lock;
  if (qk_status s = workspace_for_current(&w, lock)) return s;
  const size_t xtb = size_t(n_train) * p->width * sizeof(double);
  const size_t xsb = size_t(n_test) * p->width * sizeof(double);
  const size_t ptb = qk_planes_bytes(plan, n_train);
  const size_t psb = qk_planes_bytes(plan, n_test);
  const size_t ktb = size_t(n_train) * size_t(n_train) * sizeof(double);
  const size_t ksb = size_t(n_test) * size_t(n_train) * sizeof(double);
  if (qk_status s = w->ensure(0, xtb + xsb)) return s;
  if (qk_status s = w->ensure(1, ptb + psb)) return s;
  if (qk_status s = w->ensure(2, ktb + ksb)) return s;
  double* dXt = static_cast<double*>(w->buf[0]);
  double* dXs = dXt + size_t(n_train) * p->width;
  char* dPt = static_cast<char*>(w->buf[1]);
  char* dPs = dPt + ptb;
  double* dKt = static_cast<double*>(w->buf[2]);
  double* dKs = dKt + size_t(n_train) * size_t(n_train);
  cudaStream_t st = w->stream;
  Trace trace(st);
  DrainTarget tg[2] = {{dKt, h_K_train, n_train, n_train, kModeGram, nullptr},
                       {dKs, h_K_cross, n_test, n_train, kModeCross, nullptr}};
  const int64_t nt = qk_job_tile_count(plan, n_train, n_test);
  const int n_targets = n_test > 0 ? 2 : 1;
  // Head-first upload (module comment above choose_head).  Pageable angle arrays are copied
  // into a pinned staging buffer by the host copy pool: the head rows before the head's
  // upload, the rest while the head sweeps.
  const bool pin_in = is_pinned(h_train) && (n_test == 0 || is_pinned(h_test));
  const bool pin_out = is_pinned(h_K_train) && (n_test == 0 || is_pinned(h_K_cross));
  const int64_t tail = pin_out ? -1 : INT64_MAX;  // see rect_tail_for
  const int64_t B = choose_head(*p, n_train, n_test, pin_in ? 50e6 : 35e6);
  const bool staged = B > 0 && !pin_in;
  const double* src_tr = h_train;  // the head rows' upload source
  if (staged) {
    if (qk_status s = w->ensure_in_stage(xtb + xsb)) return s;
    src_tr = static_cast<const double*>(w->in_stage);
  }
  if (B > 0) {
    // head: its angles, its planes, then the head sweep with the rest uploading beside it
    const int64_t s1 = std::min<int64_t>(n_train, B * kTile - sample_pad(n_train));
    const size_t row = size_t(p->width) * sizeof(double);
    if (staged) copy_pool().copy(w->in_stage, h_train, size_t(s1) * row);
    if (cudaError_t e = cudaMemsetAsync(w->bad, 0xFF, 2 * sizeof(uint64_t), st))
      return cuda_err(e, "sentinel reset");
    if (cudaError_t e = cudaMemcpyAsync(dXt, src_tr, size_t(s1) * row, cudaMemcpyHostToDevice,
                                        st))
      return cuda_err(e, "H2D head");
    trace.mark(1, st);
    if (qk_status s = launch_gate_build(*p, dXt, n_train, p->width, dPt, w->bad, st, 0, B))
      return s;
    const int64_t n_head = B * (B + 1) / 2;
    // The rest (its upload, its gate builds and its sweep) runs on the h2d stream, after the
    // head planes: its gate-build CTAs and then its sweep CTAs take the SMs as the head
    // sweep's CTAs retire, so the head's last wave overlaps the rest instead of idling SMs.
    // The main stream waits for the rest at the end (the drain does not need it: it follows
    // the tile-row counters).
    cudaStream_t hs = w->h2d_stream;
    cudaEvent_t ev[2];  // head planes + resets, rest sweep done
    for (int k = 0; k < 2; ++k)
      if (cudaError_t e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming)) {
        for (int j = 0; j < k; ++j) cudaEventDestroy(ev[j]);
        return cuda_err(e, "cudaEventCreate");
      }
    struct Destroy {
      cudaEvent_t* ev;
      ~Destroy() { cudaEventDestroy(ev[0]), cudaEventDestroy(ev[1]); }
    } destroy{ev};
    if (qk_status s = run_and_drain(w, *p, tg, n_targets, [&]() -> qk_status {
          // ev[0] follows the head planes, the sentinel reset AND run_and_drain's progress
          // counter reset, so the rest sweep's counter bumps are ordered after that reset
          if (cudaError_t e = cudaEventRecord(ev[0], st)) return cuda_err(e, "cudaEventRecord");
          if (qk_status s2 = launch_job(*p, dPt, n_train, dPs, n_test, 0, n_head, dKt, dKs, st,
                                        tg[0].d_prog, tg[1].d_prog, B, nullptr, false, tail))
            return s2;
          trace.point("head_end", st);
          trace.host("head_launched");
          trace.point("rest_h2d_start", hs);
          // the rest's angles: train rows [s1, n_train), then the test set.  Staged (pageable
          // inputs): the host copy pool stages them chunk by chunk while the head sweeps, each
          // chunk's upload queued as soon as it is staged, so the staging copies and the DMA
          // overlap (measured serial: ~1.0 ms of staging, then 1.3 ms of upload, then the GPU
          // idled ~0.3 ms between the head and the rest)
          struct Seg {
            double* dev;
            const double* host;
            size_t bytes;
          } segs[2] = {{dXt + s1 * p->width, h_train + s1 * p->width, size_t(n_train - s1) * row},
                       {dXs, h_test, n_test > 0 ? xsb : 0}};
          const size_t chunk = staged ? std::max(row, (size_t(16) << 20) / row * row) : SIZE_MAX;
          if (staged) cudaStreamQuery(st);  // flush the head launch to the device first
          cudaError_t e = cudaSuccess;
          char* stage_at = staged ? static_cast<char*>(w->in_stage) + size_t(s1) * row : nullptr;
          for (const Seg& sg : segs) {
            for (size_t off = 0; off < sg.bytes && e == cudaSuccess; off += chunk) {
              const size_t n = std::min(chunk, sg.bytes - off);
              const char* from = reinterpret_cast<const char*>(sg.host) + off;
              if (staged) {
                copy_pool().copy(stage_at, from, n);
                from = stage_at;
                stage_at += n;
              }
              e = cudaMemcpyAsync(reinterpret_cast<char*>(sg.dev) + off, from, n,
                                  cudaMemcpyHostToDevice, hs);
            }
          }
          trace.host("rest_staged");
          trace.point("rest_h2d_end", hs);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(hs, ev[0], 0);  // head planes, resets
          // on a failure past this point, let the rest's queued work finish before returning
          // (it reads and writes the workspace the next call reuses)
          auto fail = [&](qk_status s2) {
            cudaStreamSynchronize(hs);
            return s2;
          };
          if (e != cudaSuccess) return fail(cuda_err(e, "H2D rest"));
          if (qk_status s2 = launch_gate_build2(*p, dXt, n_train, dPt, w->bad, dXs, n_test, dPs,
                                                w->bad + 1, hs, B))
            return fail(s2);
          trace.point("rest_sweep_start", hs);
          if (qk_status s2 = launch_job(*p, dPt, n_train, dPs, n_test, n_head, nt, dKt, dKs, hs,
                                        tg[0].d_prog, tg[1].d_prog, B, nullptr, false, tail))
            return fail(s2);
          trace.point("rest_sweep_end", hs);
          e = cudaEventRecord(ev[1], hs);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev[1], 0);
          return e == cudaSuccess ? QK_OK : fail(cuda_err(e, "rest sweep join"));
        }, &trace))
      return s;
  } else {
    if (qk_status s = upload(w, dXt, h_train, xtb)) return s;
    if (qk_status s = upload(w, dXs, h_test, xsb)) return s;
    trace.mark(1, st);
    if (cudaError_t e = cudaMemsetAsync(w->bad, 0xFF, 2 * sizeof(uint64_t), st))
      return cuda_err(e, "sentinel reset");
    if (qk_status s = launch_gate_build2(*p, dXt, n_train, dPt, w->bad, dXs, n_test, dPs,
                                         w->bad + 1, st))
      return s;
    if (qk_status s = run_and_drain(w, *p, tg, n_targets, [&] {
          return launch_job(*p, dPt, n_train, dPs, n_test, 0, nt, dKt, dKs, st, tg[0].d_prog,
                            tg[1].d_prog, 0, nullptr, false, tail);
        }, &trace))
      return s;
  }
  static const char* const names[2] = {"train", "test"};
  return check_bad(w->bad, 2, names);
}

int64_t qk_job_tile_count(const qk_plan* plan, int64_t n_train, int64_t n_test) {
  if (plan == nullptr || n_train < 0 || n_test < 0) return 0;
  return qk_gram_tile_count(plan, n_train) + qk_cross_tile_count(plan, n_test, n_train);
}

qk_status qk_job_tiles(const qk_plan* plan, const void* d_planes_train, int64_t n_train,
                       const void* d_planes_test, int64_t n_test, int64_t tile_begin,
                       int64_t tile_end, double* d_K_train, double* d_K_cross, void* stream) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  const int64_t nt = qk_job_tile_count(plan, n_train, n_test);
  if (n_train < 0 || n_test < 0 || tile_begin < 0 || tile_end < tile_begin || tile_end > nt)
    return set_error(QK_ERR_VALUE, "tile range outside the job tile list");
  if (tile_end == tile_begin) return QK_OK;
  if (!d_planes_train || !d_K_train || (n_test > 0 && (!d_planes_test || !d_K_cross)))
    return set_error(QK_ERR_VALUE, "NULL buffer");
  if (!aligned16(d_planes_train) || (n_test > 0 && !aligned16(d_planes_test)))
    return set_error(QK_ERR_VALUE, "planes must be 16-byte aligned");
  return launch_job(*p, d_planes_train, n_train, d_planes_test, n_test, tile_begin, tile_end,
                    d_K_train, d_K_cross, stream);
}

}  // extern "C"

// ---- multi-GPU result placement (CUDA IPC over NVLink / NVSwitch) ------------------------
extern "C" {

qk_status qk_shared_alloc(size_t bytes, void** out_d_ptr) {
  if (out_d_ptr == nullptr) return set_error(QK_ERR_VALUE, "NULL output");
  *out_d_ptr = nullptr;
  if (bytes == 0) bytes = 16;
  if (cudaError_t e = cudaMalloc(out_d_ptr, bytes))
    return set_error(QK_ERR_CAPACITY, std::string("shared allocation of ") +
                                          std::to_string(bytes) + " bytes failed: " +
                                          cudaGetErrorString(e));
  return QK_OK;
}

qk_status qk_shared_free(void* d_ptr) {
  if (d_ptr == nullptr) return QK_OK;
  return cuda_err(cudaFree(d_ptr), "shared free");
}

qk_status qk_ipc_export(const void* d_ptr, unsigned char out_handle[QK_IPC_HANDLE_BYTES]) {
  if (d_ptr == nullptr || out_handle == nullptr) return set_error(QK_ERR_VALUE, "NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == QK_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  if (cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)))
    return cuda_err(e, "cudaIpcGetMemHandle (pointer must come from qk_shared_alloc)");
  std::memcpy(out_handle, &h, sizeof(h));
  return QK_OK;
}

qk_status qk_ipc_import(const unsigned char handle[QK_IPC_HANDLE_BYTES], void** out_d_ptr) {
  if (handle == nullptr || out_d_ptr == nullptr) return set_error(QK_ERR_VALUE, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  *out_d_ptr = nullptr;
  return cuda_err(cudaIpcOpenMemHandle(out_d_ptr, h, cudaIpcMemLazyEnablePeerAccess),
                  "cudaIpcOpenMemHandle");
}

qk_status qk_device_bus_id(char out_bus_id[QK_BUS_ID_BYTES]) {
  if (out_bus_id == nullptr) return set_error(QK_ERR_VALUE, "NULL output");
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_err(e, "cudaGetDevice");
  return cuda_err(cudaDeviceGetPCIBusId(out_bus_id, QK_BUS_ID_BYTES, dev), "cudaDeviceGetPCIBusId");
}

qk_status qk_can_reach(const char* bus_id, int32_t* out_reachable) {
  if (bus_id == nullptr || out_reachable == nullptr) return set_error(QK_ERR_VALUE, "NULL argument");
  *out_reachable = 0;
  int dev = 0, peer = -1;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_err(e, "cudaGetDevice");
  if (cudaDeviceGetByPCIBusId(&peer, bus_id) != cudaSuccess) {
    cudaGetLastError();  // the owner's device is not visible to this process
    return QK_OK;
  }
  if (peer == dev) {
    *out_reachable = 1;
    return QK_OK;
  }
  int ok = 0;
  if (cudaError_t e = cudaDeviceCanAccessPeer(&ok, dev, peer)) return cuda_err(e, "cudaDeviceCanAccessPeer");
  *out_reachable = ok ? 1 : 0;
  return QK_OK;
}

qk_status qk_ipc_close(void* d_ptr) {
  if (d_ptr == nullptr) return QK_OK;
  return cuda_err(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
}

qk_status qk_host_register(void* h_ptr, size_t bytes) {
  if (h_ptr == nullptr || bytes == 0) return set_error(QK_ERR_VALUE, "empty host range");
  return cuda_err(cudaHostRegister(h_ptr, bytes, cudaHostRegisterPortable), "cudaHostRegister");
}

qk_status qk_host_unregister(void* h_ptr) {
  if (h_ptr == nullptr) return QK_OK;
  return cuda_err(cudaHostUnregister(h_ptr), "cudaHostUnregister");
}

qk_status qk_copy_h2d(void* d_dst, const void* h_src, size_t bytes, void* stream) {
  if (bytes == 0) return QK_OK;
  if (d_dst == nullptr || h_src == nullptr) return set_error(QK_ERR_VALUE, "NULL pointer");
  return cuda_err(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice,
                                  static_cast<cudaStream_t>(stream)),
                  "H2D copy");
}

qk_status qk_copy_d2d(void* d_dst, const void* d_src, size_t bytes, void* stream) {
  if (bytes == 0) return QK_OK;
  if (d_dst == nullptr || d_src == nullptr) return set_error(QK_ERR_VALUE, "NULL pointer");
  return cuda_err(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice,
                                  static_cast<cudaStream_t>(stream)),
                  "D2D copy");
}

qk_status qk_copy_d2h(void* h_dst, const void* d_src, size_t bytes, void* stream) {
  if (bytes == 0) return QK_OK;
  if (h_dst == nullptr || d_src == nullptr) return set_error(QK_ERR_VALUE, "NULL pointer");
  return cuda_err(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost,
                                  static_cast<cudaStream_t>(stream)),
                  "D2H copy");
}

}  // extern "C"
