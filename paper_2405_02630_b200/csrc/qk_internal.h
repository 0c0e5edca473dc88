// qk_internal.h — shared host-side definitions of libqk (not part of the ABI).
#pragma once

#include <cstdint>
#include <string>

#include "qk.h"

namespace qk {

// Sweep geometry shared by the planner, the gate-build kernel and the sweep kernels.
constexpr int kTile = 64;    // samples per plane block == tile edge T
#ifndef QK_CHUNK
#define QK_CHUNK 16
#endif
#ifndef QK_STAGES
#define QK_STAGES 4
#endif
constexpr int kChunk = QK_CHUNK;    // qubits per bulk-copy chunk Q
constexpr int kStages = QK_STAGES;  // shared-memory ring depth
constexpr int kRescaleChunks = 512 / kChunk;  // L=2: rescale the bond state by 2^-512 every 512 qubits
constexpr int kMaxLayers = 8;       // L <= 4: registers; L = 5..8: shared-memory deep sweep
constexpr int kGroup = 8;           // tile rows per super-row of the L2-friendly tile order
#ifndef QK_RECT_GROUP
#define QK_RECT_GROUP 8
#endif
// Cross tile lists: super-rows of kRectGroup tile rows walked column by column (each train
// column block is read from HBM once per super-row instead of once per tile row: config 4's
// cross pass reads 0.6 instead of 4.0 GB), except the last kRectTail tile rows, which run row
// by row so the host pipelines' final row panels drain while the sweep still runs.
constexpr int kRectGroup = QK_RECT_GROUP;
constexpr int kRectTail = 2;

struct Plan {
  int32_t width = 0;
  int32_t layers = 0;
  int32_t convention = 0;
  int32_t width_padded = 0;  // multiple of kChunk; the first (width_padded - width) rows are identity
  int32_t front_pad = 0;
  double final_scale = 1.0;  // 2^-(width_padded - 512 * rescales) for L = 2, 1 for L = 1
  qk_plan_info info{};
};

qk_status set_error(qk_status code, const std::string& msg);
qk_status check_plan(const qk_plan* p, const Plan** out);

int64_t blocks_for(int64_t n_samples);

#ifdef __CUDACC__
#define QK_HD __host__ __device__
#else
#define QK_HD
#endif

// Sample padding of a plane set: the ragged remainder sits at the FRONT of block 0 (slot
// t of block b holds sample 64 b + t - pad), so it is a tile ROW of every Gram tile that
// touches it and whole warps of those tiles can skip it.
QK_HD inline int sample_pad(int64_t n) { return int((kTile - n % kTile) % kTile); }

// Progress-counter increments per finished tile (host pipelines): L <= 2 two per tile (a tile
// of the last wave may run as two row halves, one each), L = 3, 4
// one per 16x16 sub-tile, L >= 5 one per pair group of the deep sweep (16, 8, 4, 1 pairs at
// L = 5, 6, 7, 8: Deep<M>::PP in qk_sweep.cu).
// QK_DEEP_BONDR: L = 5 in the rotated blocked form (qk_sweep.cu deep_sweep_bondr: D / 2 threads
// per pair, twice the pairs per CTA; 1, default) or one thread per column of the state (0).
// Measured (784 qubits, Gram): L = 5 3.86 -> 4.34 M entries/s.  At L = 6 the blocked form
// needs 206 registers per thread (0.72 vs 0.78 M entries/s), so L = 6 keeps the column form.
#ifndef QK_DEEP_BONDR
#define QK_DEEP_BONDR 1
#endif
QK_HD constexpr uint32_t progress_unit(int layers) {
  if (layers <= 2) return 2u;
  if (layers <= 4) return 16u;
  const int pp = layers == 5 ? (QK_DEEP_BONDR ? 32 : 16) : layers == 6 ? 8 : layers == 7 ? 4 : 1;
  return uint32_t(kTile * kTile / pp);
}

// First linear index of tile row r in the upper-triangle tile list over nb blocks.
QK_HD inline int64_t upper_row_offset(int64_t r, int64_t nb) { return r * nb - r * (r - 1) / 2; }

// Device launchers (qk_sweep.cu).  They return QK_OK or a QK_ERR_CUDA status.
qk_status launch_gate_build(const Plan& p, const double* d_angles, int64_t n, int64_t ld,
                            void* d_planes, uint64_t* d_bad, void* stream,
                            int64_t blk_begin = 0, int64_t blk_end = -1);
// Two plane sets (train and test, width-long rows) in ONE launch; set a from block blk_begin_a.
qk_status launch_gate_build2(const Plan& p, const double* d_a, int64_t n_a, void* d_planes_a,
                             uint64_t* d_bad_a, const double* d_b, int64_t n_b,
                             void* d_planes_b, uint64_t* d_bad_b, void* stream,
                             int64_t blk_begin_a = 0);
qk_status launch_sweep(const Plan& p, int mode, const void* d_rows, int64_t n_rows,
                       const void* d_cols, int64_t n_cols, int64_t tile_begin, int64_t tile_end,
                       double* d_out, int64_t ld_out, int out_mode, void* stream,
                       unsigned int* d_progress = nullptr, int64_t head_b = 0,
                       unsigned long long* counter = nullptr, bool pdl = false,
                       int64_t rect_tail = -1);
qk_status launch_unpack(const Plan& p, int mode, const double* d_packed, int64_t n_rows,
                        int64_t n_cols, int64_t tile_begin, int64_t tile_end, double* d_K,
                        int64_t ld, void* stream);
// d_amp: signed amplitudes, or (kernel_values) K under the plan's convention.
qk_status launch_pairs(const Plan& p, const void* d_a, int64_t n_a, const void* d_b, int64_t n_b,
                       const int64_t* d_pairs, int64_t n_pairs, double* d_amp, void* stream,
                       bool kernel_values = false);
qk_status launch_dfma_peak(double* out, void* stream);

enum SweepMode { kModeGram = 0, kModeCross = 1, kModeJob = 2 };

// Train Gram + test-versus-train cross block as ONE tile list: tiles [0, gram_tiles) are the
// Gram's, the rest the cross block's (dense outputs; optional per-super-row progress).
qk_status launch_job(const Plan& p, const void* d_train, int64_t n_train, const void* d_test,
                     int64_t n_test, int64_t tile_begin, int64_t tile_end, double* d_K_train,
                     double* d_K_cross, void* stream, unsigned int* d_prog_train = nullptr,
                     unsigned int* d_prog_cross = nullptr, int64_t head_b = 0,
                     unsigned long long* counter = nullptr, bool pdl = false,
                     int64_t rect_tail = -1);  // -1: kRectTail; pageable host drains: all rows
// The dynamic tile schedule's claim counter for one sweep launch, zeroed on `st` (a ring slot,
// or a stream-ordered allocation under graph capture: *owned, free it after the launch).
// Callers that reset it (all-ones) ahead of a gate build pass it to launch_job / launch_sweep
// with pdl.
qk_status acquire_tile_counter(void* stream, unsigned long long** out, bool* owned);

}  // namespace qk

struct qk_plan {
  qk::Plan p;
};
