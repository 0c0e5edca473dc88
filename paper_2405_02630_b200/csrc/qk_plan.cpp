// qk_plan.cpp — host sweep planner and the C-ABI error plumbing of libqk.
//
// Replaces the reference planner's role (plan_contraction, paths.py:529-543, over the
// simplified network of network.py:183-280): for the feature-map family
// (RY embedding + linear CNOT chain, circuit.py:121-133) the contraction order is fixed by
// the structure — a sweep along the qubit chain — so the plan only records the geometry of
// that sweep (tile edge, qubit chunk, identity padding, overflow-safe rescaling) and the
// per-entry costs the roofline is computed from.  Pure host code: no CUDA calls here.
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "qk_internal.h"

namespace qk {

static thread_local std::string g_last_error;

qk_status set_error(qk_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

qk_status check_plan(const qk_plan* p, const Plan** out) {
  if (p == nullptr) return set_error(QK_ERR_VALUE, "plan is NULL");
  *out = &p->p;
  return QK_OK;
}

int64_t blocks_for(int64_t n_samples) { return (n_samples + kTile - 1) / kTile; }

}  // namespace qk

using namespace qk;

extern "C" {

int qk_abi_version(void) { return QK_ABI_VERSION; }

const char* qk_last_error(void) { return g_last_error.c_str(); }

qk_status qk_plan_create(int32_t width, int32_t layers, int32_t convention, qk_plan** out_plan) {
  if (out_plan == nullptr) return set_error(QK_ERR_VALUE, "out_plan is NULL");
  *out_plan = nullptr;
  // FeatureMapConfig.__post_init__ (circuit.py:86-91): same messages.
  if (width < 1) return set_error(QK_ERR_VALUE, "width must be >= 1");
  if (layers < 1) return set_error(QK_ERR_VALUE, "layers must be >= 1");
  if (convention != QK_PROBABILITY && convention != QK_MAGNITUDE)
    return set_error(QK_ERR_VALUE, "unknown kernel convention " + std::to_string(convention));
  if (layers > kMaxLayers)
    return set_error(QK_ERR_CAPACITY,
                     "layers=" + std::to_string(layers) + " needs a bond-" +
                         std::to_string(int64_t(1) << (2 * (layers - 1))) +
                         " transfer state per pair; the sm_100a sweep implements layers 1 to " +
                         std::to_string(kMaxLayers) + " (shared-memory state <= 128 KB)");

  qk_plan* h = new (std::nothrow) qk_plan();
  if (h == nullptr) return set_error(QK_ERR_CAPACITY, "out of host memory");
  Plan& p = h->p;
  p.width = width;
  p.layers = layers;
  p.convention = convention;
  p.width_padded = ((width + kChunk - 1) / kChunk) * kChunk;
  p.front_pad = p.width_padded - width;
  const int nchunks = p.width_padded / kChunk;
  if ((layers >= 2 && layers <= 4) || (QK_DEEP_BONDR && layers == 5)) {
    // The rotated recurrences (bond 4, the blocked bonds 16 / 64 / 256) drop a factor 1/2 per processed
    // qubit (the identity qubits of the front padding are skipped, not processed); the kernels
    // multiply the state by 2^-512 after every kRescaleChunks chunks.
    const int rescales = (nchunks - 1) / kRescaleChunks;
    p.final_scale = std::ldexp(1.0, -(p.width - 512 * rescales));
  } else {
    p.final_scale = 1.0;
  }

  qk_plan_info& in = p.info;
  std::memset(&in, 0, sizeof(in));
  in.width = width;
  in.layers = layers;
  in.convention = convention;
  in.bond = 1 << (2 * (layers - 1));
  in.tile_edge = kTile;
  in.chunk = kChunk;
  in.width_padded = p.width_padded;
  in.stages = kStages;
  const int64_t n = width;
  if (layers == 2) {
    // per qubit per pair: 4 DMUL + 4 DADD + 8 DFMA -> 16 instr, 24 flops; epilogue 3
    in.dp_instr_per_entry = 16 * n + 3;
    in.flops_per_entry = 24 * n + 3;
    in.algorithmic_flops_per_entry = 34 * n + 4;
    in.reference_cmacs_per_entry = n >= 8 ? 1056 * n - 3912 : 0;
  } else if (layers == 1) {
    // per qubit per pair: DMUL + DFMA + DMUL
    in.dp_instr_per_entry = 3 * n;
    in.flops_per_entry = 4 * n;
    in.algorithmic_flops_per_entry = 4 * n;
    in.reference_cmacs_per_entry = 0;
  } else if (layers <= 4) {
    // rotated blocked bond (qk_sweep.cu bondr_step), M = L-1, E = 4^M: full angles 8, cos/sin
    // of the difference 4, separable sums 4, lower-level passes 4 (M-1) E (half of them FMAs),
    // the E/4 block updates 2 E (1.5 E FMAs); E/2 - 1 adds, the scale and the square last
    const int64_t M = layers - 1, E = int64_t(1) << (2 * M);
    const int64_t instr = 4 * (M - 1) * E + 2 * E + 16, fmas = 2 * (M - 1) * E + 3 * E / 2 + 4;
    in.dp_instr_per_entry = instr * n + E / 2 + 1;
    in.flops_per_entry = (instr + fmas) * n + E / 2 + 1;
    in.algorithmic_flops_per_entry = in.flops_per_entry;
    in.reference_cmacs_per_entry = 0;
  } else {
    // L >= 5, D = 2^(L-1), V is D x D (E = D^2 elements).  Per qubit per pair: two sides of
    // M = L-1 level passes, each D^2/2 rotations of 2 DMUL + 2 DFMA (6 flops); cos/sin of
    // delta/2 (2 DMUL + 2 DFMA); the RY(delta) mask (E DMUL).  E - 1 adds and the square last
    // (algorithmic).  Executed, L = 5..7 (qk_sweep.cu deep_sweep_reg, D threads per pair):
    // every thread forms cos/sin of delta/2 and 4 mask-scaled level-0 coefficients per qubit
    // (the mask is folded into the next qubit's first level), one pending mask and the sums
    // (2 E) at the end; L = 8 (shared-memory rounds) as the algorithmic count.
    const int64_t M = layers - 1, D = int64_t(1) << M, E = D * D, HB = D / 2;
    in.algorithmic_flops_per_entry = (6 * M * E + E + 6) * n + E;
    if (QK_DEEP_BONDR && layers == 5) {
      // rotated blocked form (deep_sweep_bondr): lower levels 4 (M-1) E, the E/4 block steps
      // 2 E, and per thread (HB per pair) 18 instructions of angles and coefficients; the sum
      in.dp_instr_per_entry = (4 * (M - 1) * E + 2 * E + 18 * HB) * n + E / 2 + HB;
      in.flops_per_entry = (6 * (M - 1) * E + 3 * E + 22 * HB) * n + E / 2 + HB;
    } else if (layers <= 7) {
      in.dp_instr_per_entry = (4 * M * E + 8 * D) * n + 2 * E;
      in.flops_per_entry = (6 * M * E + 10 * D) * n + 2 * E;
    } else {
      in.dp_instr_per_entry = (4 * M * E + E + 4) * n + E;
      in.flops_per_entry = in.algorithmic_flops_per_entry;
    }
    in.reference_cmacs_per_entry = 0;
  }
  *out_plan = h;
  return QK_OK;
}

qk_status qk_plan_destroy(qk_plan* plan) {
  delete plan;
  return QK_OK;
}

qk_status qk_plan_get_info(const qk_plan* plan, qk_plan_info* out_info) {
  const Plan* p;
  if (qk_status s = check_plan(plan, &p)) return s;
  if (out_info == nullptr) return set_error(QK_ERR_VALUE, "out_info is NULL");
  *out_info = p->info;
  return QK_OK;
}

size_t qk_planes_bytes(const qk_plan* plan, int64_t n_samples) {
  if (plan == nullptr || n_samples < 0) return 0;
  return static_cast<size_t>(blocks_for(n_samples)) * plan->p.width_padded * kTile * 16;
}

int64_t qk_gram_tile_count(const qk_plan* plan, int64_t n_samples) {
  if (plan == nullptr || n_samples < 0) return 0;
  const int64_t nb = blocks_for(n_samples);
  return nb * (nb + 1) / 2;
}

int64_t qk_cross_tile_count(const qk_plan* plan, int64_t n_rows, int64_t n_cols) {
  if (plan == nullptr || n_rows < 0 || n_cols < 0) return 0;
  return blocks_for(n_rows) * blocks_for(n_cols);
}

}  // extern "C"
