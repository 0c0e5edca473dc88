/*
 * qk.h — C ABI of the B200-native QSVM quantum-kernel engine (libqk.so).
 *
 * The hot path is the quantum-kernel Gram matrix
 *     K(x_i, x_j) = |<0| U(x_i)^dag U(x_j) |0>|^2        (probability convention)
 * for the reference's default feature map: per layer, RY(x_q) on every wire,
 * then the linear CNOT chain q -> q+1 (reference: pkg/src/tnkernel/circuit.py:121-133),
 * composed as U(x_j) followed by U(x_i)^dag (circuit.py:151-157).
 *
 * Every entry point takes plain pointers and sizes; device pointers are CUDA
 * global-memory addresses owned by the caller, `stream` is a cudaStream_t
 * (NULL = legacy default stream).  All launches are stream-ordered and
 * asynchronous unless stated.  No entry point falls back to the CPU: without a
 * usable CUDA device every compute call returns QK_ERR_CUDA.
 *
 * Error convention: every function returns a qk_status; the message of the
 * most recent failure on the calling thread is returned by qk_last_error().
 * The Python mirror maps the codes onto the reference's exception hierarchy
 * (reference: pkg/src/tnkernel/errors.py:8-47):
 *     QK_ERR_VALUE      -> ValueError         (circuit.py:86-91 config checks)
 *     QK_ERR_REBIND     -> RebindError        (network.py:291-296, engine.py:139-155)
 *     QK_ERR_CAPACITY   -> CapacityError      (engine.py:23,70-73; statevector.py:43-46)
 *     QK_ERR_STRUCTURAL -> StructuralError    (paths.py:96-130)
 *     QK_ERR_CUDA       -> RuntimeError       (no device / launch failure)
 */
#ifndef QK_H_
#define QK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QK_ABI_VERSION 2

typedef enum {
  QK_OK = 0,
  QK_ERR_VALUE = 1,
  QK_ERR_REBIND = 2,
  QK_ERR_CAPACITY = 3,
  QK_ERR_STRUCTURAL = 4,
  QK_ERR_CUDA = 5
} qk_status;

/* Kernel value convention (reference: statevector.py:62-70). */
typedef enum { QK_PROBABILITY = 0, QK_MAGNITUDE = 1 } qk_convention;

/* Output layouts for the Gram sweep. */
typedef enum {
  QK_OUT_DENSE = 0,  /* N x N row-major; writes K[i][j] and K[j][i] for i<j, K[i][i] = 1 */
  QK_OUT_PACKED = 1  /* tile-major: tile t -> tile_edge*tile_edge block at (t-tile_begin)*edge^2 */
} qk_out_mode;

typedef struct qk_plan qk_plan; /* opaque; immutable after creation; shareable across threads */

/* Planner report: what the structure-fixed sweep does per entry. */
typedef struct {
  int32_t width;           /* qubits n (= features per sample) */
  int32_t layers;          /* feature-map layers L */
  int32_t convention;      /* qk_convention */
  int32_t bond;            /* transfer-state size per pair: 4^(L-1) = 1, 4, 16, ..., 16384 */
  int32_t tile_edge;       /* samples per tile edge T (and per plane block) */
  int32_t chunk;           /* qubits per staged chunk Q */
  int32_t width_padded;    /* n rounded up to a multiple of Q (identity qubits in front) */
  int32_t stages;          /* shared-memory ring depth of the bulk-copy pipeline */
  int64_t dp_instr_per_entry;      /* fp64 instructions issued per pair (DFMA/DMUL/DADD) */
  int64_t flops_per_entry;         /* executed fp64 flops per pair (FMA = 2) */
  int64_t algorithmic_flops_per_entry; /* 34 n + 4 for L = 2 */
  int64_t reference_cmacs_per_entry;   /* reference planner cost (1056 n - 3912 at L = 2), report only */
} qk_plan_info;

/* ---- version / errors / device ------------------------------------------- */
int qk_abi_version(void);
const char* qk_last_error(void);
/* Make `device` current for libqk's calls on this host thread (one process may drive
 * several GPUs; launches must run on the device that owns the caller's stream and buffers). */
qk_status qk_set_device(int32_t device);

/* ---- planner: replaces plan_contraction (paths.py:529-543) + simplify (network.py:183)
 * Fixes the contraction (a qubit-chain sweep with the bond state in registers) once per
 * circuit structure (width, layers, convention); every pair reuses it ("path reuse",
 * SPEC.md:340).  Pure host code: validates like FeatureMapConfig
 * (circuit.py:86-91) and never touches the GPU.  layers 1..8: bond 4^(L-1) in registers for
 * L <= 4, in shared memory for L = 5..8; layers > 8 -> QK_ERR_CAPACITY (the reference's own
 * contraction of those circuits hits its intermediate cap or runs for hours per entry). */
qk_status qk_plan_create(int32_t width, int32_t layers, int32_t convention, qk_plan** out_plan);
qk_status qk_plan_destroy(qk_plan* plan);
qk_status qk_plan_get_info(const qk_plan* plan, qk_plan_info* out_info);

/* Byte size of the gate planes for n_samples samples (caller allocates, 16-B aligned). */
size_t qk_planes_bytes(const qk_plan* plan, int64_t n_samples);
/* Number of upper-triangle (i-block <= j-block) tiles of an n_samples Gram. */
int64_t qk_gram_tile_count(const qk_plan* plan, int64_t n_samples);
/* Number of tiles of an n_rows x n_cols cross block. */
int64_t qk_cross_tile_count(const qk_plan* plan, int64_t n_rows, int64_t n_cols);

/* ---- gate build: replaces rebind_operands/_chain_data (network.py:283-302, 42-54)
 * per SAMPLE instead of per pair: angles [n_samples x width] fp64 row-major (leading
 * dimension ld >= width) -> per-(sample, qubit) rotation planes in HBM.
 * If d_bad_sample != NULL it is atomically min-reduced with the index of every sample
 * holding a non-finite angle; the caller initialises it to UINT64_MAX (all-ones bytes),
 * which is what it still holds when every angle is finite (RebindError, network.py:295). */
qk_status qk_gate_build(const qk_plan* plan, const double* d_angles, int64_t n_samples, int64_t ld,
                        void* d_planes, uint64_t* d_bad_sample, void* stream);

/* ---- sweeps: replace contract_batch/contract/_contract_once (engine.py:52-166) ------ */
/* Train Gram, tiles [tile_begin, tile_end) of the upper-triangle tile list.
 * QK_OUT_DENSE: d_out is n_samples x n_samples (ld = n_samples); the strict upper
 * triangle is computed, mirrored, and the diagonal injected as exactly 1.0
 * (SPEC.md:398-415).  QK_OUT_PACKED: see qk_out_mode. */
qk_status qk_gram_tiles(const qk_plan* plan, const void* d_planes, int64_t n_samples,
                        int64_t tile_begin, int64_t tile_end, double* d_out, int32_t out_mode,
                        void* stream);
/* Scatter packed Gram tiles into the dense symmetric matrix. */
qk_status qk_unpack_gram(const qk_plan* plan, const double* d_packed, int64_t n_samples,
                         int64_t tile_begin, int64_t tile_end, double* d_K, void* stream);
/* Test-versus-train block: K[r][c] = k(x_rows[r], x_cols[c]) over tiles [tile_begin,
 * tile_end) of the rectangle, no symmetrisation, diagonal computed.
 * QK_OUT_DENSE: d_out is n_rows x n_cols row-major with leading dimension ld_out. */
qk_status qk_cross_tiles(const qk_plan* plan, const void* d_planes_rows, int64_t n_rows,
                         const void* d_planes_cols, int64_t n_cols, int64_t tile_begin,
                         int64_t tile_end, double* d_out, int64_t ld_out, int32_t out_mode,
                         void* stream);
/* Unpack packed cross tiles into an n_rows x n_cols row-major block (leading dim ld). */
qk_status qk_unpack_cross(const qk_plan* plan, const double* d_packed, int64_t n_rows,
                          int64_t n_cols, int64_t tile_begin, int64_t tile_end, double* d_K,
                          int64_t ld, void* stream);
/* Train Gram + test-versus-train block as ONE tile list (tiles [0, qk_gram_tile_count) are the
 * Gram's, the rest the cross block's), one persistent launch for any sub-range — the QSVM
 * train/test kernel pair of Algorithm 2.  Dense outputs: d_K_train is
 * n_train x n_train (symmetrised, unit diagonal), d_K_cross is n_test x n_train. */
int64_t qk_job_tile_count(const qk_plan* plan, int64_t n_train, int64_t n_test);
qk_status qk_job_tiles(const qk_plan* plan, const void* d_planes_train, int64_t n_train,
                       const void* d_planes_test, int64_t n_test, int64_t tile_begin,
                       int64_t tile_end, double* d_K_train, double* d_K_cross, void* stream);
/* One whole job step on DEVICE angles (train [n_train x width], test [n_test x width], row-
 * major), one host call: the job state reset (one memset), the gate planes of both sets
 * built in one launch (the rebind of network.py:283-302, per sample), then the joint tile
 * range [tile_begin, tile_end) of qk_job_tiles swept in one persistent launch that follows
 * the gate build as a programmatic dependent — the small-job path (stream-ordered,
 * capturable in a CUDA graph: three nodes).  d_planes_*: caller buffers of
 * qk_planes_bytes(n).  d_state: QK_JOB_STATE_WORDS uint64 words of device scratch owned by
 * the caller: [0], [1] = the non-finite sentinels (train, test), valid once the stream has
 * synchronised: UINT64_MAX when every angle is finite, else the first non-finite sample (the
 * caller raises the reference's RebindError, network.py:295-296); [2] = the sweep's tile-
 * claim counter.  Calls sharing one d_state must be stream-ordered. */
#define QK_JOB_STATE_WORDS 3
qk_status qk_job_run(const qk_plan* plan, const double* d_train, int64_t n_train,
                     const double* d_test, int64_t n_test, void* d_planes_train,
                     void* d_planes_test, uint64_t* d_state, int64_t tile_begin,
                     int64_t tile_end, double* d_K_train, double* d_K_cross, void* stream);
/* contract_batch drop-in (engine.py:132-166): signed real amplitudes
 * <0|U(a_p)^dag U(b_q)|0> for an explicit list of index pairs d_pairs[k] = (p, q),
 * output order = input order. */
qk_status qk_pair_amplitudes(const qk_plan* plan, const void* d_planes_a, int64_t n_a,
                             const void* d_planes_b, int64_t n_b, const int64_t* d_pairs,
                             int64_t n_pairs, double* d_amp, void* stream);
/* The same pairs as kernel values K(a_p, b_q) under the plan's convention (|amp|^2 or |amp|,
 * statevector.py:62-70) — the SPEC's `--shard k/W` partial:
 * one value per strict-upper or cross pair, in input order.  Out-of-range indices give NaN. */
qk_status qk_pair_kernel_values(const qk_plan* plan, const void* d_planes_a, int64_t n_a,
                                const void* d_planes_b, int64_t n_b, const int64_t* d_pairs,
                                int64_t n_pairs, double* d_K, void* stream);

/* ---- host-buffer entry points (the user-facing call; synchronous) ----------------
 * compute_kernel_matrix and compute_cross_kernel
 * from HOST angle arrays to HOST kernel matrices: H2D, gate build, sweep, D2H,
 * pipelined over row panels on the plan's device (CUDA current device). */
qk_status qk_kernel_matrix_host(const qk_plan* plan, const double* h_angles, int64_t n_samples,
                                double* h_K);
qk_status qk_cross_kernel_host(const qk_plan* plan, const double* h_rows, int64_t n_rows,
                               const double* h_cols, int64_t n_cols, double* h_K);
/* Both of the above in one pipeline (one upload of the train angles, one sweep launch over the
 * joint tile list, both matrices drained while it runs). */
qk_status qk_kernel_matrices_host(const qk_plan* plan, const double* h_train, int64_t n_train,
                                  const double* h_test, int64_t n_test, double* h_K_train,
                                  double* h_K_cross);

/* ---- measurement helper: fp64 FMA issue-rate microbenchmark (FLOP/s) ------------- */
qk_status qk_dfma_peak(double* out_flops_per_s, void* stream);

/* ---- multi-GPU result placement over peer memory (NVLink / NVSwitch) ------------------
 * Replaces the reference's result collection across workers (engine.py:159-166 pool
 * gather; SPEC.md:425-434 shard merge; PAPER.md:359-362 MPI/NCCL): rank 0 allocates the
 * dense kernel matrices with qk_shared_alloc and exports them; every other rank imports the
 * handle and passes the imported pointer as d_out of qk_gram_tiles / qk_cross_tiles
 * (QK_OUT_DENSE), so each sweep stores its tiles (and their mirror) straight into rank 0's
 * matrix — no gather buffer, no unpack.  CUDA IPC; requires peer access between devices. */
#define QK_IPC_HANDLE_BYTES 64
qk_status qk_shared_alloc(size_t bytes, void** out_d_ptr);
qk_status qk_shared_free(void* d_ptr);
qk_status qk_ipc_export(const void* d_ptr, unsigned char out_handle[QK_IPC_HANDLE_BYTES]);
qk_status qk_ipc_import(const unsigned char handle[QK_IPC_HANDLE_BYTES], void** out_d_ptr);
qk_status qk_ipc_close(void* d_ptr);
/* Placement decision before any import: the PCI bus id of the current device (so ranks whose
 * processes see different device orderings can name it), and whether the current device can
 * store into memory of the device with that bus id (1: the same device, or peer access over
 * NVLink / PCIe; 0: not visible to this process, or no peer access -> gather placement). */
#define QK_BUS_ID_BYTES 32
qk_status qk_device_bus_id(char out_bus_id[QK_BUS_ID_BYTES]);
qk_status qk_can_reach(const char* bus_id, int32_t* out_reachable);
/* Host side of the multi-GPU result: a row-major host matrix that every rank process maps
 * (a POSIX shared-memory segment) is page-locked in each of them (qk_host_register), and
 * each rank copies ITS row slice of rank 0's device matrix into it (qk_copy_d2h: a
 * stream-ordered copy from any device address, peer memory included), so the 8 B/entry
 * result crosses N PCIe links in parallel instead of rank 0's alone. */
qk_status qk_host_register(void* h_ptr, size_t bytes);
qk_status qk_host_unregister(void* h_ptr);
qk_status qk_copy_d2h(void* h_dst, const void* d_src, size_t bytes, void* stream);
/* The input side likewise: each rank uploads its slice of the angles into rank 0's shared
 * angle buffer (qk_copy_h2d to a peer address) and then pulls the whole set over NVLink
 * (qk_copy_d2d from the peer address). */
qk_status qk_copy_h2d(void* d_dst, const void* h_src, size_t bytes, void* stream);
qk_status qk_copy_d2d(void* d_dst, const void* d_src, size_t bytes, void* stream);

/* ---- dense state-vector ground truth (checker beyond the reference's 24-qubit guard) ----
 * Replaces the reference's brute-force simulator (statevector.py:41-70, simulate /
 * zero_amplitude / kernel_entry_oracle) for the pair circuit compose_kernel_circuit(x_i, x_j)
 * (circuit.py:150-157): every gate in the reference's order on a real fp64 state, amplitudes
 * bit-identical to the reference's complex128 simulate().  Independent of the sweep.
 *   qk_statevector_amplitude: one pair, host angle vectors x_i, x_j [width]; d_state is a
 *     caller-owned device buffer of qk_statevector_bytes(width) bytes; *out_amp (host) gets
 *     <0..0| U(x_i)^dag U(x_j) |0..0>.  Width <= 40 (memory permitting).
 *   qk_statevector_pairs: many pairs at width <= 13 (state in shared memory, one CTA per
 *     pair); host angle sets A [n_a x width], B [n_b x width], 0-based pairs (row of A,
 *     row of B), host amplitudes out.  Synchronous. */
size_t qk_statevector_bytes(int32_t width);
qk_status qk_statevector_amplitude(int32_t width, int32_t layers, const double* x_i,
                                   const double* x_j, double* d_state, double* out_amp,
                                   void* stream);
qk_status qk_statevector_pairs(int32_t width, int32_t layers, const double* h_a, int64_t n_a,
                               const double* h_b, int64_t n_b, const int64_t* h_pairs,
                               int64_t n_pairs, double* h_amp);

#ifdef __cplusplus
}
#endif
#endif /* QK_H_ */
