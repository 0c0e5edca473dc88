"""Kernel-matrix pipeline — the north-star boundary (module kernel_pipeline).

Same operation names, argument meaning, orientation and error behaviour as SPEC's
``kernel_pipeline`` over the reference engine, so precomputed-kernel SVC training,
one-vs-rest multiclass and accuracy reporting downstream are unchanged:

  * :func:`enumerate_pairs`     SPEC.md:389-397 (1-based, strict upper triangle, row-major)
  * :func:`symmetrize`          SPEC.md:398-406 (K + K^T + I, precondition-checked)
  * :func:`compute_kernel_matrix`  SPEC.md:407-415 (train Gram, diagonal injected as 1.0)
  * :func:`compute_cross_kernel`   SPEC.md:416-424 (test x train, diagonal computed)
  * :func:`shard_merge`         SPEC.md:425-434 (deterministic placement, gap/overlap errors)

Underneath, the reference's ``contract_batch`` over a rebind-per-pair network
(engine.py:132-166) is replaced by libqk: one host sweep plan per structure, a per-sample
gate-build kernel and the pair-tiled sm_100a sweep.  Host (numpy) inputs go through the
C-ABI host entry points (H2D, sweep, D2H pipelined over row panels); CUDA torch tensors
stay on the device.  There is no CPU compute path.
"""
from __future__ import annotations

import atexit
import ctypes
import mmap
import os
from dataclasses import dataclass, field
from math import ceil, prod
from typing import Any, Iterable

import numpy as np

from . import _native
from .config import FeatureMapConfig, as_config, check_convention
from .errors import RebindError, ShardMergeError, StructuralError
from .planner import SweepPlan, plan_for


@dataclass
class KernelMatrix:
    """Dense real kernel block.

    ``entries`` is a row-major float64 ``numpy.ndarray`` of shape (rows, cols) — or a CUDA
    ``torch.Tensor`` when the inputs were device tensors.
    """

    rows: int
    cols: int
    entries: Any
    convention: str = "probability"
    metadata: dict = field(default_factory=dict)

    def __post_init__(self):
        shape = tuple(self.entries.shape)
        if shape != (self.rows, self.cols):
            raise StructuralError(f"entries shape {shape} != ({self.rows}, {self.cols})")
        check_convention(self.convention)

    def to_numpy(self) -> np.ndarray:
        e = self.entries
        if isinstance(e, np.ndarray):
            return e
        return e.detach().cpu().numpy()


# ---------------------------------------------------------------------------------------
# pair enumeration / symmetrisation / sharding (pure host logic)
# ---------------------------------------------------------------------------------------
def enumerate_pairs(n_a: int, n_b: int, symmetric: bool) -> list[tuple[int, int]]:
    """1-based pair indices: strict upper triangle of n_a x n_a (row-major) when symmetric,
    else the full n_a x n_b cross product."""
    if n_a < 1 or n_b < 1:
        raise ValueError("n_a and n_b must be >= 1")
    if symmetric:
        return [(i + 1, j + 1) for i in range(n_a) for j in range(i + 1, n_a)]
    return [(i + 1, j + 1) for i in range(n_a) for j in range(n_b)]


def symmetrize(upper: KernelMatrix) -> KernelMatrix:
    """K <- K + K^T + I for a strictly-upper matrix (Algorithm 2 step 5)."""
    if upper.rows != upper.cols:
        raise StructuralError(f"symmetrize needs a square matrix, got {upper.rows}x{upper.cols}")
    U = np.asarray(upper.to_numpy(), dtype=np.float64)
    if np.any(np.tril(U) != 0.0):
        raise StructuralError("symmetrize precondition violated: strictly-lower or diagonal "
                              "entries are nonzero (already symmetrised?)")
    K = U + U.T + np.eye(upper.rows)
    return KernelMatrix(upper.rows, upper.cols, K, upper.convention, dict(upper.metadata))


def shard_range(n_items: int, shard: int, n_shards: int) -> tuple[int, int]:
    """Contiguous ceil(P/W) shard of a linearised enumeration."""
    if n_shards < 1 or not 0 <= shard < n_shards:
        raise ValueError(f"bad shard spec {shard}/{n_shards}")
    size = ceil(n_items / n_shards) if n_items else 0
    lo = min(n_items, shard * size)
    return lo, min(n_items, lo + size)


def shard_merge(partials: Iterable[tuple[list, list]], n_a: int | None = None,
                n_b: int | None = None, symmetric: bool = True,
                convention: str = "probability", metadata: dict | None = None) -> KernelMatrix:
    """Place per-shard (pair list, value list) partials by pair index.

    Pair indices are 1-based as produced by :func:`enumerate_pairs`.  Overlaps and gaps in
    the coverage of the enumeration raise :class:`ShardMergeError` naming the pair.
    Symmetric merges are symmetrised (K + K^T + I)."""
    parts = [(list(p), list(v)) for p, v in partials]
    for k, (p, v) in enumerate(parts):
        if len(p) != len(v):
            raise ShardMergeError(f"shard {k}: {len(p)} pairs but {len(v)} values")
    allp = [pq for p, _ in parts for pq in p]
    if n_a is None:
        n_a = max((max(i, j) if symmetric else i) for i, j in allp) if allp else 1
    if n_b is None:
        n_b = n_a if symmetric else (max(j for _, j in allp) if allp else 1)
    K = np.zeros((n_a, n_b))
    seen = np.zeros((n_a, n_b), dtype=bool)
    for p, v in parts:
        for (i, j), val in zip(p, v):
            if not (1 <= i <= n_a and 1 <= j <= n_b) or (symmetric and i >= j):
                raise ShardMergeError(f"pair ({i}, {j}) is outside the enumeration")
            if seen[i - 1, j - 1]:
                raise ShardMergeError(f"shards overlap at pair ({i}, {j})")
            seen[i - 1, j - 1] = True
            K[i - 1, j - 1] = val
    mask = np.triu(np.ones((n_a, n_b), dtype=bool), k=1) if symmetric else \
        np.ones((n_a, n_b), dtype=bool)
    missing = np.argwhere(mask & ~seen)
    if len(missing):
        i, j = missing[0]
        raise ShardMergeError(f"shards leave a gap at pair ({i + 1}, {j + 1}) "
                              f"({len(missing)} missing)")
    km = KernelMatrix(n_a, n_b, K, convention, dict(metadata or {}))
    return symmetrize(km) if symmetric else km


# ---------------------------------------------------------------------------------------
# compute entry points
# ---------------------------------------------------------------------------------------
def _resolve_plan(cfg: FeatureMapConfig, plan, convention: str) -> SweepPlan:
    if isinstance(plan, SweepPlan):
        if (plan.width, plan.layers, plan.convention) != (cfg.width, cfg.layers, convention):
            raise StructuralError(
                f"plan for (width={plan.width}, layers={plan.layers}, {plan.convention}) does "
                f"not match config (width={cfg.width}, layers={cfg.layers}, {convention})")
        return plan
    # None or a reference PlanOptions: the sweep order is structural, options do not apply.
    return plan_for(cfg, convention)


def _check_workers(workers) -> None:
    if int(workers) < 1:
        raise ValueError("workers must be >= 1")


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


class _HostCache:
    """Recycles the large anonymous mappings behind result matrices.

    Results of at least ``QK_MAPPED_MIN_MB`` (default 1 MB) use it.  A fresh 960 MB result
    (config 4) costs page faults on first touch (taken by the copy-out
    pool while the sweep runs) and ~2 ms of munmap when the caller drops it — on the caller's
    critical path.  Mappings of dropped results are kept here (up to ``QK_HOST_CACHE_MB``,
    default 4096; 0 disables) and handed to the next result of the same size, already faulted
    in.  A result's numpy array holds its mapping through :class:`_Mapping`, whose finaliser
    runs only once every view of the array is gone.

    New mappings are also page-locked once (``qk_host_register``, ``QK_PIN_RESULTS=0``
    disables): the host pipelines then drain the results straight into them per 64-row tile
    row, as for caller-pinned buffers, instead of through the pinned staging pair and the copy
    pool (whose last panels trail the sweep by ~1 ms at config 4).  The registration cost is
    paid when the mapping is created and amortised by the recycling; a mapping is unregistered
    before it is unmapped.  Without a usable CUDA device the mapping simply stays pageable."""

    def __init__(self):
        import threading

        self.limit = int(os.environ.get("QK_HOST_CACHE_MB", "4096")) << 20
        self.pin = os.environ.get("QK_PIN_RESULTS", "1") != "0"
        self.pinned: dict[int, int] = {}  # id(mapping) -> registered address
        self.free: dict[int, list] = {}
        self.bytes = 0
        self.lock = threading.Lock()

    def get(self, nbytes: int):
        with self.lock:
            lst = self.free.get(nbytes)
            if lst:
                self.bytes -= nbytes
                return lst.pop()
        buf = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        try:
            buf.madvise(mmap.MADV_HUGEPAGE)
        except (AttributeError, OSError):  # pragma: no cover - platform without THP advice
            pass
        if self.pin:
            self._register(buf)
        return buf

    def _register(self, buf) -> None:
        # a failed registration (no CUDA device, locked-memory limit) leaves a pageable result,
        # which the pipelines drain correctly through the staging pair
        lib = _native.lib()  # NativeLibraryError propagates: there is no engine without it
        _native.bind_current_device()
        c = ctypes.c_char.from_buffer(buf)
        addr = ctypes.addressof(c)
        del c  # release the export (the mapping must stay closable)
        if lib.qk_host_register(ctypes.c_void_p(addr), ctypes.c_size_t(len(buf))) == 0:
            self.pinned[id(buf)] = addr

    def _release(self, buf) -> None:
        addr = self.pinned.pop(id(buf), None)
        if addr is not None and _native.lib().qk_host_unregister(ctypes.c_void_p(addr)) != 0:
            return  # still registered: leave it mapped rather than unmap locked pages
        buf.close()

    def drop_all(self) -> None:
        """Unregister and unmap every cached mapping (atexit, before CUDA tears down)."""
        with self.lock:
            bufs = [b for lst in self.free.values() for b in lst]
            self.free.clear()
            self.bytes = 0
        for b in bufs:
            self._release(b)

    def put(self, buf) -> None:
        n = len(buf)
        with self.lock:
            if self.bytes + n <= self.limit:
                self.free.setdefault(n, []).append(buf)
                self.bytes += n
                return
        self._release(buf)


_host_cache = _HostCache()
# results from this size up come from the cache (QK_MAPPED_MIN_MB, default 1): page-locked,
# they drain per tile row (config 2's default call measured 1.19 -> 0.42 ms, config 3's 4.31
# -> 3.81 ms against the staged drain into np.empty results; profiles/r2/configs_e2e_r2l.jsonl)
_MAPPED_MIN = int(float(os.environ.get("QK_MAPPED_MIN_MB", "1")) * (1 << 20))
atexit.register(_host_cache.drop_all)


class _Mapping:
    """Buffer-protocol owner of one cached mapping (numpy keeps it as the array's base)."""

    __slots__ = ("buf",)

    def __init__(self, buf):
        self.buf = buf

    def __buffer__(self, flags):
        return memoryview(self.buf)

    def __release_buffer__(self, view):
        view.release()

    def __del__(self):
        cache = _host_cache
        if cache is not None and self.buf is not None:
            cache.put(self.buf)
            self.buf = None


def host_empty(shape) -> np.ndarray:
    """Uninitialised float64 host array; large ones are anonymous mappings advised to use
    transparent huge pages (the first touch by the copy-out pool faults 2 MB at a time),
    recycled through :class:`_HostCache` once the caller drops them."""
    nbytes = prod(shape) * 8
    if nbytes < _MAPPED_MIN:
        return np.empty(shape, dtype=np.float64)
    return np.frombuffer(_Mapping(_host_cache.get(nbytes)), dtype=np.float64).reshape(shape)


def _host_angles(x, width: int) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.ndim == 1 and a.size == 0:
        a = a.reshape(0, width)
    if a.ndim != 2:
        raise RebindError(f"operand set 0: expected a 2-D feature array, got shape {a.shape}")
    return a


def _width_error(w_a: int, w_b: int, width: int) -> RebindError:
    # engine.py:139-144
    return RebindError(f"operand set 0: vectors of lengths {w_a}/{w_b} do not match width "
                       f"{width}")


def _first_bad_gram_pair(X: np.ndarray) -> int:
    bad = np.flatnonzero(~np.isfinite(X).all(axis=1))
    s = int(bad[0])
    return 0 if s == 0 else s - 1  # pair (0, s) is the first containing s, row-major


def _first_bad_cross_pair(T: np.ndarray, R: np.ndarray) -> int:
    cands = []
    bt = np.flatnonzero(~np.isfinite(T).all(axis=1))
    br = np.flatnonzero(~np.isfinite(R).all(axis=1))
    if len(bt):
        cands.append(int(bt[0]) * R.shape[0])
    if len(br):
        cands.append(int(br[0]))
    return min(cands)


def _metadata(cfg: FeatureMapConfig, plan: SweepPlan, dataset_id, kind: str) -> dict:
    return {"qubits": cfg.width, "layers": cfg.layers, "dataset": dataset_id,
            "config_hash": cfg.config_hash(), "kind": kind, "engine": "libqk sm_100a",
            "plan": dict(plan.info)}


def compute_kernel_matrix(features, cfg, plan=None, workers: int = 1, *,
                          convention: str = "probability", dataset_id: str | None = None,
                          out: np.ndarray | None = None) -> KernelMatrix:
    """Train Gram matrix K(x_i, x_j) = |<0|U(x_i)^dag U(x_j)|0>|^2.

    The strict upper triangle is contracted, mirrored, and the diagonal injected as exactly
    1.0.  ``plan`` may be None, a :class:`SweepPlan`, or the reference's PlanOptions (the
    sweep order is structural, so path options do not apply).  ``workers`` is accepted for
    signature compatibility (>= 1); one process drives one GPU — multi-GPU runs go through
    :mod:`paper_2405_02630_b200.distributed`.  ``out`` may supply a preallocated (e.g.
    pinned) C-contiguous float64 (N, N) host array to receive the entries."""
    cfg = as_config(cfg)
    convention = check_convention(convention)
    _check_workers(workers)
    sp = _resolve_plan(cfg, plan, convention)
    if _is_cuda_tensor(features):
        return _compute_kernel_matrix_device(features, cfg, sp, convention, dataset_id)
    X = _host_angles(features, cfg.width)
    N = X.shape[0]
    if N >= 2 and X.shape[1] != cfg.width:
        raise _width_error(X.shape[1], X.shape[1], cfg.width)
    if out is None:
        out = host_empty((N, N))
    elif out.shape != (N, N) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float64 array of shape ({N}, {N})")
    if N == 1:
        out[0, 0] = 1.0
    elif N >= 2:
        _native.bind_current_device()
        status = _native.lib().qk_kernel_matrix_host(sp.handle, X.ctypes.data, N,
                                                     out.ctypes.data)
        if status == _native.QK_ERR_REBIND:
            raise RebindError(f"operand set {_first_bad_gram_pair(X)}: feature angles must be "
                              "finite")
        _native.check(status)
    return KernelMatrix(N, N, out, convention, _metadata(cfg, sp, dataset_id, "gram"))


def compute_cross_kernel(test, train, cfg, plan=None, workers: int = 1, *,
                         convention: str = "probability", dataset_id: str | None = None,
                         out: np.ndarray | None = None) -> KernelMatrix:
    """Test-versus-train block K[r][c] = k(test_r, train_c).

    Full rectangle, rows = test, no symmetrisation, diagonal computed (not injected)."""
    cfg = as_config(cfg)
    convention = check_convention(convention)
    _check_workers(workers)
    sp = _resolve_plan(cfg, plan, convention)
    if _is_cuda_tensor(test) or _is_cuda_tensor(train):
        return _compute_cross_kernel_device(test, train, cfg, sp, convention, dataset_id)
    T = _host_angles(test, cfg.width)
    R = _host_angles(train, cfg.width)
    Nt, Nr = T.shape[0], R.shape[0]
    if Nt and Nr and (T.shape[1] != cfg.width or R.shape[1] != cfg.width):
        raise _width_error(T.shape[1], R.shape[1], cfg.width)
    if out is None:
        out = host_empty((Nt, Nr))
    elif out.shape != (Nt, Nr) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float64 array of shape ({Nt}, {Nr})")
    if Nt and Nr:
        _native.bind_current_device()
        status = _native.lib().qk_cross_kernel_host(sp.handle, T.ctypes.data, Nt,
                                                     R.ctypes.data, Nr, out.ctypes.data)
        if status == _native.QK_ERR_REBIND:
            raise RebindError(f"operand set {_first_bad_cross_pair(T, R)}: feature angles "
                              "must be finite")
        _native.check(status)
    return KernelMatrix(Nt, Nr, out, convention, _metadata(cfg, sp, dataset_id, "cross"))


def compute_kernel_matrices(train, test, cfg, plan=None, workers: int = 1, *,
                            convention: str = "probability", dataset_id: str | None = None,
                            out_train: np.ndarray | None = None,
                            out_test: np.ndarray | None = None):
    """The QSVM train/test kernel pair of Algorithm 2 in one call:
    ``(compute_kernel_matrix(train), compute_cross_kernel(test, train))`` with identical
    results, computed as ONE sweep over the joint tile list (one upload of the train angles,
    both matrices drained to the host while the sweep runs)."""
    cfg = as_config(cfg)
    convention = check_convention(convention)
    _check_workers(workers)
    sp = _resolve_plan(cfg, plan, convention)
    if _is_cuda_tensor(train) or _is_cuda_tensor(test):
        return (_compute_kernel_matrix_device(train, cfg, sp, convention, dataset_id),
                _compute_cross_kernel_device(test, train, cfg, sp, convention, dataset_id))
    R = _host_angles(train, cfg.width)
    T = _host_angles(test, cfg.width)
    Nr, Nt = R.shape[0], T.shape[0]
    if Nr and (R.shape[1] != cfg.width or (Nt and T.shape[1] != cfg.width)):
        raise _width_error(R.shape[1], T.shape[1] if Nt else R.shape[1], cfg.width)
    K = host_empty((Nr, Nr)) if out_train is None else out_train
    Kx = host_empty((Nt, Nr)) if out_test is None else out_test
    for arr, shape in ((K, (Nr, Nr)), (Kx, (Nt, Nr))):
        if arr.shape != shape or arr.dtype != np.float64 or not arr.flags.c_contiguous:
            raise ValueError(f"outputs must be C-contiguous float64 arrays of shape {shape}")
    if Nr == 1:
        K[0, 0] = 1.0
    if Nr >= 2 or (Nr and Nt):
        _native.bind_current_device()
        status = _native.lib().qk_kernel_matrices_host(sp.handle, R.ctypes.data, Nr,
                                                       T.ctypes.data, Nt, K.ctypes.data,
                                                       Kx.ctypes.data)
        if status == _native.QK_ERR_REBIND:
            if not np.isfinite(R).all() and Nr >= 2:
                raise RebindError(f"operand set {_first_bad_gram_pair(R)}: feature angles "
                                  "must be finite")
            raise RebindError(f"operand set {_first_bad_cross_pair(T, R)}: feature angles "
                              "must be finite")
        _native.check(status)
        if Nr == 1:
            K[0, 0] = 1.0
    return (KernelMatrix(Nr, Nr, K, convention, _metadata(cfg, sp, dataset_id, "gram")),
            KernelMatrix(Nt, Nr, Kx, convention, _metadata(cfg, sp, dataset_id, "cross")))


# ---------------------------------------------------------------------------------------
# device-resident variants (CUDA torch tensors in -> CUDA torch tensor entries)
# ---------------------------------------------------------------------------------------
def _compute_kernel_matrix_device(features, cfg, sp, convention, dataset_id) -> KernelMatrix:
    import torch

    from . import device as dev

    X = dev.angles_to_device(features)
    if X.dim() != 2:
        raise RebindError(f"operand set 0: expected a 2-D feature array, got shape "
                          f"{tuple(X.shape)}")
    N = X.shape[0]
    if N >= 2 and X.shape[1] != cfg.width:
        raise _width_error(X.shape[1], X.shape[1], cfg.width)
    if N < 2:
        K = torch.ones((N, N), dtype=torch.float64, device=X.device)
        return KernelMatrix(N, N, K, convention, _metadata(cfg, sp, dataset_id, "gram"))
    planes = dev.gate_build(sp, X)
    K = dev.gram(planes)
    bad = planes.bad_sample()
    if bad is not None:
        raise RebindError(f"operand set {0 if bad == 0 else bad - 1}: feature angles must be "
                          "finite")
    return KernelMatrix(N, N, K, convention, _metadata(cfg, sp, dataset_id, "gram"))


def _compute_cross_kernel_device(test, train, cfg, sp, convention, dataset_id) -> KernelMatrix:
    import torch

    from . import device as dev

    T = dev.angles_to_device(test)
    R = dev.angles_to_device(train, device=T.device)
    Nt, Nr = T.shape[0], R.shape[0]
    if Nt and Nr and (T.shape[1] != cfg.width or R.shape[1] != cfg.width):
        raise _width_error(T.shape[1], R.shape[1], cfg.width)
    if not (Nt and Nr):
        K = torch.empty((Nt, Nr), dtype=torch.float64, device=T.device)
        return KernelMatrix(Nt, Nr, K, convention, _metadata(cfg, sp, dataset_id, "cross"))
    pt = dev.gate_build(sp, T)
    pr = dev.gate_build(sp, R)
    K = dev.cross(pt, pr)
    bt, br = pt.bad_sample(), pr.bad_sample()
    if bt is not None or br is not None:
        cands = ([bt * Nr] if bt is not None else []) + ([br] if br is not None else [])
        raise RebindError(f"operand set {min(cands)}: feature angles must be finite")
    return KernelMatrix(Nt, Nr, K, convention, _metadata(cfg, sp, dataset_id, "cross"))


# ---------------------------------------------------------------------------------------
# shard-run-then-merge (CLI `--shard k/W`)
# ---------------------------------------------------------------------------------------
def compute_kernel_shard(features, cfg, shard: int, n_shards: int, *, test=None,
                         convention: str = "probability"):
    """Values of shard k (0-based) of W: the contiguous ceil(P/W) range of the row-major pair
    enumeration (strict upper triangle of the train Gram, or the test x train rectangle when
    ``test`` is given).  Returns ``(pair_range, values)``; merging every shard's partial
    (container.merge_partials) reproduces compute_kernel_matrix / compute_cross_kernel bit
    for bit — the pair-list kernel runs the sweep's exact arithmetic."""
    import torch

    from . import device as dev
    from .container import enumeration_pairs, shard_pair_range

    cfg = as_config(cfg)
    convention = check_convention(convention)
    sp = plan_for(cfg, convention)
    X = _host_angles(features, cfg.width) if not _is_cuda_tensor(features) else features
    T = None if test is None else (_host_angles(test, cfg.width) if not _is_cuda_tensor(test)
                                   else test)
    symmetric = T is None
    n_a = (X.shape[0] if symmetric else T.shape[0])
    n_b = X.shape[0]
    lo, hi = shard_pair_range(n_a, n_b, symmetric, shard, n_shards)
    if hi <= lo:
        return (lo, hi), np.empty(0)
    pairs = torch.as_tensor(enumeration_pairs(n_a, n_b, symmetric, lo, hi), device="cuda")
    px = dev.gate_build(sp, dev.angles_to_device(X))
    pa = px if symmetric else dev.gate_build(sp, dev.angles_to_device(T))
    vals = dev.pair_kernel_values(pa, px, pairs)  # |amp|^2 or |amp| in the pair kernel
    bad = [b for b in (px.bad_sample(), None if symmetric else pa.bad_sample()) if b is not None]
    if bad:
        raise RebindError("feature angles must be finite")
    return (lo, hi), vals.cpu().numpy()
