"""Multi-GPU sharding of the kernel-matrix job: one process per GPU.

The reference parallelises over pairs only — a fork pool in code (engine.py:159-166),
shard-run-then-merge in SPEC, MPI + NCCL across A100s in the paper
(PAPER.md:359-362).  Here the unit is the sweep tile: the job's linearised tile list (train
Gram upper-triangle tiles, then test x train cross tiles) is split into contiguous ranges of
equal estimated cost (SPEC's contiguous ceil(P/W) rule at tile granularity; tile_costs).  Each
rank builds the gate planes of every sample (cheap) and
sweeps its range.  Two ways to land the results on rank 0:

* ``placement="p2p"`` (default): rank 0 allocates the dense matrices and exports them over
  CUDA IPC; every rank's sweep kernel stores its tiles — and their mirror — straight into
  rank 0's memory over NVLink / NVSwitch while it computes.  Completion is one barrier.  No
  gather buffer, no unpack: the collective is fused into the compute kernel's epilogue.
* ``placement="gather"``: packed tiles padded to the common range length, one ``gather`` to
  rank 0 (NCCL), then the unpack kernel.  For fabrics without peer access.

Host buffers (``KernelJob.run_host``): the inputs go up per rank, the p2p job runs, and each
rank then copies ITS row slice of rank 0's matrices into a host matrix every rank maps
(:class:`SharedHostMatrix`, a POSIX shared-memory segment page-locked in each process), so
the 8 B/entry result leaves the GPUs over N PCIe links in parallel.

World size 1 writes the dense matrices directly.  The partition / placement logic is
device-agnostic (tested with gloo on CPU); the p2p path is tested with two processes sharing
one GPU (CUDA IPC works within a device), the sweeps/unpacks by the GPU parity tests.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from math import ceil
from multiprocessing import shared_memory

import numpy as np

import torch
import torch.distributed as dist

from . import _native
from .errors import RebindError
from .kernel_pipeline import shard_range
from .planner import SweepPlan


def _log(msg: str) -> None:
    import sys

    print(f"[qk] {msg}", file=sys.stderr, flush=True)


def device_bus_id() -> str:
    """PCI bus id of the current device (names it across processes with different orderings)."""
    _native.bind_current_device()
    buf = ctypes.create_string_buffer(32)
    _native.check(_native.lib().qk_device_bus_id(buf))
    return buf.value.decode()


def can_reach(bus_id: str) -> bool:
    """Whether this process's current device can store into the device with ``bus_id``."""
    _native.bind_current_device()
    out = ctypes.c_int32(0)
    _native.check(_native.lib().qk_can_reach(bus_id.encode(), ctypes.byref(out)))
    return bool(out.value)


def agree_placement(reachable: bool, group=None) -> bool:
    """All ranks agree on the p2p placement only if every rank can reach rank 0's memory
    (one MIN all-reduce; a gloo group reduces on the CPU)."""
    flag = torch.tensor([1.0 if reachable else 0.0], dtype=torch.float64,
                        device="cpu" if dist.get_backend(group) == "gloo" else "cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item() >= 1.0)


@dataclass(frozen=True)
class Segment:
    """A contiguous run of one tile list inside a rank's union range."""

    kind: str          # "gram" or "cross"
    tile_begin: int    # within that list
    tile_end: int
    offset: int        # tile offset inside the rank's packed buffer


@dataclass(frozen=True)
class JobLayout:
    n_train: int
    n_test: int
    gram_tiles: int
    cross_tiles: int
    world: int
    tile_elems: int
    bounds: tuple = ()  # world + 1 tile-list boundaries (cost-balanced); () = equal counts

    @property
    def total_tiles(self) -> int:
        return self.gram_tiles + self.cross_tiles

    @property
    def range_len(self) -> int:
        if not self.total_tiles:
            return 0
        return max(hi - lo for lo, hi in (self.union_range(r) for r in range(self.world)))

    def union_range(self, rank: int) -> tuple[int, int]:
        if self.bounds:
            return self.bounds[rank], self.bounds[rank + 1]
        return shard_range(self.total_tiles, rank, self.world)

    def segments(self, rank: int) -> list[Segment]:
        lo, hi = self.union_range(rank)
        segs = []
        g_lo, g_hi = lo, min(hi, self.gram_tiles)
        if g_hi > g_lo:
            segs.append(Segment("gram", g_lo, g_hi, 0))
        c_lo, c_hi = max(lo, self.gram_tiles), hi
        if c_hi > c_lo:
            segs.append(Segment("cross", c_lo - self.gram_tiles, c_hi - self.gram_tiles,
                                c_lo - lo))
        return segs

    def entries(self) -> int:
        """Kernel entries the job defines: strict-upper Gram + full cross (the metric unit)."""
        return self.n_train * (self.n_train - 1) // 2 + self.n_test * self.n_train

    def rank_entries(self, rank: int) -> int:
        """Entries inside this rank's tile range (its share of the metric)."""
        lo, hi = self.union_range(rank)
        edge = int(round(self.tile_elems ** 0.5))
        return int(tile_entries(self.n_train, self.n_test, edge)[lo:hi].sum())


def _pad(n: int, edge: int) -> int:
    return (edge - n % edge) % edge


def tile_costs(n_train: int, n_test: int, edge: int, group: int = 8) -> np.ndarray:
    """Relative sweep cost of every tile of the joint list (Gram then cross, both in the
    kernel's grouped orders; qk_sweep.cu decode_upper / decode_rect): 1, except the tiles of
    tile row 0, whose front padding rows skip the sweep in whole 4-row warps (16 real rows of
    64 cost ~1/4 of a tile, measured)."""
    nb = -(-n_train // edge) if n_train else 0
    nbt = -(-n_test // edge) if n_test else 0
    w = np.ones(nb * (nb + 1) // 2 + nbt * nb)
    def row0_weight(n):
        pad = _pad(n, edge)
        return -(-(edge - pad) // 4) / (edge // 4)
    if nb:
        h = min(group, nb)
        cols = np.arange(nb)
        idx = np.where(cols < h, cols * (cols + 1) // 2, h * (h + 1) // 2 + h * (cols - h))
        w[idx] = row0_weight(n_train)  # Gram tile row 0 lies in super-row 0
    if nbt:
        g0 = nb * (nb + 1) // 2
        bi, _ = rect_tile_coords(nbt, nb)
        w[g0 + np.flatnonzero(bi == 0)] = row0_weight(n_test)  # cross tile row 0 (test block 0)
    return w


RECT_GROUP, RECT_TAIL = 8, 2  # qk_internal.h kRectGroup / kRectTail


def rect_tile_coords(nb_rows: int, nb_cols: int) -> tuple[np.ndarray, np.ndarray]:
    """(bi, bj) of every cross tile in the sweep kernel's list order (qk_sweep.cu decode_rect:
    super-rows of RECT_GROUP tile rows walked column by column, the last RECT_TAIL rows
    row-major)."""
    grouped = nb_rows - RECT_TAIL if nb_rows > RECT_TAIL else 0
    bis, bjs = [], []
    for r0 in range(0, grouped, RECT_GROUP):
        h = min(RECT_GROUP, grouped - r0)
        bis.append(np.tile(np.arange(r0, r0 + h), nb_cols))
        bjs.append(np.repeat(np.arange(nb_cols), h))
    for r in range(grouped, nb_rows):
        bis.append(np.full(nb_cols, r))
        bjs.append(np.arange(nb_cols))
    if not bis:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(bis).astype(np.int64), np.concatenate(bjs).astype(np.int64)


def gram_tile_coords(nb: int, group: int = 8) -> tuple[np.ndarray, np.ndarray]:
    """(bi, bj) of every Gram tile in the sweep kernel's list order (qk_sweep.cu decode_upper:
    super-rows of `group` tile rows, each walked column by column)."""
    bis, bjs = [], []
    for r0 in range(0, nb, group):
        h = min(group, nb - r0)
        for c in range(h):  # the super-row's triangle: column r0 + c holds rows r0..r0+c
            bis.append(np.arange(r0, r0 + c + 1))
            bjs.append(np.full(c + 1, r0 + c))
        cols = np.arange(r0 + h, nb)  # then full columns of h rows
        bis.append(np.tile(np.arange(r0, r0 + h), len(cols)))
        bjs.append(np.repeat(cols, h))
    if not bis:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(bis).astype(np.int64), np.concatenate(bjs).astype(np.int64)


def tile_entries(n_train: int, n_test: int, edge: int) -> np.ndarray:
    """Kernel entries (the metric unit: strict-upper Gram pairs, cross pairs) inside every
    tile of the joint list, in list order — for per-rank accounting of cost-balanced ranges."""
    def real(n):  # real samples per plane block (the ragged remainder fills block 0's end)
        nb = -(-n // edge) if n else 0
        r = np.full(nb, edge, dtype=np.int64)
        if nb:
            r[0] = edge - _pad(n, edge)
        return r
    rt = real(n_train)
    bi, bj = gram_tile_coords(len(rt))
    gram = np.where(bi == bj, rt[bi] * (rt[bi] - 1) // 2, rt[bi] * rt[bj])
    rs = real(n_test)
    ci, cj = rect_tile_coords(len(rs), len(rt))
    cross = rs[ci] * rt[cj]
    return np.concatenate([gram, cross])


def layout_for(plan: SweepPlan, n_train: int, n_test: int, world: int) -> JobLayout:
    """The job's tile list split into contiguous per-rank ranges of equal estimated COST
    (tile_costs): the ranks holding the cheap padding tile rows take more tiles."""
    edge = plan.tile_edge
    gram = plan.gram_tile_count(n_train)
    cross = plan.cross_tile_count(n_test, n_train) if n_test else 0
    bounds = ()
    if world > 1 and gram + cross:
        cum = np.concatenate([[0.0], np.cumsum(tile_costs(n_train, n_test, edge))])
        targets = cum[-1] * np.arange(world + 1) / world
        b = np.searchsorted(cum, targets, side="left")
        b[0], b[-1] = 0, gram + cross
        bounds = tuple(int(x) for x in np.maximum.accumulate(b))
    return JobLayout(n_train, n_test, gram, cross, world, edge * edge, bounds)


def gather_packed(local: torch.Tensor, layout: JobLayout, group=None) -> list | None:
    """Gather every rank's padded packed buffer to rank 0 (one collective).  gloo has no
    CUDA gather, so a gloo group moves the buffers through host memory."""
    rank = dist.get_rank(group)
    if layout.world == 1:
        return [local]
    src = local
    if dist.get_backend(group) == "gloo" and local.is_cuda:
        src = local.cpu()
    bufs = [torch.empty_like(src) for _ in range(layout.world)] if rank == 0 else None
    dist.gather(src, bufs, dst=0, group=group)
    if bufs is not None and local.is_cuda:
        bufs = [b.to(local.device) for b in bufs]
    return bufs


class SharedMatrix:
    """Dense row-major fp64 matrix in device memory that peer processes can store into.

    The owner allocates it with ``qk_shared_alloc`` and exports a CUDA IPC handle; peers
    import the handle and get a device address of the same memory (over NVLink when the
    owner is another GPU).  The owner's view is also a torch tensor (``tensor``)."""

    def __init__(self, rows: int, cols: int, handle: bytes | None = None):
        self.rows, self.cols = int(rows), int(cols)
        self.owner = handle is None
        lib = _native.lib()
        _native.bind_current_device()
        p = ctypes.c_void_p()
        if self.owner:
            _native.check(lib.qk_shared_alloc(max(1, self.rows * self.cols) * 8,
                                              ctypes.byref(p)))
        else:
            _native.check(lib.qk_ipc_import(handle, ctypes.byref(p)))
        self.ptr = int(p.value)
        self.__cuda_array_interface__ = {"shape": (self.rows, self.cols), "typestr": "<f8",
                                         "data": (self.ptr, False), "version": 3,
                                         "strides": None}

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _native.check(_native.lib().qk_ipc_export(self.ptr, buf))
        return buf.raw

    def tensor(self) -> torch.Tensor:
        assert self.owner, "only the owner views the matrix as a tensor"
        return torch.as_tensor(self, device=torch.device("cuda", torch.cuda.current_device()))

    def close(self) -> None:
        if self.ptr and _native._lib is not None:
            lib = _native._lib
            (lib.qk_shared_free if self.owner else lib.qk_ipc_close)(self.ptr)
        self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class SharedHostMatrix:
    """Row-major fp64 host matrix shared by the rank processes of one node: a POSIX
    shared-memory segment (or, when /dev/shm is too small for it, a file under the temp
    directory mapped MAP_SHARED) that rank 0 creates (``name=None``) and the others attach by
    name, page-locked in every process (``qk_host_register``) so each rank's copy engine can
    DMA its slice of the result into it.  ``array`` is the numpy view."""

    def __init__(self, rows: int, cols: int, name: str | None = None):
        import mmap
        import os
        import tempfile

        self.rows, self.cols = int(rows), int(cols)
        nbytes = max(8, self.rows * self.cols * 8)
        self.owner = name is None
        self._shm = self._file = None
        if self.owner:
            try:
                st = os.statvfs("/dev/shm")
                use_shm = st.f_bavail * st.f_frsize >= nbytes + (64 << 20)
            except OSError:
                use_shm = False
            if use_shm:
                self._shm = shared_memory.SharedMemory(create=True, size=nbytes)
                self.name = "shm:" + self._shm.name
            else:
                fd, path = tempfile.mkstemp(prefix="qk_host_", suffix=".f64")
                os.ftruncate(fd, nbytes)
                self._file = (fd, path)
                self.name = "file:" + path
        else:
            kind, _, ident = name.partition(":")
            if kind == "shm":
                self._shm = shared_memory.SharedMemory(name=ident, create=False)
                try:  # the creator unlinks it; keep this process's tracker out of it
                    from multiprocessing import resource_tracker
                    resource_tracker.unregister(self._shm._name, "shared_memory")
                except Exception:  # pragma: no cover - tracker internals differ
                    pass
            else:
                self._file = (os.open(ident, os.O_RDWR), ident)
            self.name = name
        if self._shm is not None:
            buf = self._shm.buf
        else:
            self._map = mmap.mmap(self._file[0], nbytes, flags=mmap.MAP_SHARED)
            buf = self._map
        self.array = np.ndarray((self.rows, self.cols), dtype=np.float64, buffer=buf)
        self._ptr = self.array.ctypes.data
        self._nbytes = nbytes
        _native.bind_current_device()
        _native.check(_native.lib().qk_host_register(self._ptr, nbytes))
        self._registered = True

    def close(self) -> None:
        import os

        if getattr(self, "_registered", False) and _native._lib is not None:
            _native._lib.qk_host_unregister(self._ptr)
            self._registered = False
        self.array = None
        if getattr(self, "_shm", None) is not None:
            self._shm.close()
            if self.owner:
                try:
                    self._shm.unlink()
                except FileNotFoundError:  # pragma: no cover
                    pass
            self._shm = None
        if getattr(self, "_file", None) is not None:
            self._map.close()
            os.close(self._file[0])
            if self.owner:
                try:
                    os.unlink(self._file[1])
                except FileNotFoundError:  # pragma: no cover
                    pass
            self._file = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class KernelJob:
    """Train Gram (+ optional test x train cross block) over a process group."""

    def __init__(self, plan: SweepPlan, n_train: int, n_test: int = 0, group=None,
                 placement: str = "p2p", graph_mode: bool | None = None):
        if placement not in ("p2p", "gather"):
            raise ValueError(f"unknown placement {placement!r}")
        self.graph_mode = graph_mode  # None: auto (small single-GPU jobs replay a graph)
        self.plan = plan
        self.group = group
        self.placement = placement
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.layout = layout_for(plan, n_train, n_test, self.world)
        self.packed = None
        self.K_train = None
        self.K_cross = None
        self._shared = None
        self._bad = None             # [3] int64 job state: non-finite sentinels (train, test),
                                     # qk_job_run's tile-claim counter
        self._planes = [None, None]  # gate-plane buffers reused across runs
        self._g = None               # captured single-GPU job (small jobs)

    # ---- world size 1 ----------------------------------------------------------------
    def _run_local(self, p_train, p_test, devc):
        from . import device as dev

        lay = self.layout
        if self.K_train is None:
            self.K_train = torch.empty((lay.n_train, lay.n_train), dtype=torch.float64,
                                       device=devc)
            if lay.n_test:
                self.K_cross = torch.empty((lay.n_test, lay.n_train), dtype=torch.float64,
                                           device=devc)
        dev.job_into(p_train, p_test, self.K_train.data_ptr(),
                     self.K_cross.data_ptr() if lay.n_test else 0)
        return self.K_train, self.K_cross

    # ---- p2p placement: sweeps store into rank 0's matrices ----------------------------
    def _setup_shared(self):
        """Collective: rank 0 allocates and exports the matrices with its device's PCI bus id;
        every other rank checks it can store into that device (qk_can_reach: the same device,
        or peer access) and imports the handles.  All ranks then agree on the placement: any
        rank without a path to rank 0's memory sends everyone to the gather placement.  A
        failing import on a rank that CAN reach rank 0 is a bug and is raised, not hidden."""
        lay = self.layout
        if self.rank == 0:
            mats = [SharedMatrix(lay.n_train, lay.n_train)]
            if lay.n_test:
                mats.append(SharedMatrix(lay.n_test, lay.n_train))
            payload = ([m.export() for m in mats], device_bus_id())
        else:
            mats, payload = [], None
        box = [payload]
        dist.broadcast_object_list(box, src=0, group=self.group)
        handles, owner_bus = box[0]
        reach = True if self.rank == 0 else can_reach(owner_bus)
        if reach and self.rank != 0:
            shapes = [(lay.n_train, lay.n_train), (lay.n_test, lay.n_train)]
            mats = [SharedMatrix(r, c, handle=h) for (r, c), h in zip(shapes, handles)]
        if not agree_placement(reach, self.group):
            for m in mats:
                m.close()
            self.placement = "gather"
            if self.rank == 0:
                _log(f"placement: gather (a rank cannot store into {owner_bus})")
            return False
        self._shared = mats
        if self.rank == 0:
            self.K_train = mats[0].tensor()
            self.K_cross = mats[1].tensor() if lay.n_test else None
            _log(f"placement: p2p, {self.world} ranks store into rank 0's matrices on "
                 f"{owner_bus}")
        return True

    def _run_p2p(self, p_train, p_test, devc):
        from . import device as dev

        if self._shared is None and not self._setup_shared():
            return self._run_gather(p_train, p_test, devc)
        lay = self.layout
        lo, hi = lay.union_range(self.rank)  # one launch over this rank's joint tile range
        # rank 0 may still be reading the matrices it returned from the previous run (they
        # alias the shared memory): nobody stores until every rank has entered this run and
        # drained its stream
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)
        dev.job_into(p_train, p_test, self._shared[0].ptr,
                     self._shared[1].ptr if lay.n_test else 0, lo, hi)
        torch.cuda.current_stream().synchronize()  # this rank's stores have landed
        dist.barrier(group=self.group)
        if self.rank != 0:
            return None, None
        return self.K_train, self.K_cross

    # ---- gather placement --------------------------------------------------------------
    def _run_gather(self, p_train, p_test, devc):
        from . import device as dev

        lay = self.layout
        if self.packed is None:
            self.packed = torch.empty(max(lay.range_len, 1) * lay.tile_elems,
                                      dtype=torch.float64, device=devc)
        for seg in lay.segments(self.rank):
            view = self.packed[seg.offset * lay.tile_elems:
                               (seg.offset + seg.tile_end - seg.tile_begin) * lay.tile_elems]
            if seg.kind == "gram":
                dev.gram(p_train, out=view, tile_begin=seg.tile_begin, tile_end=seg.tile_end,
                         packed=True)
            else:
                dev.cross(p_test, p_train, out=view, tile_begin=seg.tile_begin,
                          tile_end=seg.tile_end, packed=True)
        bufs = gather_packed(self.packed, lay, self.group)
        if self.rank != 0:
            return None, None
        if self.K_train is None:
            self.K_train = torch.empty((lay.n_train, lay.n_train), dtype=torch.float64,
                                       device=devc)
            if lay.n_test:
                self.K_cross = torch.empty((lay.n_test, lay.n_train), dtype=torch.float64,
                                           device=devc)
        for r, buf in enumerate(bufs):
            for seg in lay.segments(r):
                view = buf[seg.offset * lay.tile_elems:
                           (seg.offset + seg.tile_end - seg.tile_begin) * lay.tile_elems]
                if seg.kind == "gram":
                    dev.unpack_gram(self.plan, view, lay.n_train, seg.tile_begin, seg.tile_end,
                                    self.K_train)
                else:
                    dev.unpack_cross(self.plan, view, lay.n_test, lay.n_train, seg.tile_begin,
                                     seg.tile_end, self.K_cross)
        return self.K_train, self.K_cross

    # Jobs below this many entry-qubits (~1 ms of sweep) replay a CUDA graph by default: the
    # per-call host work of the eager path (~30-50 us) is comparable with the job itself.
    GRAPH_ENTRY_QUBITS = 2e9

    def run(self, train_angles: torch.Tensor, test_angles: torch.Tensor | None = None,
            check_finite: bool = True):
        """Returns (K_train, K_cross) on rank 0 (device tensors), (None, None) elsewhere.

        Single-GPU jobs of up to ~1 ms (``GRAPH_ENTRY_QUBITS``, unless ``graph_mode=False``)
        run as a CUDA-graph replay of one qk_job_run (sentinel reset, both gate builds in
        one launch, the sweep) after the inputs are copied into job-owned buffers.
        ``check_finite`` (default) synchronises once to raise the reference's RebindError for
        a non-finite angle; pass False to keep the call asynchronous."""
        from . import device as dev

        capturing = torch.cuda.is_current_stream_capturing()
        if self.world == 1 and not capturing and self._graph_eligible():
            self._run_graph(train_angles, test_angles)
            if check_finite:
                self._check_finite(self.layout.n_test > 0)
            return self.K_train, self.K_cross
        devc = train_angles.device
        if self._bad is None or self._bad.device != devc:
            self._bad = torch.empty(3, dtype=torch.int64, device=devc)
            self._planes = [None, None]
        self._bad.fill_(-1)  # both plane sets' non-finite sentinels, one fill
        p_train = dev.gate_build(self.plan, train_angles, out=self._planes[0],
                                 bad=self._bad[0:1])
        self._planes[0] = p_train.buf
        p_test = None
        if self.layout.n_test:
            p_test = dev.gate_build(self.plan, test_angles, out=self._planes[1],
                                    bad=self._bad[1:2])
            self._planes[1] = p_test.buf
        if self.world == 1:
            out = self._run_local(p_train, p_test, devc)
        elif self.placement == "p2p":
            out = self._run_p2p(p_train, p_test, devc)
        else:
            out = self._run_gather(p_train, p_test, devc)
        if check_finite and not capturing:
            # every rank built every sample's planes, so every rank sees the same sentinel
            self._check_finite(p_test is not None)
        return out

    def _graph_eligible(self) -> bool:
        mode = getattr(self, "graph_mode", None)
        if mode is not None:
            return bool(mode)
        return self.layout.entries() * self.plan.width <= self.GRAPH_ENTRY_QUBITS

    def _check_job_inputs(self, train_angles, test_angles) -> None:
        from . import device as dev

        lay, plan = self.layout, self.plan
        dev._require(train_angles, "train angles", torch.float64)
        if lay.n_test:
            dev._require(test_angles, "test angles", torch.float64)
        if train_angles.shape != (lay.n_train, plan.width) or (
                lay.n_test and test_angles.shape != (lay.n_test, plan.width)):
            raise RebindError(f"operand set 0: feature arrays of shapes "
                              f"{tuple(train_angles.shape)} / "
                              f"{tuple(test_angles.shape) if lay.n_test else ()} do not match "
                              f"the job ({lay.n_train}, {lay.n_test}) x width {plan.width}")

    def _ensure_job_buffers(self, devc) -> None:
        """Job-owned device buffers of the single-GPU qk_job_run path: both plane sets, the
        job state (sentinels + tile-claim counter) and the two matrices."""
        if getattr(self, "_jb_dev", None) == devc:
            return
        lay, plan = self.layout, self.plan
        f64 = dict(dtype=torch.float64, device=devc)
        self._g_planes = [torch.empty(max(plan.planes_bytes(n), 16), dtype=torch.uint8,
                                      device=devc) for n in (lay.n_train, lay.n_test)]
        self._bad = torch.empty(3, dtype=torch.int64, device=devc)  # QK_JOB_STATE_WORDS
        self.K_train = torch.empty((lay.n_train, lay.n_train), **f64)
        self.K_cross = torch.empty((lay.n_test, lay.n_train), **f64) if lay.n_test else None
        self._nt = int(_native.lib().qk_job_tile_count(plan.handle, lay.n_train, lay.n_test))
        self._g = None
        self._jb_dev = devc

    def _job_run_call(self, train_ptr: int, test_ptr: int | None) -> None:
        """One qk_job_run on the current stream: state reset, both gate builds in one launch,
        the sweep as a programmatic dependent of the build (three graph nodes when captured)."""
        from . import device as dev

        lay = self.layout
        _native.check(_native.lib().qk_job_run(
            self.plan.handle, train_ptr, lay.n_train, test_ptr if lay.n_test else None,
            lay.n_test, self._g_planes[0].data_ptr(),
            self._g_planes[1].data_ptr() if lay.n_test else None, self._bad.data_ptr(), 0,
            self._nt, self.K_train.data_ptr(),
            self.K_cross.data_ptr() if lay.n_test else None, dev._stream()))

    def _capture_job(self, train_ptr: int, test_ptr: int | None, devc):
        side = torch.cuda.Stream(device=devc)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._job_run_call(train_ptr, test_ptr)  # first use (launch caches), uncaptured
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._job_run_call(train_ptr, test_ptr)
        return g

    def _run_graph(self, train_angles, test_angles) -> None:
        lay, plan = self.layout, self.plan
        self._check_job_inputs(train_angles, test_angles)
        devc = train_angles.device
        self._ensure_job_buffers(devc)
        if self._g is None:
            f64 = dict(dtype=torch.float64, device=devc)
            self._g_in = [torch.zeros((lay.n_train, plan.width), **f64),
                          torch.zeros((max(lay.n_test, 1), plan.width), **f64)]
            self._g = self._capture_job(self._g_in[0].data_ptr(), self._g_in[1].data_ptr(),
                                        devc)
        self._g_in[0].copy_(train_angles)
        if lay.n_test:
            self._g_in[1].copy_(test_angles)
        self._g.replay()

    def _check_finite(self, has_test: bool) -> None:
        """The reference's RebindError for a non-finite angle (network.py:295-296), indexed
        like the single-process API: the first Gram pair (row-major) holding a
        bad train sample, else the first cross pair holding a bad test sample."""
        bad_train, bad_test = self._bad[:2].tolist()  # one device sync for both sentinels
        if bad_train != -1:
            raise RebindError(f"operand set {0 if bad_train == 0 else bad_train - 1}: feature "
                              "angles must be finite")
        if has_test and bad_test != -1:
            raise RebindError(f"operand set {bad_test * self.layout.n_train}: feature angles "
                              "must be finite")

    def graph(self, train_angles: torch.Tensor, test_angles: torch.Tensor | None = None):
        """CUDA-graph capture of one job step (world size 1): returns ``(replay, K_train,
        K_cross)``; ``replay()`` recomputes both matrices into the same tensors from the
        current contents of ``train_angles`` / ``test_angles`` with one graph launch (the
        captured qk_job_run: state reset, gate build, sweep) — for small jobs repeated many
        times (below ~64 qubits the per-call host work of ``run``, ~0.05 ms, is comparable
        with the sweep itself).  Non-finite angles are not checked on replay: the sentinels
        are in ``self._bad[:2]`` (see :meth:`run`)."""
        if self.world != 1:
            raise ValueError("graph capture is single-process (the multi-rank job synchronises "
                             "ranks between launches)")
        self._check_job_inputs(train_angles, test_angles)
        devc = train_angles.device
        self._ensure_job_buffers(devc)
        g = self._capture_job(train_angles.data_ptr(),
                              test_angles.data_ptr() if self.layout.n_test else None, devc)
        self._graph = g  # keeps the graph alive with the job
        return g.replay, self.K_train, self.K_cross

    # ---- host buffers in and out ----------------------------------------------------------
    def host_outputs(self) -> tuple:
        """(K_train, K_cross) host matrices for :meth:`run_host`: shared-memory segments that
        rank 0 creates and every rank maps (collective call).  Rank 0 reads the results from
        their ``array`` views."""
        lay = self.layout
        if self.world == 1:
            return (SharedHostMatrix(lay.n_train, lay.n_train),
                    SharedHostMatrix(lay.n_test, lay.n_train) if lay.n_test else None)
        names = None
        if self.rank == 0:
            mats = [SharedHostMatrix(lay.n_train, lay.n_train),
                    SharedHostMatrix(lay.n_test, lay.n_train) if lay.n_test else None]
            names = [m.name if m is not None else None for m in mats]
        box = [names]
        dist.broadcast_object_list(box, src=0, group=self.group)
        if self.rank != 0:
            mats = [SharedHostMatrix(lay.n_train, lay.n_train, name=box[0][0]),
                    SharedHostMatrix(lay.n_test, lay.n_train, name=box[0][1])
                    if lay.n_test else None]
        dist.barrier(group=self.group)
        return tuple(mats)

    def run_host(self, train_host, test_host, out_train: SharedHostMatrix,
                 out_test: SharedHostMatrix | None = None) -> None:
        """Host angles in (pinned numpy arrays avoid a staging copy), host matrices out: the
        job runs as :meth:`run` (p2p placement: every rank's sweep stores into rank 0's
        matrices), then each rank copies rows [r N / W, (r + 1) N / W) of both matrices from
        rank 0's GPU into the shared host matrices over its own PCIe link."""
        lay = self.layout
        dev_ = torch.device("cuda", torch.cuda.current_device())
        Xtr = np.ascontiguousarray(train_host, dtype=np.float64)
        Xte = np.ascontiguousarray(test_host, dtype=np.float64) if lay.n_test else None
        if self.world > 1 and self.placement == "p2p" and self._shared is None:
            self._setup_shared()  # collective; falls back to the gather placement if needed
        if self.world == 1 or self.placement != "p2p":
            tr = torch.from_numpy(Xtr).to(dev_, non_blocking=True)
            te = torch.from_numpy(Xte).to(dev_, non_blocking=True) if lay.n_test else None
        else:
            tr, te = self._upload_split(Xtr, Xte, dev_)
        K, Kx = self.run(tr, te)
        if self.world > 1 and self.placement != "p2p":
            # gather placement: the matrices exist on rank 0 only
            if self.rank == 0:
                self._drain(K.data_ptr(), out_train, 0, lay.n_train)
                if lay.n_test:
                    self._drain(Kx.data_ptr(), out_test, 0, lay.n_test)
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)
            return
        if self.world == 1:
            srcs = (K.data_ptr(), Kx.data_ptr() if lay.n_test else 0)
        else:
            srcs = (self._shared[0].ptr, self._shared[1].ptr if lay.n_test else 0)
        for src, out, rows in ((srcs[0], out_train, lay.n_train),
                               (srcs[1], out_test, lay.n_test)):
            if rows:
                lo, hi = shard_range(rows, self.rank, self.world)
                self._drain(src, out, lo, hi)
        torch.cuda.current_stream().synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)

    def _upload_split(self, Xtr: np.ndarray, Xte, dev_):
        """Each rank uploads its row slice of the angles into rank 0's shared angle buffer
        (its own PCIe link), then every rank pulls the whole set from rank 0 over NVLink."""
        lay = self.layout
        width = Xtr.shape[1]
        rows = lay.n_train + lay.n_test
        if getattr(self, "_angles", None) is None:
            if self.rank == 0:
                mat = SharedMatrix(rows, width)
                handle = mat.export()
            else:
                mat, handle = None, None
            box = [handle]
            dist.broadcast_object_list(box, src=0, group=self.group)
            if self.rank != 0:
                mat = SharedMatrix(rows, width, handle=box[0])
            self._angles = mat
            self._angles_local = torch.empty((rows, width), dtype=torch.float64, device=dev_)
        mat, local = self._angles, self._angles_local
        lib = _native.lib()
        stream = torch.cuda.current_stream().cuda_stream
        row = width * 8
        for X, base, n in ((Xtr, 0, lay.n_train), (Xte, lay.n_train, lay.n_test)):
            if n:
                lo, hi = shard_range(n, self.rank, self.world)
                if hi > lo:
                    _native.check(lib.qk_copy_h2d(mat.ptr + (base + lo) * row,
                                                  X.ctypes.data + lo * row, (hi - lo) * row,
                                                  stream))
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)
        _native.check(lib.qk_copy_d2d(local.data_ptr(), mat.ptr, rows * row, stream))
        return local[:lay.n_train], (local[lay.n_train:] if lay.n_test else None)

    @staticmethod
    def _drain(src_ptr: int, out: SharedHostMatrix, lo: int, hi: int) -> None:
        if hi <= lo:
            return
        row = out.cols * 8
        _native.check(_native.lib().qk_copy_d2h(out.array.ctypes.data + lo * row,
                                                src_ptr + lo * row, (hi - lo) * row,
                                                torch.cuda.current_stream().cuda_stream))

    def close(self) -> None:
        if self._shared:
            for m in self._shared:
                m.close()
            self._shared = None
        if getattr(self, "_angles", None) is not None:
            self._angles.close()
            self._angles = None
