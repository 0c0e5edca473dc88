"""Multi-GPU sharding of the kernel-matrix job: one process per GPU, one gather.

The reference parallelises over pairs only — a fork pool in code (engine.py:159-166),
shard-run-then-merge in SPEC, MPI + NCCL across A100s in the paper
(PAPER.md:359-362).  Here the unit is the sweep tile: the job's linearised tile list (train
Gram upper-triangle tiles, then test x train cross tiles) is split into contiguous equal
ranges (SPEC's contiguous ceil(P/W) rule at tile granularity; every tile costs the same, so
equal counts are balanced).  Each rank builds the gate planes of every sample (cheap),
sweeps its range into a packed buffer padded to the common range length, and ONE
``gather`` over NCCL (NVLink / NVSwitch) brings the packed tiles to rank 0, which scatters
them into the dense matrices with the unpack kernel.  World size 1 writes the dense
matrices directly.

The partition / gather / placement logic is device-agnostic (tested with gloo on CPU);
the sweeps and unpacks are the CUDA kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import ceil

import torch
import torch.distributed as dist

from .kernel_pipeline import shard_range
from .planner import SweepPlan


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

    @property
    def total_tiles(self) -> int:
        return self.gram_tiles + self.cross_tiles

    @property
    def range_len(self) -> int:
        return ceil(self.total_tiles / self.world) if self.total_tiles else 0

    def union_range(self, rank: int) -> tuple[int, int]:
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


def layout_for(plan: SweepPlan, n_train: int, n_test: int, world: int) -> JobLayout:
    return JobLayout(n_train, n_test, plan.gram_tile_count(n_train),
                     plan.cross_tile_count(n_test, n_train) if n_test else 0, world,
                     plan.tile_edge * plan.tile_edge)


def gather_packed(local: torch.Tensor, layout: JobLayout, group=None) -> list | None:
    """Gather every rank's padded packed buffer to rank 0 (one collective)."""
    rank = dist.get_rank(group)
    if layout.world == 1:
        return [local]
    bufs = [torch.empty_like(local) for _ in range(layout.world)] if rank == 0 else None
    dist.gather(local, bufs, dst=0, group=group)
    return bufs


class KernelJob:
    """Train Gram (+ optional test x train cross block) over a process group."""

    def __init__(self, plan: SweepPlan, n_train: int, n_test: int = 0, group=None):
        self.plan = plan
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.layout = layout_for(plan, n_train, n_test, self.world)
        self.packed = None
        self.K_train = None
        self.K_cross = None

    def run(self, train_angles: torch.Tensor, test_angles: torch.Tensor | None = None):
        """Returns (K_train, K_cross) on rank 0 (device tensors), (None, None) elsewhere."""
        from . import device as dev

        lay = self.layout
        p_train = dev.gate_build(self.plan, train_angles)
        p_test = dev.gate_build(self.plan, test_angles) if lay.n_test else None
        devc = train_angles.device
        if self.world == 1:
            if self.K_train is None:
                self.K_train = torch.empty((lay.n_train, lay.n_train), dtype=torch.float64,
                                           device=devc)
                if lay.n_test:
                    self.K_cross = torch.empty((lay.n_test, lay.n_train), dtype=torch.float64,
                                               device=devc)
            dev.gram(p_train, out=self.K_train)
            if lay.n_test:
                dev.cross(p_test, p_train, out=self.K_cross)
            return self.K_train, self.K_cross
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
