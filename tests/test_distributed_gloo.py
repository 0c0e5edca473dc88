"""Multi-process (world_size 2, gloo on CPU) check of the tile sharding + gather contract used
by the multi-GPU path: every tile of the job is owned by exactly one rank, the padded packed
buffers gather to rank 0, and placing them by (segment, tile) rebuilds the dense matrices.
The sweeps/unpacks themselves are CUDA kernels (covered by the gpu tests); here each rank
fills its packed tiles with a known function of the global (i, j) coordinates."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_02630_b200 import SweepPlan
from paper_2405_02630_b200.distributed import gather_packed, layout_for

N_TRAIN, N_TEST, WIDTH = 300, 70, 8


def f(i, j):
    return 1.0 + i * 1e-3 + j * 1e-7


def upper_tile(g, nb):
    r, off = 0, 0
    while off + (nb - r) <= g:
        off += nb - r
        r += 1
    return r, r + (g - off)


def fill(buf, lay, rank, T):
    for seg in lay.segments(rank):
        for t in range(seg.tile_begin, seg.tile_end):
            if seg.kind == "gram":
                bi, bj = upper_tile(t, -(-lay.n_train // T))
            else:
                nbc = -(-lay.n_train // T)
                bi, bj = divmod(t, nbc)
            il, jl = np.meshgrid(np.arange(T), np.arange(T), indexing="ij")
            base = (seg.offset + t - seg.tile_begin) * T * T
            buf[base:base + T * T] = torch.from_numpy(f(bi * T + il, bj * T + jl).ravel())


def place(bufs, lay, T):
    K = np.zeros((lay.n_train, lay.n_train))
    Kx = np.zeros((lay.n_test, lay.n_train))
    nb = -(-lay.n_train // T)
    for r, buf in enumerate(bufs):
        b = buf.numpy()
        for seg in lay.segments(r):
            for t in range(seg.tile_begin, seg.tile_end):
                tile = b[(seg.offset + t - seg.tile_begin) * T * T:][:T * T].reshape(T, T)
                bi, bj = upper_tile(t, nb) if seg.kind == "gram" else divmod(t, nb)
                for il in range(T):
                    i = bi * T + il
                    for jl in range(T):
                        j = bj * T + jl
                        if seg.kind == "gram":
                            if i < j < lay.n_train:
                                K[i, j] = K[j, i] = tile[il, jl]
                            elif i == j < lay.n_train:
                                K[i, i] = 1.0
                        elif i < lay.n_test and j < lay.n_train:
                            Kx[i, j] = tile[il, jl]
    return K, Kx


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = SweepPlan(WIDTH, 2)
    T = plan.tile_edge
    lay = layout_for(plan, N_TRAIN, N_TEST, world)
    buf = torch.full((lay.range_len * lay.tile_elems,), np.nan, dtype=torch.float64)
    fill(buf, lay, rank, T)
    bufs = gather_packed(buf, lay)
    if rank == 0:
        K, Kx = place(bufs, lay, T)
        i, j = np.meshgrid(np.arange(N_TRAIN), np.arange(N_TRAIN), indexing="ij")
        Kref = np.where(i == j, 1.0, f(np.minimum(i, j), np.maximum(i, j)))
        ti, tj = np.meshgrid(np.arange(N_TEST), np.arange(N_TRAIN), indexing="ij")
        q.put((bool(np.array_equal(K, Kref)), bool(np.array_equal(Kx, f(ti, tj)))))
    dist.destroy_process_group()


def placement_worker(rank, world, port, reach, q):
    """KernelJob._setup_shared's placement protocol over gloo with the device calls faked:
    rank 0 exports, the others check reachability of rank 0's device and import."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_02630_b200 import distributed as D

    events = []

    class FakeMatrix:
        def __init__(self, rows, cols, handle=None):
            events.append("import" if handle is not None else "alloc")
            self.rows, self.cols, self.ptr = rows, cols, 1

        def export(self):
            return b"h" * 64

        def tensor(self):
            return torch.zeros((self.rows, self.cols), dtype=torch.float64)

        def close(self):
            events.append("close")

    D.SharedMatrix = FakeMatrix
    D.device_bus_id = lambda: "0000:1b:00.0"
    D.can_reach = lambda bus: (bus == "0000:1b:00.0") and reach[rank]
    job = D.KernelJob(SweepPlan(WIDTH, 2), N_TRAIN, N_TEST)
    ok = job._setup_shared()
    q.put((rank, ok, job.placement, events))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("reach", [(True, True, True), (True, True, False)])
def test_p2p_placement_agreement_world3(reach):
    """Every rank ends on the same placement: p2p only if every rank can reach rank 0's
    device; otherwise all fall back to the gather and release what they mapped (a rank that
    cannot reach rank 0 never attempts the import)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=placement_worker, args=(r, 3, port, reach, q))
             for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    want = all(reach)
    for rank, ok, placement, events in res:
        assert ok == want and placement == ("p2p" if want else "gather")
        if rank == 0:
            assert events[:2] == ["alloc", "alloc"]
        elif reach[rank]:
            assert events[:2] == ["import", "import"]
        else:
            assert "import" not in events
        if not want:
            assert events.count("close") == events.count("alloc") + events.count("import")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_layout_partitions_every_tile_exactly_once():
    plan = SweepPlan(WIDTH, 2)
    for world in (1, 2, 3, 8):
        lay = layout_for(plan, N_TRAIN, N_TEST, world)
        seen = {"gram": [], "cross": []}
        for r in range(world):
            for seg in lay.segments(r):
                seen[seg.kind].extend(range(seg.tile_begin, seg.tile_end))
                assert seg.offset + seg.tile_end - seg.tile_begin <= lay.range_len
        assert seen["gram"] == list(range(lay.gram_tiles))
        assert seen["cross"] == list(range(lay.cross_tiles))
    assert lay.entries() == N_TRAIN * (N_TRAIN - 1) // 2 + N_TEST * N_TRAIN


@pytest.mark.timeout(300)
def test_gather_rebuilds_dense_matrices_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok == (True, True)
    assert all(p.exitcode == 0 for p in procs)


def test_cost_balanced_ranges_cover_the_list_once():
    """layout_for splits the joint tile list into contiguous ranges of equal estimated cost:
    they tile the list exactly, and the ranks holding the padding tile rows (cost 1/4) get
    more tiles."""
    from paper_2405_02630_b200.distributed import tile_costs
    plan = SweepPlan(784, 2)
    for world in (1, 2, 3, 4, 8):
        lay = layout_for(plan, 10000, 2000, world)
        rngs = [lay.union_range(r) for r in range(world)]
        assert rngs[0][0] == 0 and rngs[-1][1] == lay.total_tiles
        assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
        cost = tile_costs(10000, 2000, 64)
        per = [cost[lo:hi].sum() for lo, hi in rngs]
        assert max(per) - min(per) <= 2.0  # one tile of granularity per boundary
    lay = layout_for(plan, 10000, 2000, 8)
    sizes = [hi - lo for lo, hi in (lay.union_range(r) for r in range(8))]
    assert sizes[0] > sizes[1]  # rank 0 holds the Gram's padding tile row
