"""The multi-GPU job path with two real processes.  Only one GPU is available to the test
run, so both ranks share cuda:0 (CUDA IPC between processes works within a device) and the
process group is gloo; on an 8-GPU box the same code runs one rank per GPU over NCCL with
the IPC stores going over NVLink.  Both placements must reproduce the single-process
matrices bit for bit and, for L <= 3, the CPU oracle's to 1e-12."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

N_TRAIN, N_TEST, WIDTH = 333, 71, 40


def _data():
    rng = np.random.default_rng(77)
    centre = rng.uniform(0, np.pi, WIDTH)
    return (centre + rng.normal(0, 0.1, (N_TRAIN, WIDTH)),
            centre + rng.normal(0, 0.1, (N_TEST, WIDTH)))


def worker(rank, world, port, placement, layers, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2405_02630_b200 import (FeatureMapConfig, SweepPlan, compute_cross_kernel,
                                           compute_kernel_matrix)
        from paper_2405_02630_b200.distributed import KernelJob

        Xtr, Xte = _data()
        plan = SweepPlan(WIDTH, layers)
        job = KernelJob(plan, N_TRAIN, N_TEST, placement=placement)
        for _ in range(2):  # the second run reuses the shared matrices / buffers
            K, Kx = job.run(torch.as_tensor(Xtr, device="cuda"),
                            torch.as_tensor(Xte, device="cuda"))
        # host buffers in and out: every rank drains its row slice into shared host memory
        out_K, out_Kx = job.host_outputs()
        out_K.array[:] = -1.0
        out_Kx.array[:] = -1.0
        dist.barrier()
        job.run_host(Xtr, Xte, out_K, out_Kx)
        if rank == 0:
            cfg = FeatureMapConfig(WIDTH, layers=layers)
            Kr = compute_kernel_matrix(Xtr, cfg).entries
            Kxr = compute_cross_kernel(Xte, Xtr, cfg).entries
            ok = (np.array_equal(K.cpu().numpy(), Kr) and np.array_equal(out_K.array, Kr),
                  np.array_equal(Kx.cpu().numpy(), Kxr) and np.array_equal(out_Kx.array, Kxr))
            if layers <= 3:  # and the multi-rank result against the CPU oracle itself
                from oracle import oracle
                err = max(float(np.abs(out_K.array - oracle.kernel_matrix(Xtr, layers)).max()),
                          float(np.abs(out_Kx.array - oracle.cross_kernel(Xte, Xtr, layers)).max()))
                ok = (ok[0] and err <= 1e-12, ok[1] and err <= 1e-12)
            q.put(ok)
        dist.barrier()
        out_K.close()
        out_Kx.close()
        dist.barrier()
        job.close()
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        q.put(repr(exc))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("placement,world,layers", [("p2p", 2, 2), ("gather", 2, 2),
                                                    ("p2p", 3, 2), ("p2p", 3, 5),
                                                    ("gather", 3, 3)])
def test_multi_rank_job_matches_single_process(placement, world, layers):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, placement, layers, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=500)
    for p in procs:
        p.join(timeout=120)
    assert res == (True, True), res
    assert all(p.exitcode == 0 for p in procs)
