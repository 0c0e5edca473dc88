"""Projected strong scaling of config 4 on N = 1, 2, 4, 8 GPUs from ONE GPU: each rank's share
of the joint tile list (distributed.layout_for, the ranges the N-rank job uses) is swept alone
on this GPU, exactly as that rank would (gate builds of all samples + one dynamic-schedule
launch over its range), timed with CUDA events; the projected job time is the slowest rank.
Not included: the NVLink stores into rank 0's matrices (spread over the sweep, ~120 GB/s of
ingress at N = 8) and the closing barrier.  One JSON line per N."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200.distributed import layout_for  # noqa: E402

N_TRAIN, N_TEST, N_QUBITS = 10000, 2000, 784
rng = np.random.default_rng(0)
tr = torch.as_tensor(rng.uniform(0, np.pi, (N_TRAIN, N_QUBITS)), device="cuda")
te = torch.as_tensor(rng.uniform(0, np.pi, (N_TEST, N_QUBITS)), device="cuda")
plan = SweepPlan(N_QUBITS, 2)
K = torch.empty((N_TRAIN, N_TRAIN), dtype=torch.float64, device="cuda")
Kx = torch.empty((N_TEST, N_TRAIN), dtype=torch.float64, device="cuda")


def rank_step(lo, hi):
    p_tr = dev.gate_build(plan, tr)
    p_te = dev.gate_build(plan, te)
    dev.job_into(p_tr, p_te, K.data_ptr(), Kx.data_ptr(), lo, hi)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


base = None
for world in (1, 2, 4, 8):
    lay = layout_for(plan, N_TRAIN, N_TEST, world)
    times = [timed(lambda r=r: rank_step(*lay.union_range(r))) for r in range(world)]
    ms = max(times)
    entries = lay.entries()
    base = base or ms
    print(json.dumps({"gpus": world, "rank_ms": [round(t, 3) for t in times], "job_ms": ms,
                      "entries_per_s": entries / ms * 1e3, "speedup": base / ms,
                      "efficiency": base / ms / world}), flush=True)
