"""Small-job efficiency (BASELINE configs[1] = C2 and the configs[4] qubit sweep = C5):
device-resident KernelJob.run vs its CUDA-graph replay, ms per job (median of runs of 50),
FP64-pipe fraction of the whole job (executed DP instructions / (SMs x 64 lanes x clock x
time)), and the sweep kernel's own share (CUDA events around the launch).

usage: python tools/small_jobs.py [--only c2] [--reps 50]   (one JSON line per point)"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as qdev  # noqa: E402
from paper_2405_02630_b200.data import config_data  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402

POINTS = {
    "c1": dict(cid=1, n=8, n_train=100, n_test=50, features=8),
    "c2": dict(cid=2, n=50, n_train=1000, n_test=500, features=50),
    "c5_16": dict(cid=5, n=16, n_train=1000, n_test=1000),
    "c5_32": dict(cid=5, n=32, n_train=1000, n_test=1000),
    "c5_64": dict(cid=5, n=64, n_train=1000, n_test=1000),
    "c5_128": dict(cid=5, n=128, n_train=1000, n_test=1000),
    "c5_256": dict(cid=5, n=256, n_train=1000, n_test=1000),
}


def median_ms(fn, reps):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps)
    return float(np.median(out))


def point(name, cid, n, n_train, n_test, features=None, reps=50):
    if features is not None:
        Atr, _, Ate, _ = config_data(cid, n_train, n_test, "mnist", features=features,
                                     binary=(2, 6))
    else:
        rng = np.random.default_rng(n)
        Atr, Ate = rng.uniform(0, np.pi, (n_train, n)), rng.uniform(0, np.pi, (n_test, n))
    tr = torch.as_tensor(Atr, device="cuda")
    te = torch.as_tensor(Ate, device="cuda")
    plan = SweepPlan(n, 2)
    job = KernelJob(plan, n_train, n_test)
    entries = job.layout.entries()
    plain = median_ms(lambda: job.run(tr, te), reps)
    # sweep kernel alone (CUDA events around job_into)
    p_tr, p_te = qdev.gate_build(plan, tr), qdev.gate_build(plan, te)
    K, Kx = job.run(tr, te)
    sweep = median_ms(lambda: qdev.job_into(p_tr, p_te, K.data_ptr(), Kx.data_ptr()), reps)
    replay, K2, Kx2 = job.graph(tr, te)
    graph = median_ms(replay, reps)
    same = bool(torch.equal(K, K2) and torch.equal(Kx, Kx2))
    props = torch.cuda.get_device_properties(0)
    cap = props.multi_processor_count * 64 * 1.965e9
    dp = entries * plan.info["dp_instr_per_entry"]
    return {"point": name, "qubits": n, "n_train": n_train, "n_test": n_test,
            "entries": entries, "ms_job": plain, "ms_graph": graph, "ms_sweep_kernel": sweep,
            "fp64_pipe_job": dp / (plain * 1e-3) / cap,
            "fp64_pipe_graph": dp / (graph * 1e-3) / cap,
            "fp64_pipe_sweep": dp / (sweep * 1e-3) / cap,
            "entries_per_s_graph": entries / (graph * 1e-3), "graph_same_bits": same}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    names = [a.only] if a.only else list(POINTS)
    for nm in names:
        print(json.dumps(point(nm, reps=a.reps, **POINTS[nm])), flush=True)
