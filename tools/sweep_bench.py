"""BASELINE configs[4] on one GPU: entries/s over a qubit-count sweep (16 -> 784) at a fixed
1000 x 1000 train Gram + 1000 x 1000 cross, and over a dataset-size sweep (1k -> 20k train,
2k test) at 784 qubits.  Device-resident inputs, CUDA events, one joint sweep launch per
step; prints one JSON line per point."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402


def point(n, n_train, n_test, steps=5):
    rng = np.random.default_rng(n * 7 + n_train)
    tr = torch.as_tensor(rng.uniform(0, np.pi, (n_train, n)), device="cuda")
    te = torch.as_tensor(rng.uniform(0, np.pi, (n_test, n)), device="cuda")
    plan = SweepPlan(n, 2)
    job = KernelJob(plan, n_train, n_test)
    job.run(tr, te)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        job.run(tr, te)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3 / steps
    entries = job.layout.entries()
    dp = plan.info["dp_instr_per_entry"]
    props = torch.cuda.get_device_properties(0)
    pipe = entries * dp / s / (props.multi_processor_count * 64 * 1.965e9)
    return {"qubits": n, "n_train": n_train, "n_test": n_test, "entries": entries,
            "ms": 1e3 * s, "entries_per_s": entries / s,
            "qubit_entries_per_s": entries * n / s, "fp64_pipe_frac": pipe}


if __name__ == "__main__":
    for n in (16, 32, 50, 64, 128, 256, 512, 784):
        print(json.dumps(dict(point(n, 1000, 1000), sweep="qubits")), flush=True)
    for N in (1000, 2000, 5000, 10000, 20000):
        print(json.dumps(dict(point(784, N, 2000, steps=3 if N >= 10000 else 5),
                              sweep="dataset")), flush=True)
