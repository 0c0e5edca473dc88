"""Device-resident vs end-to-end (pinned host arrays in and out) rate for each BASELINE config
on one GPU: KernelJob.run on resident angles (CUDA events) against compute_kernel_matrices
host→host (wall clock), best of `reps`; and the default call (pageable numpy angles in,
library-allocated results out: `default_ms`).  One JSON line per config."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices, plan_for  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402

CONFIGS = [(1, 8, 100, 50), (2, 50, 1000, 500), (3, 784, 2000, 1000), (4, 784, 10000, 2000)]


def pin(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
    t[...] = a
    return t


reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(0)
for cid, n, ntr, nte in CONFIGS:
    X, T = pin(rng.uniform(0, np.pi, (ntr, n))), pin(rng.uniform(0, np.pi, (nte, n)))
    K, Kx = pin(np.empty((ntr, ntr))), pin(np.empty((nte, ntr)))
    cfg = FeatureMapConfig(n)
    entries = ntr * (ntr - 1) // 2 + nte * ntr
    job = KernelJob(plan_for(cfg), ntr, nte)
    tr, te = torch.as_tensor(X, device="cuda"), torch.as_tensor(T, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    Xp, Tp = np.array(X), np.array(T)  # pageable copies for the default call
    dev_ms, e2e_ms, def_ms = [], [], []
    for _ in range(reps + 2):
        e0.record()
        job.run(tr, te)
        e1.record()
        torch.cuda.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
        t = time.perf_counter()
        compute_kernel_matrices(X, T, cfg, out_train=K, out_test=Kx)
        e2e_ms.append((time.perf_counter() - t) * 1e3)
        t = time.perf_counter()
        compute_kernel_matrices(Xp, Tp, cfg)
        def_ms.append((time.perf_counter() - t) * 1e3)
    d, e, f = min(dev_ms[2:]), min(e2e_ms[2:]), min(def_ms[2:])
    print(json.dumps({"config": cid, "qubits": n, "n_train": ntr, "n_test": nte,
                      "entries": entries, "device_ms": d, "e2e_ms": e, "default_ms": f,
                      "device_entries_per_s": entries / d * 1e3,
                      "e2e_entries_per_s": entries / e * 1e3, "e2e_over_device": d / e}),
          flush=True)
