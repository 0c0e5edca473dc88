"""Pair-list kernel (contract_batch / compute_kernel_shard path) throughput at 784 qubits:
1M (p, q) pairs over 10,000 samples, in enumeration (row-major upper-triangle) order and in
random order; device-resident planes, CUDA events.  One JSON line per case."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402

rng = np.random.default_rng(0)
N, n, P = 10000, 784, 1 << 20
X = torch.as_tensor(rng.uniform(0, np.pi, (N, n)), device="cuda")
plan = SweepPlan(n, 2)
planes = dev.gate_build(plan, X)
i, j = np.triu_indices(N, 1)
cases = {"enumeration": np.stack([i[:P], j[:P]], 1),
         "random": np.stack([rng.integers(0, N, P), rng.integers(0, N, P)], 1)}
for name, pr in cases.items():
    pairs = torch.as_tensor(pr, device="cuda")
    dev.pair_amplitudes(planes, planes, pairs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        dev.pair_amplitudes(planes, planes, pairs)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 3e3
    print(json.dumps({"case": name, "pairs": P, "qubits": n, "s": s, "pairs_per_s": P / s}))
