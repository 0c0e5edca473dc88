"""Minimal driver for ncu: one config-4 train Gram sweep (+ optional cross) at 784 qubits."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402

n, N = 784, int(sys.argv[1]) if len(sys.argv) > 1 else 10000
rng = np.random.default_rng(0)
X = torch.as_tensor(rng.uniform(0, np.pi, (N, n)), device="cuda")
plan = SweepPlan(n, 2)
planes = dev.gate_build(plan, X)
K = dev.gram(planes)
if len(sys.argv) > 2:
    K2 = dev.cross(planes, planes)
torch.cuda.synchronize()
print("ok", float(K[0, 1]))
