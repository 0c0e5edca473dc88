"""Minimal driver for ncu: one train Gram at depth L (default L = 5, 784 qubits, 512 samples),
device-resident angles.  usage: python tools/profile_deep.py [L width samples]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402

L, n, N = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (5, 784, 512)))
X = torch.as_tensor(np.random.default_rng(L).uniform(0, np.pi, (N, n)), device="cuda")
plan = SweepPlan(n, L)
K = dev.gram(dev.gate_build(plan, X))
torch.cuda.synchronize()
print("ok", float(K[0, 1]))
