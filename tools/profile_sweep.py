"""Minimal driver for ncu: the config-4 job (784 qubits, 10000 train Gram + 2000 x 10000
cross) as ONE joint sweep launch, exactly as bench.py runs it."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200.data import config_data  # noqa: E402

Atr, _, Ate, _ = config_data(4, 10000, 2000, "mnist", bw=1.0)
plan = SweepPlan(784, 2)
pt = dev.gate_build(plan, torch.as_tensor(Atr, device="cuda"))
ps = dev.gate_build(plan, torch.as_tensor(Ate, device="cuda"))
K = torch.empty((10000, 10000), dtype=torch.float64, device="cuda")
Kx = torch.empty((2000, 10000), dtype=torch.float64, device="cuda")
dev.job_into(pt, ps, K.data_ptr(), Kx.data_ptr())
torch.cuda.synchronize()
print("ok", float(K[0, 1]), float(Kx[0, 0]))
