"""Device time of the config-4 job: two launches (Gram, cross) vs the joint tile list."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200.data import config_data  # noqa: E402

Atr, _, Ate, _ = config_data(4, 10000, 2000, "mnist", bw=1.0)
plan = SweepPlan(784, 2)
tr, te = torch.as_tensor(Atr, device="cuda"), torch.as_tensor(Ate, device="cuda")
pt, ps = dev.gate_build(plan, tr), dev.gate_build(plan, te)
K = torch.empty((10000, 10000), dtype=torch.float64, device="cuda")
Kx = torch.empty((2000, 10000), dtype=torch.float64, device="cuda")


def two():
    dev.gram(pt, out=K)
    dev.cross(ps, pt, out=Kx)


def one():
    dev.job_into(pt, ps, K.data_ptr(), Kx.data_ptr())


for name, fn in [("two", two), ("one", one), ("two", two), ("one", one)]:
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms  {69995000 / ms / 1e6:.4f} G entries/s")
