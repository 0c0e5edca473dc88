"""Single-path drivers for compute-sanitizer racecheck: a device Gram at 784 qubits (the long-
chain ring refills), the same without half tiles, or the head-first host pipeline.
usage: compute-sanitizer --tool racecheck python tools/racecheck_probe.py gram|gram_nosplit|head"""
import sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import FeatureMapConfig, SweepPlan, compute_kernel_matrices
from paper_2405_02630_b200 import device as dev
mode = sys.argv[1]
rng = np.random.default_rng(0)
if mode == "gram":  # device Gram at 784 qubits, 1100 samples (whole tiles + half-tile tail)
    X = torch.as_tensor(rng.uniform(0, 0.05, (1100, 784)), device="cuda")
    K = dev.gram(dev.gate_build(SweepPlan(784, 2), X))
elif mode == "gram_nosplit":
    X = torch.as_tensor(rng.uniform(0, 0.05, (1100, 784)), device="cuda")
    K = dev.gram(dev.gate_build(SweepPlan(784, 2), X))
elif mode == "head":
    Xh = torch.empty((1100, 784), dtype=torch.float64, pin_memory=True).numpy()
    Xh[:] = rng.uniform(0, 0.05, Xh.shape)
    Th = torch.empty((70, 784), dtype=torch.float64, pin_memory=True).numpy()
    Th[:] = rng.uniform(0, 0.05, Th.shape)
    compute_kernel_matrices(Xh, Th, FeatureMapConfig(784))
torch.cuda.synchronize()
print("ok", mode)
