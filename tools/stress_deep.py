"""Randomised check of the L = 5..8 sweeps: for random widths and sample counts, every Gram
and cross entry of the tile kernel equals the pair-list kernel's value bit for bit (both run
deep_sweep), and sampled entries match the CPU oracle within the parity gate.
usage: python tools/stress_deep.py [seconds]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402  (the checker)
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(11)
t0, cases, entries, worst = time.time(), 0, 0, 0.0
while time.time() - t0 < budget:
    L = int(rng.choice([5, 5, 6, 7, 8]))
    n = int(rng.integers(1, {5: 60, 6: 24, 7: 10, 8: 5}[L]))
    N = int(rng.integers(2, {5: 200, 6: 90, 7: 40, 8: 12}[L]))
    M = int(rng.integers(1, max(2, N // 2)))
    X = rng.uniform(0, 0.4, (N, n)) + rng.uniform(0, np.pi, n)
    T = rng.uniform(0, 0.4, (M, n)) + rng.uniform(0, np.pi, n)
    plan = SweepPlan(n, L)
    px = dev.gate_build(plan, torch.as_tensor(X, device="cuda"))
    pt = dev.gate_build(plan, torch.as_tensor(T, device="cuda"))
    K = dev.gram(px).cpu().numpy()
    Kx = dev.cross(pt, px).cpu().numpy()
    i, j = np.triu_indices(N, 1)
    g = dev.pair_kernel_values(px, px, torch.as_tensor(np.stack([i, j], 1), device="cuda"))
    assert np.array_equal(g.cpu().numpy(), K[i, j]), ("gram", L, n, N)
    r, c = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    x = dev.pair_kernel_values(pt, px, torch.as_tensor(np.stack([r.ravel(), c.ravel()], 1),
                                                       device="cuda"))
    assert np.array_equal(x.cpu().numpy(), Kx.ravel()), ("cross", L, n, N, M)
    assert np.all(np.diag(K) == 1.0) and np.array_equal(K, K.T)
    k = min(len(i), 4)
    sel = rng.choice(len(i), k, replace=False) if len(i) else []
    if len(sel):
        ref = np.abs(oracle.amplitudes(X, X, np.stack([i[sel], j[sel]], 1), L)) ** 2
        worst = max(worst, float(np.abs(K[i[sel], j[sel]] - ref).max()))
        assert worst <= 1e-12, (L, n, N, worst)
    cases += 1
    entries += len(i) + M * N
print(f"stress_deep ok: {cases} cases, {entries} entries (tile == pair bit for bit), "
      f"max |dK| vs oracle {worst:.2e}, {time.time() - t0:.0f} s")
