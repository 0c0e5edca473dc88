"""Small end-to-end run of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): gate build (vector and scalar loads, one and two plane sets), joint sweep
(L = 1..8), dense + packed + unpack, pair kernel, host pipelines (pinned and pageable, the
head-first two-stream upload), and the CUDA-graph replay of qk_job_run (KernelJob)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import (FeatureMapConfig, SweepPlan,  # noqa: E402
                                   compute_kernel_matrices)
from paper_2405_02630_b200 import device as dev  # noqa: E402

rng = np.random.default_rng(0)
for L, n in ((2, 40), (1, 20), (3, 6), (4, 5), (5, 4), (6, 3), (7, 3), (8, 2)):
    Ntr, Nte = (150, 70) if L <= 4 else (40, 9) if L <= 6 else (12, 3)
    Xtr = rng.uniform(0, 1, (Ntr, n))
    Xte = rng.uniform(0, 1, (Nte, n))
    cfg = FeatureMapConfig(n, layers=L)
    K, Kx = compute_kernel_matrices(Xtr, Xte, cfg)
    plan = SweepPlan(n, L)
    pt = dev.gate_build(plan, torch.as_tensor(Xtr, device="cuda"))
    ps = dev.gate_build(plan, torch.as_tensor(Xte, device="cuda"))
    nt = plan.gram_tile_count(Ntr)
    packed = dev.gram(pt, packed=True)
    Kd = torch.zeros((Ntr, Ntr), dtype=torch.float64, device="cuda")
    dev.unpack_gram(plan, packed, Ntr, 0, nt, Kd)
    Kxd = dev.cross(ps, pt)
    pairs = torch.as_tensor(np.array([[0, 1], [5, Ntr - 1], [Ntr - 1, 0]]), device="cuda")
    amp = dev.pair_amplitudes(pt, pt, pairs)
    kv = dev.pair_kernel_values(pt, pt, pairs)
    torch.cuda.synchronize()
    assert torch.equal(kv, amp * amp)
    assert np.array_equal(Kd.cpu().numpy(), K.entries)
    assert np.array_equal(Kxd.cpu().numpy(), Kx.entries)
    print("L", L, "ok", float(amp[0]))
pinned = torch.empty((150, 150), dtype=torch.float64, pin_memory=True).numpy()
compute_kernel_matrices(rng.uniform(0, 1, (150, 40)), rng.uniform(0, 1, (3, 40)),
                        FeatureMapConfig(40), out_train=pinned)
# head-first pipeline (pinned inputs large enough for a head: 1100 samples at 784 qubits)
Xh = torch.empty((1100, 784), dtype=torch.float64, pin_memory=True).numpy()
Xh[:] = rng.uniform(0, 0.05, Xh.shape)
Th = torch.empty((70, 784), dtype=torch.float64, pin_memory=True).numpy()
Th[:] = rng.uniform(0, 0.05, Th.shape)
Kh, Kxh = compute_kernel_matrices(Xh, Th, FeatureMapConfig(784))
Kh2, Kxh2 = compute_kernel_matrices(np.array(Xh), np.array(Th), FeatureMapConfig(784))
assert np.array_equal(Kh.entries, Kh2.entries) and np.array_equal(Kxh.entries, Kxh2.entries)
# the small-job graph path (vector gate build at 64 qubits, scalar at 50)
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402
for n in (64, 50):
    tr = torch.as_tensor(rng.uniform(0, 1, (200, n)), device="cuda")
    te = torch.as_tensor(rng.uniform(0, 1, (30, n)), device="cuda")
    Kg, Kxg = KernelJob(SweepPlan(n, 2), 200, 30).run(tr, te)
    Ke, Kxe = KernelJob(SweepPlan(n, 2), 200, 30, graph_mode=False).run(tr, te)
    assert torch.equal(Kg, Ke) and torch.equal(Kxg, Kxe)
    # explicit capture (KernelJob.graph): the captured qk_job_run on the caller's tensors
    replay, Kr, Kxr = KernelJob(SweepPlan(n, 2), 200, 30).graph(tr, te)
    replay()
    torch.cuda.synchronize()
    assert torch.equal(Kr, Ke) and torch.equal(Kxr, Kxe)
print("sanitize smoke ok")
