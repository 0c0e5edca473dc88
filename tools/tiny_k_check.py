"""Check the bench workload's pairs whose K is tiny but normal (1e-296 .. 1e-4 at bw = 1)
through every engine path against the oracle: KernelJob.run (device-resident, the bench's
`value` path), compute_kernel_matrices (host pipeline) and the pair kernel (contract_batch).

usage: python tools/tiny_k_check.py [n_pairs]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices, plan_for  # noqa: E402
from paper_2405_02630_b200 import device as qdev  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
Atr, Ate = bench.workload_data()
A = np.concatenate([Atr, Ate])
pairs = bench.sample_pairs(np.random.default_rng(7), P)
amp = np.real(oracle.amplitudes(A, A, pairs, 2, 16))
Kref = amp * amp
sel = Kref > 0
print(f"{sel.sum()} of {P} pairs with K > 0 (min {Kref[sel].min():.3e})", flush=True)

cfg = FeatureMapConfig(784, layers=2)
plan = plan_for(cfg)
job = KernelJob(plan, bench.N_TRAIN, bench.N_TEST)
K, Kx = (k.cpu().numpy() for k in job.run(torch.as_tensor(Atr, device="cuda"),
                                           torch.as_tensor(Ate, device="cuda")))


def pick(K, Kx):
    i, j = pairs[:, 0], pairs[:, 1]
    return np.where(i < bench.N_TRAIN, K[np.minimum(i, bench.N_TRAIN - 1), j],
                    Kx[np.maximum(i - bench.N_TRAIN, 0), j])


def report(name, ours):
    d = np.abs(ours - Kref)
    rel = np.abs(ours[sel] - Kref[sel]) / Kref[sel]
    worst = int(np.argmax(np.where(sel, np.abs(ours - Kref) / np.where(sel, Kref, 1), 0)))
    rec = {"path": name, "max_abs_dK": float(d.max()), "max_rel_dK_nonzero": float(rel.max()),
           "worst_pair": pairs[worst].tolist(), "worst_ref": float(Kref[worst]),
           "worst_ours": float(ours[worst])}
    print(json.dumps(rec), flush=True)


report("KernelJob.run", pick(K, Kx))
Kh, Kxh = compute_kernel_matrices(Atr, Ate, cfg)
report("compute_kernel_matrices", pick(Kh.entries, Kxh.entries))
t = torch.as_tensor(A, device="cuda")
pl = qdev.gate_build(plan, t)
amps = qdev.pair_amplitudes(pl, pl, torch.as_tensor(pairs, device="cuda")).cpu().numpy()
report("pair kernel", amps ** 2)

# SURVEY §8(d) amplitude gate |d amp| <= 1e-9 |amp_ref| + 1e-300, binned by K_ref
a_ours = np.abs(amps)
a_ref = np.abs(amp)
ratio = np.abs(a_ours - a_ref) / (1e-9 * a_ref + 1e-300)
for lo, hi in ((1e-12, 2.0), (1e-50, 1e-12), (1e-100, 1e-50), (1e-200, 1e-100),
               (1e-300, 1e-200), (0.0, 1e-300)):
    m = (Kref >= lo) & (Kref < hi) if lo > 0 else (Kref < hi)
    if m.any():
        rel = np.abs(a_ours[m] - a_ref[m]) / np.maximum(a_ref[m], 1e-320)
        print(json.dumps({"K_range": [lo, hi], "pairs": int(m.sum()),
                          "amp_gate_max_ratio": float(ratio[m].max()),
                          "amp_gate_fail": int((ratio[m] > 1).sum()),
                          "max_rel_d_amp": float(rel.max()),
                          "median_rel_d_amp": float(np.median(rel))}), flush=True)
