"""Time the UNMODIFIED reference's CPU path (baseline/_ref: /root/reference/pkg installed with
pip --target) on a sample of the bench workload — the reference-side baseline of
BASELINE.md §3: contract_batch(template, pairs, plan, workers=os.cpu_count())
(pkg/src/tnkernel/engine.py:132-166, fork pool :159-166) over the simplified kernel network
(network.py:125-302) with one plan_contraction (paths.py:529-543) reused for every pair.

Run by bench.py in a subprocess with no CUDA device visible:
    python tools/ref_baseline.py angles.npy pairs.npy out.json [repeats]
angles.npy: [N, width] fp64; pairs.npy: [P, 2] int64 row indices into it (x_i, x_j).
Writes {"entries_per_s", "plan_s", "runs_s", "workers", "amplitudes_re", ...}."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

import numpy as np  # noqa: E402
from tnkernel.circuit import FeatureMapConfig, compose_kernel_circuit  # noqa: E402
from tnkernel.engine import contract_batch  # noqa: E402
from tnkernel.network import circuit_to_network, simplify  # noqa: E402
from tnkernel.paths import plan_contraction  # noqa: E402


def main():
    angles = np.load(sys.argv[1])
    pairs = np.load(sys.argv[2])
    out = Path(sys.argv[3])
    repeats = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    width = angles.shape[1]
    cfg = FeatureMapConfig(width, layers=2)
    t = time.perf_counter()
    template = simplify(circuit_to_network(compose_kernel_circuit(np.zeros(width),
                                                                  np.zeros(width), cfg)))
    plan = plan_contraction(template)
    plan_s = time.perf_counter() - t
    ops = [(angles[i], angles[j]) for i, j in pairs]
    workers = os.cpu_count() or 1
    runs, amps = [], None
    for _ in range(repeats):
        t = time.perf_counter()
        amps = contract_batch(template, ops, plan, workers=workers)
        runs.append(time.perf_counter() - t)
    med = float(np.median(runs))
    out.write_text(json.dumps({
        "entries_per_s": len(ops) / med, "pairs": len(ops), "plan_s": plan_s, "runs_s": runs,
        "workers": workers, "amplitudes_re": [float(np.real(a)) for a in amps],
        "amplitudes_im_max": float(max(abs(np.imag(a)) for a in amps))}))


if __name__ == "__main__":
    main()
