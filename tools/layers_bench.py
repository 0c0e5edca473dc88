"""Entries/s of the train Gram by feature-map depth L = 1..8 on one GPU (device-resident
angles, CUDA events, one warm-up), with the planner's executed FP64 flops per entry -> TFLOP/s.
Prints one JSON line per L.  usage: python tools/layers_bench.py [L | L:width:samples ...]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402

# (width, samples) per L: ~0.1-2 s per Gram
CASES = {1: (784, 8192), 2: (784, 4096), 3: (784, 1024), 4: (784, 512), 5: (784, 160),
         6: (784, 64), 7: (128, 48), 8: (32, 40)}


def point(L, n=None, N=None):
    if n is None:
        n, N = CASES[L]
    rng = np.random.default_rng(L)
    X = torch.as_tensor(rng.uniform(0, np.pi, (N, n)), device="cuda")
    plan = SweepPlan(n, L)
    planes = dev.gate_build(plan, X)
    out = torch.empty((N, N), dtype=torch.float64, device="cuda")
    dev.gram(planes, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.time()
    e0.record()
    reps = 0
    while True:
        dev.gram(planes, out=out)
        reps += 1
        torch.cuda.synchronize()
        if time.time() - t > 1.0 or reps >= 20:
            break
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3 / reps
    entries = N * (N - 1) // 2
    info = plan.info
    return {"layers": L, "qubits": n, "samples": N, "entries": entries, "s_per_gram": s,
            "entries_per_s": entries / s, "bond": info["bond"],
            "dp_instr_per_entry": info["dp_instr_per_entry"],
            "tflops_executed": entries * info["flops_per_entry"] / s / 1e12}


if __name__ == "__main__":
    for a in sys.argv[1:] or [str(L) for L in CASES]:
        f = [int(v) for v in a.split(":")]
        print(json.dumps(point(*f)), flush=True)
