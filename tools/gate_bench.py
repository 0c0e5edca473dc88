"""Gate-build kernel alone: algorithmic HBM bandwidth (8 B angle read + 16 B plane write per
(sample, plane qubit)), CUDA events around each launch, a 512 MB L2 flush between launches
(cold inputs, like the bench step), median of 20.  One JSON line per case."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan, _native  # noqa: E402
from paper_2405_02630_b200 import device as qdev  # noqa: E402


def case(n, n_a, n_b, reps=20):
    plan = SweepPlan(n, 2)
    rng = np.random.default_rng(0)
    A = torch.as_tensor(rng.uniform(0, np.pi, (n_a, n)), device="cuda")
    B = torch.as_tensor(rng.uniform(0, np.pi, (max(n_b, 1), n)), device="cuda")
    pa = torch.empty(plan.planes_bytes(n_a), dtype=torch.uint8, device="cuda")
    pb = torch.empty(max(plan.planes_bytes(n_b), 16), dtype=torch.uint8, device="cuda")
    bad = torch.full((3,), -1, dtype=torch.int64, device="cuda")
    Ktr = torch.empty((1, 1), dtype=torch.float64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    lib = _native.lib()
    st = torch.cuda.current_stream().cuda_stream
    times = []
    for _ in range(reps + 2):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        # qk_job_run with an empty tile range: the sentinel reset + the gate build of both sets
        _native.check(lib.qk_job_run(plan.handle, A.data_ptr(), n_a,
                                     B.data_ptr() if n_b else None, n_b, pa.data_ptr(),
                                     pb.data_ptr() if n_b else None, bad.data_ptr(), 0, 0,
                                     Ktr.data_ptr(), Ktr.data_ptr() if n_b else None, st))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(times[2:]))
    blocks = lambda m: -(-m // 64) if m else 0  # noqa: E731
    n_pad = plan.info["width_padded"]
    nbytes = 8 * n * (n_a + n_b) + 16 * n_pad * 64 * (blocks(n_a) + blocks(n_b))
    return {"qubits": n, "n_a": n_a, "n_b": n_b, "us": t * 1e6, "alg_bytes": nbytes,
            "alg_TBps": nbytes / t / 1e12}


if __name__ == "__main__":
    for args in ((784, 10000, 0), (784, 10000, 2000), (784, 2000, 0), (50, 1000, 500)):
        print(json.dumps(case(*args)), flush=True)
