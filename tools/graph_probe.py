"""Small jobs: host-launch overhead vs a CUDA-graph replay of KernelJob.run (device inputs).
Prints ms per job both ways for 1000 x 1000 at several widths and checks equal results."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402


def timed(fn, steps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for n in (16, 64, 256, 784):
    rng = np.random.default_rng(n)
    tr = torch.as_tensor(rng.uniform(0, np.pi, (1000, n)), device="cuda")
    te = torch.as_tensor(rng.uniform(0, np.pi, (1000, n)), device="cuda")
    job = KernelJob(SweepPlan(n, 2), 1000, 1000)
    K0, Kx0 = [t.clone() for t in job.run(tr, te)]
    plain = timed(lambda: job.run(tr, te))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        job.run(tr, te)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        K, Kx = job.run(tr, te)
    graph = timed(g.replay)
    same = bool(torch.equal(K, K0) and torch.equal(Kx, Kx0))
    print(json.dumps({"qubits": n, "ms_plain": plain, "ms_graph": graph, "same": same}), flush=True)
