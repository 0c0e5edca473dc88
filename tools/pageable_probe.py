"""Where the pageable e2e call (config 4, plain numpy in and out) spends its wall time outside
the traced GPU phases: output allocation, the call itself, and the release of the previous
call's 960 MB of results.  One line per variant, median of 5 calls.

usage: [QK_TRACE=1] python tools/pageable_probe.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices  # noqa: E402
from paper_2405_02630_b200.kernel_pipeline import host_empty  # noqa: E402

X, T = bench.workload_data()
cfg = FeatureMapConfig(784)
compute_kernel_matrices(X, T, cfg)


def med(v):
    return round(float(np.median(v)) * 1e3, 3)


alloc, call, free, keep = [], [], [], []
for _ in range(5):
    t0 = time.perf_counter()
    K = host_empty((10000, 10000))
    Kx = host_empty((2000, 10000))
    t1 = time.perf_counter()
    r = compute_kernel_matrices(X, T, cfg, out_train=K, out_test=Kx)
    t2 = time.perf_counter()
    del r, K, Kx
    t3 = time.perf_counter()
    alloc.append(t1 - t0), call.append(t2 - t1), free.append(t3 - t2)
print(json.dumps({"variant": "fresh outputs", "alloc_ms": med(alloc), "call_ms": med(call),
                  "free_ms": med(free)}), flush=True)
K = host_empty((10000, 10000))
Kx = host_empty((2000, 10000))
for _ in range(5):
    t1 = time.perf_counter()
    compute_kernel_matrices(X, T, cfg, out_train=K, out_test=Kx)
    keep.append(time.perf_counter() - t1)
print(json.dumps({"variant": "reused (already faulted) pageable outputs",
                  "call_ms": med(keep)}), flush=True)
plain = []
for _ in range(5):
    t1 = time.perf_counter()
    compute_kernel_matrices(X, T, cfg)
    plain.append(time.perf_counter() - t1)
print(json.dumps({"variant": "default call, result dropped", "call_ms": med(plain)}), flush=True)
