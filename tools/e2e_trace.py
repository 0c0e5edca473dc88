"""Host-pipeline phase timing (QK_TRACE=1 prints h2d / gate / sweep / tail / host per call):
config 4 (10,000 x 784 train, 2,000 test) through compute_kernel_matrices with pinned
buffers, or (--pageable) plain numpy arrays in and fresh ones out.
usage: QK_TRACE=1 [QK_HEAD_SPLIT=0] python tools/e2e_trace.py [calls] [--pageable]
       [--shape N_TRAIN,N_TEST,QUBITS]   (default 10000,2000,784)"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices  # noqa: E402


def pin(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
    t[...] = a
    return t


pageable = "--pageable" in sys.argv
shape = (10000, 2000, 784)
if "--shape" in sys.argv:
    shape = tuple(int(v) for v in sys.argv[sys.argv.index("--shape") + 1].split(","))
args = [a for a in sys.argv[1:] if not a.startswith("--") and "," not in a]
rng = np.random.default_rng(0)
N, M, n = shape
X = rng.uniform(0, np.pi, (N, n))
T = rng.uniform(0, np.pi, (M, n))
kw = {}
if not pageable:
    X, T = pin(X), pin(T)
    kw = {"out_train": pin(np.empty((N, N))), "out_test": pin(np.empty((M, N)))}
cfg = FeatureMapConfig(n)
for _ in range(int(args[0]) if args else 4):
    t = time.perf_counter()
    compute_kernel_matrices(X, T, cfg, **kw)
    print(f"wall {(time.perf_counter() - t) * 1e3:.3f} ms", flush=True)
