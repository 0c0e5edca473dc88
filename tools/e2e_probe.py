"""Where does the end-to-end time go?  Times the pieces of the bench's e2e step separately."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import (FeatureMapConfig, compute_cross_kernel,  # noqa: E402
                                   compute_kernel_matrix, plan_for)
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200.data import config_data  # noqa: E402

out = {}
d = torch.empty(960_000_000 // 8, dtype=torch.float64, device="cuda")
h = torch.empty_like(d, device="cpu").pin_memory()
for name, fn in [("d2h_pinned_GBs", lambda: h.copy_(d)), ("h2d_pinned_GBs", lambda: d.copy_(h))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize()
    out[name] = 0.96 / (time.perf_counter() - t)
del d, h
Atr, _, Ate, _ = config_data(4, 10000, 2000, "mnist", bw=1.0)
cfg = FeatureMapConfig(784)
h_tr = torch.from_numpy(Atr).pin_memory().numpy()
h_te = torch.from_numpy(Ate).pin_memory().numpy()
h_K = torch.empty((10000, 10000), dtype=torch.float64).pin_memory().numpy()
h_Kx = torch.empty((2000, 10000), dtype=torch.float64).pin_memory().numpy()
for rep in range(3):
    t = time.perf_counter(); compute_kernel_matrix(h_tr, cfg, out=h_K); t1 = time.perf_counter()
    compute_cross_kernel(h_te, h_tr, cfg, out=h_Kx); t2 = time.perf_counter()
out["gram_host_ms"] = 1e3 * (t1 - t)
out["cross_host_ms"] = 1e3 * (t2 - t1)
for rep in range(2):
    t = time.perf_counter(); compute_kernel_matrix(Atr, cfg); out[f"gram_host_default_out_ms_{rep}"] = 1e3 * (time.perf_counter() - t)
    t = time.perf_counter(); compute_kernel_matrix(Atr, cfg, out=np.empty((10000, 10000))); out[f"gram_host_npempty_out_ms_{rep}"] = 1e3 * (time.perf_counter() - t)
plan = plan_for(cfg)
tr = torch.as_tensor(Atr, device="cuda"); te = torch.as_tensor(Ate, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    p = dev.gate_build(plan, tr); K = dev.gram(p); torch.cuda.synchronize(); t1 = time.perf_counter()
    q = dev.gate_build(plan, te); Kx = dev.cross(q, p); torch.cuda.synchronize(); t2 = time.perf_counter()
    out[f"gram_device_ms_{rep}"] = 1e3 * (t1 - t)
    out[f"cross_device_ms_{rep}"] = 1e3 * (t2 - t1)
print(json.dumps(out))
