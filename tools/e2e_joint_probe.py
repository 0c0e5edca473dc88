"""Phase timing of the joint host pipeline (QK_TRACE=1 → qk_trace lines on stderr) next to the
device-only job, config 4.  Usage: python tools/e2e_joint_probe.py [reps]"""
import os
import sys
import time
from pathlib import Path

os.environ["QK_TRACE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices, plan_for  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200.data import config_data  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Atr, _, Ate, _ = config_data(4, 10000, 2000, "mnist", bw=1.0)
cfg = FeatureMapConfig(784)
h_tr = torch.from_numpy(Atr).pin_memory().numpy()
h_te = torch.from_numpy(Ate).pin_memory().numpy()
h_K = torch.empty((10000, 10000), dtype=torch.float64).pin_memory().numpy()
h_Kx = torch.empty((2000, 10000), dtype=torch.float64).pin_memory().numpy()
for r in range(reps):
    t = time.perf_counter()
    compute_kernel_matrices(h_tr, h_te, cfg, out_train=h_K, out_test=h_Kx)
    print(f"joint_host_ms {1e3 * (time.perf_counter() - t):.3f}", file=sys.stderr, flush=True)
plan = plan_for(cfg)
tr = torch.as_tensor(Atr, device="cuda"); te = torch.as_tensor(Ate, device="cuda")
K = torch.empty((10000, 10000), dtype=torch.float64, device="cuda")
Kx = torch.empty((2000, 10000), dtype=torch.float64, device="cuda")
for r in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    p = dev.gate_build(plan, tr); q = dev.gate_build(plan, te)
    dev.job_into(p, q, K.data_ptr(), Kx.data_ptr())
    e.record(); torch.cuda.synchronize()
    print(f"device_job_ms {s.elapsed_time(e):.3f}", file=sys.stderr, flush=True)
