"""Per-CTA timeline of one sweep launch (needs the -DQK_TIMELINE build:
`python tools/build_variant.py tl -DQK_TIMELINE`, run with QK_LIB_PATH=.../libqk_tl.so).

Prints, averaged over CTAs: launch skew (first CTA entry to each CTA's entry), prologue
(entry -> first item start), and per item: claim-barrier gap (previous epilogue end -> item
start), first-stage wait, sweep, epilogue; plus each CTA's end relative to the first entry.
usage: QK_LIB_PATH=... python tools/timeline_probe.py --qubits 16 --n-train 1000 --n-test 1000"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2405_02630_b200 import SweepPlan, _native  # noqa: E402
from paper_2405_02630_b200 import device as qdev  # noqa: E402
from paper_2405_02630_b200.distributed import KernelJob  # noqa: E402

SLOTS = 256
ap = argparse.ArgumentParser()
ap.add_argument("--qubits", type=int, default=16)
ap.add_argument("--n-train", type=int, default=1000)
ap.add_argument("--n-test", type=int, default=1000)
ap.add_argument("--globaltimer", action="store_true")
a = ap.parse_args()
rng = np.random.default_rng(a.qubits)
tr = torch.as_tensor(rng.uniform(0, np.pi, (a.n_train, a.qubits)), device="cuda")
te = torch.as_tensor(rng.uniform(0, np.pi, (a.n_test, a.qubits)), device="cuda")
plan = SweepPlan(a.qubits, 2)
job = KernelJob(plan, a.n_train, a.n_test)
K, Kx = job.run(tr, te)
p_tr, p_te = qdev.gate_build(plan, tr), qdev.gate_build(plan, te)
lib = _native.lib()
fn = lib.qk_timeline_read
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
n_cta = torch.cuda.get_device_properties(0).multi_processor_count
buf = np.zeros((1024, SLOTS), dtype=np.uint64)
for _ in range(3):
    torch.cuda.synchronize()
    fn(buf.ctypes.data, 1024, 1)
    qdev.job_into(p_tr, p_te, K.data_ptr(), Kx.data_ptr())
    torch.cuda.synchronize()
    fn(buf.ctypes.data, 1024, 0)
t = buf[:n_cta].astype(np.float64)
if not a.globaltimer:  # SM cycles -> ns at the nominal clock
    t = t / 1.965
t0 = t[:, 0][t[:, 0] > 0].min()
us = lambda x: (x - t0) / 1e3  # noqa: E731
entry = us(t[:, 0])
pro = (t[:, 1] - t[:, 0]) / 1e3
items = []
for k in range(23):
    s, w, c, e = (t[:, 2 + 4 * k + j] for j in range(4))
    ok = (s > 0) & (e > 0)
    if not ok.any():
        break
    prev = t[:, 1] if k == 0 else t[:, 5 + 4 * (k - 1)]
    items.append({"k": k, "ctas": int(ok.sum()),
                  "gap_us": float(np.mean((s - prev)[ok]) / 1e3),
                  "first_stage_wait_us": float(np.mean((w - s)[ok]) / 1e3),
                  "sweep_us": float(np.mean((c - w)[ok]) / 1e3),
                  "epilogue_us": float(np.mean((e - c)[ok]) / 1e3),
                  "start_us_mean": float(np.mean(us(s[ok]))),
                  "issued_before_start_us": float(np.mean((s - t[:, 96 + k])[ok & (t[:, 96 + k] > 0)]) / 1e3),
                  "ready_at_start": float(np.mean(t[:, 128 + k][ok] == 2)),
                  "wait_us_warp0_idle": float(np.mean((w - s)[ok & (t[:, 192 + k] == 2)]) / 1e3) if (ok & (t[:, 192 + k] == 2)).any() else None,
                  "wait_us_warp0_busy": float(np.mean((w - s)[ok & (t[:, 192 + k] == 1)]) / 1e3) if (ok & (t[:, 192 + k] == 1)).any() else None,
                  "sweep_us_warp0_busy": float(np.mean((c - w)[ok & (t[:, 192 + k] == 1)]) / 1e3) if (ok & (t[:, 192 + k] == 1)).any() else None,
                  "released_after_start_us": float(np.mean((t[:, 160 + k] - s)[ok & (t[:, 160 + k] > 0)]) / 1e3)})
last = np.zeros(n_cta)
dur = np.zeros(n_cta)
n_items = np.zeros(n_cta, dtype=int)
for i in range(n_cta):
    marks = t[i][:96][t[i][:96] > 0]
    last[i] = us(marks.max())
    dur[i] = (marks.max() - t[i, 0]) / 1e3
    n_items[i] = int(sum(t[i, 5 + 4 * k] > 0 for k in range(23)))
print(json.dumps({"qubits": a.qubits, "n_train": a.n_train, "n_test": a.n_test,
                  "entry_skew_us": [float(entry.min()), float(np.median(entry)), float(entry.max())],
                  "prologue_us": [float(pro.min()), float(np.median(pro)), float(pro.max())],
                  "cta_end_us": [float(last.min()), float(np.median(last)), float(last.max())],
                  "cta_duration_us": [float(dur.min()), float(np.median(dur)), float(dur.max())],
                  "items_per_cta": np.bincount(n_items).tolist(),
                  "items": items}, indent=1))
