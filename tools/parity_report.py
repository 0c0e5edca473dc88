"""Parity report over the BASELINE configs (run on a GPU box): the engine's kernel matrices
against the CPU oracle (oracle/, pinned to the reference's own outputs) on the same inputs —
every entry where the oracle can afford it (configs 1, 2), sampled entries at 784 qubits
(configs 3, 4) — plus the downstream precomputed-kernel SVC predictions.  Prints one JSON
object; tools/parity_report.py > profiles/r1_parity.json."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle  # noqa: E402  (the checker)
from paper_2405_02630_b200 import FeatureMapConfig, compute_kernel_matrices  # noqa: E402
from paper_2405_02630_b200.data import config_data  # noqa: E402

THREADS = os.cpu_count() or 1


def amp_err(K, Kr):
    """Worst |amp - amp_ref| / (1e-9 |amp_ref| + 1e-18): <= 1 passes the amplitude gate of the
    GPU parity tests (relative 1e-9, with a 1e-18 floor for amplitudes that are themselves
    cancellation residues of much larger terms)."""
    a, b = np.sqrt(K), np.sqrt(Kr)
    return float(np.max(np.abs(a - b) / (1e-9 * b + 1e-18)))


def svc(K, ytr, Kx, yte, ovr):
    from sklearn.multiclass import OneVsRestClassifier
    from sklearn.svm import SVC
    m = SVC(kernel="precomputed", C=1.0)
    m = OneVsRestClassifier(m) if ovr else m
    p = m.fit(K, ytr).predict(Kx)
    return p, float((p == yte).mean())


def full_case(cid, n_tr, n_te, kind, features, binary):
    Atr, ytr, Ate, yte = config_data(cid, n_tr, n_te, kind, features=features, binary=binary)
    cfg = FeatureMapConfig(Atr.shape[1])
    t = time.perf_counter()
    K, Kx = compute_kernel_matrices(Atr, Ate, cfg)
    t_gpu = time.perf_counter() - t
    t = time.perf_counter()
    Kr, Kxr = oracle.kernel_matrix(Atr, 2, threads=THREADS), oracle.cross_kernel(Ate, Atr, 2,
                                                                                threads=THREADS)
    t_cpu = time.perf_counter() - t
    p, acc = svc(K.entries, ytr, Kx.entries, yte, ovr=binary is None)
    pr, accr = svc(Kr, ytr, Kxr, yte, ovr=binary is None)
    return {"config": cid, "qubits": int(Atr.shape[1]), "n_train": n_tr, "n_test": n_te,
            "entries_checked": int(n_tr * (n_tr - 1) // 2 + n_te * n_tr), "scope": "every entry",
            "max_abs_dK": float(max(np.abs(K.entries - Kr).max(), np.abs(Kx.entries - Kxr).max())),
            "amp_gate_ratio": max(amp_err(K.entries, Kr), amp_err(Kx.entries, Kxr)),
            "median_K": float(np.median(Kr[np.triu_indices(n_tr, 1)])),
            "gram_symmetric_exact": bool(np.array_equal(K.entries, K.entries.T)),
            "gram_diag_exact_1": bool(np.all(np.diag(K.entries) == 1.0)),
            "svc_predictions_identical": bool(np.array_equal(p, pr)),
            "svc_accuracy": acc, "svc_accuracy_oracle_K": accr,
            "gpu_s": t_gpu, "oracle_s": t_cpu, "oracle_threads": THREADS}


def sampled_case(cid, n_tr, n_te, kind, bw, n_samp, ovr_acc):
    Atr, ytr, Ate, yte = config_data(cid, n_tr, n_te, kind, bw=bw)
    cfg = FeatureMapConfig(784)
    K, Kx = compute_kernel_matrices(Atr, Ate, cfg)
    rng = np.random.default_rng(cid)
    i, j = rng.integers(0, n_tr, n_samp), rng.integers(0, n_tr, n_samp)
    keep = i != j
    i, j = i[keep], j[keep]
    ref = np.abs(oracle.amplitudes(Atr, Atr, np.stack([i, j], 1), 2, threads=THREADS)) ** 2
    r, c = rng.integers(0, n_te, n_samp), rng.integers(0, n_tr, n_samp)
    refx = np.abs(oracle.amplitudes(Ate, Atr, np.stack([r, c], 1), 2, threads=THREADS)) ** 2
    got, gotx = K.entries[i, j], Kx.entries[r, c]
    out = {"config": cid, "qubits": 784, "n_train": n_tr, "n_test": n_te, "angle_bandwidth": bw,
           "entries_checked": int(len(i) + len(r)), "scope": "sampled entries",
           "max_abs_dK": float(max(np.abs(got - ref).max(), np.abs(gotx - refx).max())),
           "amp_gate_ratio": max(amp_err(got, ref), amp_err(gotx, refx)),
           "median_K": float(np.median(ref)),
           "gram_symmetric_exact": bool(np.array_equal(K.entries, K.entries.T)),
           "gram_diag_exact_1": bool(np.all(np.diag(K.entries) == 1.0)),
           "range_ok": bool(K.entries.min() >= 0 and K.entries.max() <= 1 + 1e-9)}
    if ovr_acc:
        _, acc = svc(K.entries, ytr, Kx.entries, yte, ovr=True)
        out["svc_ovr_accuracy"] = acc
    return out


if __name__ == "__main__":
    rep = {"tolerances": {"abs_dK": 1e-12, "amp": "|da| <= 1e-9 |a| + 1e-18 (amp_gate_ratio <= 1)"},
           "oracle": "oracle/qk_oracle.c (complex128 TN contraction of the uncancelled kernel "
                     "network), pinned to the reference's contract_batch goldens",
           "cases": [full_case(1, 100, 50, "mnist", 8, (2, 6)),
                     full_case(2, 1000, 500, "mnist", 50, (2, 6)),
                     sampled_case(3, 2000, 1000, "fashion", 0.02, 2000, True),
                     sampled_case(4, 10000, 2000, "mnist", 0.05, 2000, False)]}
    print(json.dumps(rep, indent=1))
