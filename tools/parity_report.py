"""Parity report over the BASELINE configs (run on a GPU box): the engine's kernel matrices
against the CPU oracle (oracle/, pinned to the reference's own outputs) on the same inputs —
EVERY entry of every config, 784-qubit ones included — plus the downstream precomputed-kernel
SVC (binary for configs 1-2, 10-class one-vs-rest for 3-4): predictions and decision values
from the engine's K against those from the oracle's K.

The 784-qubit configs use bandwidth-scaled angles (median off-diagonal K in [1e-3, 0.5],
SURVEY.md §8(d)) on overlapping classes (data.synthetic_images(mix=0.6)), so one-vs-rest
accuracy is well below 1 and "identical predictions" is a real gate.

usage: python tools/parity_report.py [out.json] [--configs 1,2,3,4] [--merge earlier.json]
Writes the JSON report (partial results after every chunk, so a cut-off run still leaves
evidence) and prints it at the end.  Reference: PAPER.md:322-326 (10-class accuracy table),
SPEC.md:407-424, engine.py:132-166."""
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

THREADS = oracle.default_threads()
K_ABS = 1e-12


def amp_err(K, Kr):
    """Worst |amp - amp_ref| / (1e-9 |amp_ref| + 1e-18): <= 1 passes the amplitude gate of the
    GPU parity tests (relative 1e-9, with a 1e-18 floor for amplitudes that are themselves
    cancellation residues of much larger terms)."""
    a, b = np.sqrt(K), np.sqrt(Kr)
    return float(np.max(np.abs(a - b) / (1e-9 * b + 1e-18)))


def svc(K, ytr, Kx, ovr):
    from sklearn.multiclass import OneVsRestClassifier
    from sklearn.svm import SVC
    m = SVC(kernel="precomputed", C=1.0)
    m = OneVsRestClassifier(m, n_jobs=min(10, THREADS)) if ovr else m
    m.fit(K, ytr)
    return m.predict(Kx), m.decision_function(Kx)


def oracle_blocks(Atr, Ate, rows_per_chunk, log):
    """Oracle Gram (strict upper, mirrored, unit diagonal) and cross block, computed in row
    chunks so progress is visible; yields nothing, returns (K, Kx, seconds)."""
    n_tr, n_te = len(Atr), len(Ate)
    K = np.eye(n_tr)
    Kx = np.empty((n_te, n_tr))
    t0 = time.perf_counter()
    done, total = 0, n_tr * (n_tr - 1) // 2 + n_te * n_tr
    for r0 in range(0, n_tr, rows_per_chunk):
        r1 = min(n_tr, r0 + rows_per_chunk)
        rows = np.arange(r0, r1)
        pi = np.repeat(rows, n_tr - 1 - rows)
        pj = np.concatenate([np.arange(r + 1, n_tr) for r in rows])
        if len(pi):
            v = np.abs(oracle.amplitudes(Atr, Atr, np.stack([pi, pj], 1), 2,
                                         threads=THREADS)) ** 2
            K[pi, pj] = v
            K[pj, pi] = v
            done += len(pi)
        log(done, total, time.perf_counter() - t0)
    for r0 in range(0, n_te, rows_per_chunk):
        r1 = min(n_te, r0 + rows_per_chunk)
        r, c = np.meshgrid(np.arange(r0, r1), np.arange(n_tr), indexing="ij")
        Kx[r0:r1] = (np.abs(oracle.amplitudes(Ate, Atr, np.stack([r.ravel(), c.ravel()], 1), 2,
                                              threads=THREADS)) ** 2).reshape(r1 - r0, n_tr)
        done += (r1 - r0) * n_tr
        log(done, total, time.perf_counter() - t0)
    return K, Kx, time.perf_counter() - t0


def case(cid, n_tr, n_te, kind, *, features=None, binary=None, bw=1.0, mix=0.0, chunk=0,
         progress=None):
    Atr, ytr, Ate, yte = config_data(cid, n_tr, n_te, kind, features=features, binary=binary,
                                     bw=bw, mix=mix)
    assert (len(Atr), len(Ate)) == (n_tr, n_te), (len(Atr), len(Ate))
    cfg = FeatureMapConfig(Atr.shape[1])
    t = time.perf_counter()
    K, Kx = compute_kernel_matrices(Atr, Ate, cfg)
    t_gpu = time.perf_counter() - t
    K, Kx = K.entries, Kx.entries

    def log(done, total, sec):
        if progress is not None:
            progress({"config": cid, "oracle_entries_done": int(done),
                      "oracle_entries_total": int(total), "oracle_s": round(sec, 1)})

    Kr, Kxr, t_cpu = oracle_blocks(Atr, Ate, chunk or n_tr, log)
    iu = np.triu_indices(n_tr, 1)
    ovr = binary is None
    t = time.perf_counter()
    p, dec = svc(K, ytr, Kx, ovr)
    pr, decr = svc(Kr, ytr, Kxr, ovr)
    t_svc = time.perf_counter() - t
    return {"config": cid, "kind": kind, "qubits": int(Atr.shape[1]), "layers": 2,
            "n_train": n_tr, "n_test": n_te, "angle_bandwidth": bw if features is None else None,
            "class_mix": mix, "classes": 2 if binary else 10,
            "entries_checked": int(n_tr * (n_tr - 1) // 2 + n_te * n_tr),
            "entries_total": int(n_tr * (n_tr - 1) // 2 + n_te * n_tr), "scope": "every entry",
            "max_abs_dK": float(max(np.abs(K - Kr).max(), np.abs(Kx - Kxr).max())),
            "max_abs_dK_gram": float(np.abs(K - Kr).max()),
            "max_abs_dK_cross": float(np.abs(Kx - Kxr).max()),
            "within_1e-12": bool(max(np.abs(K - Kr).max(), np.abs(Kx - Kxr).max()) <= K_ABS),
            "amp_gate_ratio": max(amp_err(K, Kr), amp_err(Kx, Kxr)),
            "median_K_offdiag": float(np.median(Kr[iu])), "median_K_cross": float(np.median(Kxr)),
            "gram_symmetric_exact": bool(np.array_equal(K, K.T)),
            "gram_diag_exact_1": bool(np.all(np.diag(K) == 1.0)),
            "range_ok": bool(K.min() >= 0 and K.max() <= 1 + 1e-9 and Kx.min() >= 0
                             and Kx.max() <= 1 + 1e-9),
            "svc": "OneVsRestClassifier(SVC(kernel='precomputed', C=1))" if ovr
                   else "SVC(kernel='precomputed', C=1)",
            "svc_predictions_identical": bool(np.array_equal(p, pr)),
            "svc_decision_max_abs_diff": float(np.abs(np.asarray(dec) - np.asarray(decr)).max()),
            "svc_accuracy_engine_K": float((p == yte).mean()),
            "svc_accuracy_oracle_K": float((pr == yte).mean()),
            "gpu_call_s": round(t_gpu, 3), "oracle_s": round(t_cpu, 1),
            "oracle_threads": THREADS, "svc_s": round(t_svc, 1)}


CASES = {
    1: dict(cid=1, n_tr=100, n_te=50, kind="mnist", features=8, binary=(2, 6)),
    2: dict(cid=2, n_tr=1000, n_te=500, kind="mnist", features=50, binary=(2, 6)),
    3: dict(cid=3, n_tr=2000, n_te=1000, kind="fashion", bw=0.06, mix=0.6, chunk=250),
    4: dict(cid=4, n_tr=10000, n_te=2000, kind="mnist", bw=0.06, mix=0.6, chunk=500),
}


def main():
    args = [a for k, a in enumerate(sys.argv[1:], 1)
            if not a.startswith("--") and sys.argv[k - 1] not in ("--configs", "--merge")]
    out = Path(args[0]) if args else None
    cfgs = [1, 2, 3, 4]
    if "--configs" in sys.argv:
        cfgs = [int(c) for c in sys.argv[sys.argv.index("--configs") + 1].split(",")]
    import torch
    rep = {"tolerances": {"abs_dK": K_ABS,
                          "amp": "|da| <= 1e-9 |a| + 1e-18 (amp_gate_ratio <= 1)",
                          "svc": "identical predictions from engine K and oracle K"},
           "oracle": "oracle/qk_oracle.c (complex128 TN contraction of the uncancelled kernel "
                     "network), pinned to the reference's contract_batch goldens "
                     "(tests/test_oracle.py)",
           "gpu": torch.cuda.get_device_name(0), "host_threads": THREADS,
           "cpu_model": _cpu_model(), "cases": [], "progress": None}

    def dump():
        if out is not None:
            out.write_text(json.dumps(rep, indent=1))

    def progress(p):
        rep["progress"] = p
        dump()

    if "--merge" in sys.argv:  # keep the other configs' cases of an earlier report
        old = json.loads(Path(sys.argv[sys.argv.index("--merge") + 1]).read_text())
        rep["cases"] = [c for c in old["cases"] if c["config"] not in cfgs]
    for c in cfgs:
        rep["cases"].append(case(**CASES[c], progress=progress))
        rep["cases"].sort(key=lambda c: c["config"])
        rep["progress"] = None
        dump()
    rep["all_within_1e-12"] = all(c["within_1e-12"] for c in rep["cases"])
    rep["all_predictions_identical"] = all(c["svc_predictions_identical"] for c in rep["cases"])
    dump()
    print(json.dumps(rep, indent=1))


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if __name__ == "__main__":
    main()
