"""Generate the golden vectors by running the REFERENCE package itself.

Run in the build container only (it imports /root/reference/pkg/src/tnkernel, which does
not exist on the GPU box):

    python tests/golden/make_golden.py        # the contract_batch cases + known answers
    python tests/golden/make_golden.py sv     # the state-vector cases (sv_*.npz)
    python tests/golden/make_golden.py l4     # layers = 4 cases
    python tests/golden/make_golden.py deep   # layers 5 to 8 cases

Each case stores the angles, the pair list and the reference amplitudes returned by
``contract_batch(template, pairs, plan_contraction(template), workers)``
(reference: pkg/src/tnkernel/engine.py:132-166, paths.py:529-543, network.py:125-302),
i.e. the reference's own plan-once / rebind-per-pair path.  Gram cases additionally store
K = |amp|^2 over the strict upper triangle symmetrised as K + K^T + I.
Known answers from the reference tests are stored alongside (test_circuit.py:79-84,
test_statevector.py:63-70).
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    from tnkernel.circuit import FeatureMapConfig, compose_kernel_circuit
    from tnkernel.engine import contract_batch
    from tnkernel.network import circuit_to_network, simplify
    from tnkernel.paths import plan_contraction
    from tnkernel.statevector import kernel_entry_oracle

    return FeatureMapConfig, compose_kernel_circuit, contract_batch, circuit_to_network, \
        simplify, plan_contraction, kernel_entry_oracle


def ref_amplitudes(A, B, pairs, layers, workers=8):
    FMC, compose, contract_batch, c2n, simplify, plan_contraction, _ = _ref()
    n = A.shape[1]
    cfg = FMC(n, layers=layers)
    template = simplify(c2n(compose(np.zeros(n), np.zeros(n), cfg)))
    t0 = time.time()
    plan = plan_contraction(template)
    t_plan = time.time() - t0
    ops = [(A[p], B[q]) for p, q in pairs]
    t0 = time.time()
    amps = contract_batch(template, ops, plan, workers=workers)
    t_run = time.time() - t0
    return np.array(amps, dtype=np.complex128), t_plan, t_run


def clustered_angles(rng, N, n, spread, center_scale=np.pi):
    """Samples around a few random centres: small inter-sample angle differences keep the
    kernel away from the concentrated K ~ 0 regime (SURVEY finding 5)."""
    centres = rng.uniform(0, center_scale, (3, n))
    lab = rng.integers(0, 3, N)
    return centres[lab] + rng.normal(0.0, spread, (N, n))


def gram_case(name, rng, N, n, layers, spread, workers=8):
    X = clustered_angles(rng, N, n, spread)
    i, j = np.triu_indices(N, k=1)
    pairs = np.stack([i, j], 1).astype(np.int64)
    amps, tp, tr = ref_amplitudes(X, X, pairs, layers, workers)
    K = np.zeros((N, N))
    K[i, j] = np.abs(amps) ** 2
    K = K + K.T + np.eye(N)
    np.savez_compressed(OUT / f"{name}.npz", kind="gram", layers=layers, A=X, B=X, pairs=pairs,
                        amp_re=amps.real, amp_im=amps.imag, K=K)
    print(f"{name}: n={n} L={layers} pairs={len(pairs)} plan {tp:.2f}s run {tr:.2f}s "
          f"median K={np.median(K[i, j]):.3g}")


def cross_case(name, rng, Nt, Nr, n, layers, spread, workers=8):
    X = clustered_angles(rng, Nt + Nr, n, spread)
    T, R = X[:Nt], X[Nt:]
    r, c = np.meshgrid(np.arange(Nt), np.arange(Nr), indexing="ij")
    pairs = np.stack([r.ravel(), c.ravel()], 1).astype(np.int64)
    amps, tp, tr = ref_amplitudes(T, R, pairs, layers, workers)
    K = (np.abs(amps) ** 2).reshape(Nt, Nr)
    np.savez_compressed(OUT / f"{name}.npz", kind="cross", layers=layers, A=T, B=R, pairs=pairs,
                        amp_re=amps.real, amp_im=amps.imag, K=K)
    print(f"{name}: n={n} L={layers} pairs={len(pairs)} plan {tp:.2f}s run {tr:.2f}s "
          f"median K={np.median(K):.3g}")


def sampled_case(name, rng, N, n, layers, spread, n_pairs, workers=8):
    X = clustered_angles(rng, N, n, spread)
    i, j = np.triu_indices(N, k=1)
    sel = rng.choice(len(i), size=min(n_pairs, len(i)), replace=False)
    pairs = np.stack([i[sel], j[sel]], 1).astype(np.int64)
    amps, tp, tr = ref_amplitudes(X, X, pairs, layers, workers)
    np.savez_compressed(OUT / f"{name}.npz", kind="pairs", layers=layers, A=X, B=X, pairs=pairs,
                        amp_re=amps.real, amp_im=amps.imag)
    k = np.abs(amps) ** 2
    print(f"{name}: n={n} L={layers} pairs={len(pairs)} plan {tp:.2f}s run {tr:.2f}s "
          f"K range [{k.min():.3g}, {k.max():.3g}]")


def known_answers():
    FMC, compose, contract_batch, c2n, simplify, plan_contraction, oracle = _ref()
    rows = []
    # n = 1: amp = cos((b - a)/2)  (test_circuit.py:79-84)
    for a, b in [(0.3, 1.1), (-2.0, 0.5), (0.0, np.pi)]:
        for L in (1, 2, 3):
            rows.append((1, L, a, b, oracle([a], [b], FMC(1, layers=L), "magnitude")))
    # K(pi/2, 0) = 0.5 probability (test_statevector.py:63-70)
    rows.append((1, 2, np.pi / 2, 0.0, oracle([np.pi / 2], [0.0], FMC(1, layers=2))))
    np.savez_compressed(OUT / "known_answers.npz",
                        rows=np.array(rows, dtype=np.float64))
    print("known_answers:", len(rows))


def sv_cases():
    """Reference brute-force amplitudes (statevector.py:57-59 zero_amplitude of
    compose_kernel_circuit) for the GPU state-vector simulator's bit-identity test."""
    sys.path.insert(0, str(REF))
    from tnkernel.circuit import FeatureMapConfig, compose_kernel_circuit
    from tnkernel.statevector import zero_amplitude

    rng = np.random.default_rng(240502630 + 77)
    for n, L, n_pairs, spread in [(1, 2, 4, 1.0), (5, 1, 6, 0.8), (5, 2, 8, 0.8),
                                  (9, 2, 8, 0.4), (12, 3, 4, 0.3), (13, 2, 6, 0.3),
                                  (16, 2, 3, 0.2), (19, 2, 2, 0.15)]:
        X = clustered_angles(rng, 6, n, spread)
        pairs = rng.integers(0, 6, (n_pairs, 2)).astype(np.int64)
        cfg = FeatureMapConfig(n, layers=L)
        t0 = time.time()
        amps = np.array([zero_amplitude(compose_kernel_circuit(X[p], X[q], cfg))
                         for p, q in pairs], dtype=np.complex128)
        name = f"sv_n{n}_L{L}"
        np.savez_compressed(OUT / f"{name}.npz", kind="statevector", layers=L, A=X, B=X,
                            pairs=pairs, amp_re=amps.real, amp_im=amps.imag)
        print(f"{name}: {n_pairs} pairs in {time.time() - t0:.1f}s, "
              f"|amp| range [{np.abs(amps).min():.3g}, {np.abs(amps).max():.3g}]")


def l4_cases():
    """layers = 4 (bond-64 transfer): the reference's contract_batch (its planner slices)."""
    rng = np.random.default_rng(240502630 + 4)
    gram_case("gram_n5_L4", rng, 8, 5, 4, 0.4)
    sampled_case("pairs_n24_L4", rng, 10, 24, 4, 0.1, 12)


def deep_cases():
    """layers 5 to 8 (bond 4^(L-1) transfer; the GPU's shared-memory deep sweep): the
    reference's contract_batch on small widths (its cost grows ~4^L per qubit)."""
    rng = np.random.default_rng(240502630 + 5)
    gram_case("gram_n5_L5", rng, 8, 5, 5, 0.4)
    sampled_case("pairs_n24_L5", rng, 10, 24, 5, 0.1, 8)
    cross_case("cross_n7_L6", rng, 3, 4, 7, 6, 0.3)
    sampled_case("pairs_n10_L6", rng, 8, 10, 6, 0.2, 6)
    sampled_case("pairs_n8_L7", rng, 6, 8, 7, 0.3, 5)
    sampled_case("pairs_n6_L8", rng, 5, 6, 8, 0.4, 4)


def main():
    if sys.argv[1:] == ["deep"]:
        deep_cases()
        return
    if sys.argv[1:] == ["sv"]:
        sv_cases()
        return
    if sys.argv[1:] == ["l4"]:
        l4_cases()
        return
    rng = np.random.default_rng(240502630)
    known_answers()
    gram_case("gram_n8_L2", rng, 24, 8, 2, 0.35)
    cross_case("cross_n8_L2", rng, 6, 24, 8, 2, 0.35)
    gram_case("gram_n3_L2", rng, 9, 3, 2, 0.8)
    gram_case("gram_n17_L2", rng, 12, 17, 2, 0.2)
    gram_case("gram_n16_L1", rng, 12, 16, 1, 0.3)
    gram_case("gram_n6_L3", rng, 8, 6, 3, 0.4)
    sampled_case("pairs_n50_L2", rng, 40, 50, 2, 0.12, 60)
    sampled_case("pairs_n100_L2", rng, 40, 100, 2, 0.08, 40)
    sampled_case("pairs_n784_L2", rng, 16, 784, 2, 0.025, 24)
    sampled_case("pairs_n784_L2_spread", rng, 8, 784, 2, 1.0, 8)


if __name__ == "__main__":
    main()
