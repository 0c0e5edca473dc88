"""Pin the oracle (the CPU checker) to the reference's own outputs (tests/golden/*.npz,
produced by tests/golden/make_golden.py from the reference's contract_batch) and to the
reference tests' known answers."""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden
from oracle import oracle


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    amp = oracle.amplitudes(g["A"], g["B"], g["pairs"], int(g["layers"]), threads=4)
    ref = g["amp_re"] + 1j * g["amp_im"]
    assert np.all(np.abs(amp - ref) <= 1e-12 + 1e-9 * np.abs(ref))
    assert np.all(amp.imag == 0.0)  # RY/CNOT are real (reference asserts imag == 0.0)
    if "K" in g and str(g["kind"]) == "gram":
        K = oracle.kernel_matrix(g["A"], int(g["layers"]), threads=4)
        assert np.abs(K - g["K"]).max() <= 1e-12
        assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)
    if "K" in g and str(g["kind"]) == "cross":
        K = oracle.cross_kernel(g["A"], g["B"], int(g["layers"]), threads=4)
        assert np.abs(K - g["K"]).max() <= 1e-12


@pytest.mark.parametrize("name", [c for c in GOLDEN_CASES
                                  if load_golden(c)["A"].shape[1] <= 20])
def test_statevector_restatement_matches_golden(name):
    g = load_golden(name)
    ref = g["amp_re"] + 1j * g["amp_im"]
    for k in range(0, len(g["pairs"]), 7):
        p, q = g["pairs"][k]
        sv = oracle.statevector_amplitude(g["A"][p], g["B"][q], int(g["layers"]))
        assert abs(sv - ref[k]) <= 1e-12


def test_known_answers():
    rows = load_golden("known_answers")["rows"]
    for n, L, a, b, val in rows:
        amp = oracle.amplitudes(np.array([[a]]), np.array([[b]]), [[0, 0]], int(L))[0]
        if a == np.pi / 2 and b == 0.0:
            assert abs(amp) ** 2 == pytest.approx(val, abs=1e-15)  # K(pi/2, 0) = 0.5
        else:
            assert abs(amp) == pytest.approx(val, abs=1e-15)
            # one wire, no CNOTs: U(x) = RY(L x), amp = cos(L (b - a) / 2)
            assert abs(amp) == pytest.approx(abs(np.cos(L * (b - a) / 2)), abs=1e-15)


def test_identical_features_give_unit_amplitude(rng):
    for L in (1, 2, 3):
        x = rng.uniform(-3, 3, (1, 11))
        assert oracle.amplitudes(x, x, [[0, 0]], L)[0] == pytest.approx(1.0, abs=1e-12)


def test_thread_count_does_not_change_results(rng):
    X = rng.uniform(0, np.pi, (12, 9))
    pairs = oracle.upper_pairs(12)
    a1 = oracle.amplitudes(X, X, pairs, 2, threads=1)
    a4 = oracle.amplitudes(X, X, pairs, 2, threads=4)
    assert np.array_equal(a1, a4)  # bit-identical across workers (test_engine.py:110-120)


def test_empty_and_bad_inputs():
    assert oracle.amplitudes(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 2))).size == 0
    with pytest.raises(IndexError):
        oracle.amplitudes(np.zeros((1, 3)), np.zeros((1, 3)), [[0, 1]])
