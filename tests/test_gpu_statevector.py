"""GPU state-vector simulator (paper_2405_02630_b200.statevector, csrc/qk_statevector.cu):
bit-identical to the reference's brute-force simulate() on its own golden amplitudes
(tests/golden/sv_*.npz from statevector.py zero_amplitude), and the independent check of the
tile sweep at widths beyond the reference's 24-qubit guard."""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2405_02630_b200 import FeatureMapConfig, SweepPlan, compute_kernel_matrix  # noqa: E402
from paper_2405_02630_b200 import device as dev  # noqa: E402
from paper_2405_02630_b200 import statevector as sv  # noqa: E402

SV_CASES = [c for c in GOLDEN_CASES if c.startswith("sv_")]


@pytest.mark.parametrize("name", SV_CASES)
def test_bit_identical_to_reference_simulator(name):
    g = load_golden(name)
    cfg = FeatureMapConfig(g["A"].shape[1], int(g["layers"]))
    amp = sv.amplitudes(g["A"], g["B"], g["pairs"], cfg)
    assert np.array_equal(amp, g["amp_re"]) and np.all(g["amp_im"] == 0.0)
    # the one-pair whole-GPU path gives the same bits as the batched shared-memory path
    p, q = g["pairs"][0]
    assert sv.zero_amplitude(g["A"][p], g["B"][q], cfg) == g["amp_re"][0]


def _clustered(rng, N, n, spread):
    return rng.uniform(0, np.pi, n)[None, :] + rng.normal(0.0, spread, (N, n))


@pytest.mark.parametrize("n,layers,spread", [(22, 2, 0.12), (26, 2, 0.1), (28, 1, 0.15),
                                             (24, 3, 0.08)])
def test_sweep_matches_statevector_beyond_the_reference_guard(n, layers, spread):
    rng = np.random.default_rng(n * 10 + layers)
    X = _clustered(rng, 3, n, spread)
    pairs = np.array([[0, 1], [1, 2], [2, 0]], dtype=np.int64)
    cfg = FeatureMapConfig(n, layers)
    ref = sv.amplitudes(X, X, pairs, cfg)
    plan = SweepPlan(n, layers)
    P = dev.gate_build(plan, torch.as_tensor(X, device="cuda"))
    amp = dev.pair_amplitudes(P, P, torch.as_tensor(pairs, device="cuda")).cpu().numpy()
    assert np.abs(amp ** 2 - ref ** 2).max() <= 1e-12
    assert np.all(np.abs(amp - ref) <= 1e-9 * np.abs(ref) + 1e-300)
    assert np.abs(ref).min() > 1e-6  # a meaningful (non-concentrated) check
    # the dense Gram from the tile sweep agrees as well
    K = compute_kernel_matrix(X, cfg).entries
    assert abs(K[0, 1] - ref[0] ** 2) <= 1e-12 and abs(K[1, 2] - ref[1] ** 2) <= 1e-12


def test_config1_gram_against_statevector():
    """C1-shaped (8 qubits, 100 samples): the whole Gram by brute force, one CTA per pair."""
    from paper_2405_02630_b200.data import config_data

    Atr, _, _, _ = config_data(1, 100, 50, "mnist", features=8, binary=(2, 6))
    cfg = FeatureMapConfig(8)
    i, j = np.triu_indices(len(Atr), k=1)
    amp = sv.amplitudes(Atr, Atr, np.stack([i, j], 1), cfg)
    K = compute_kernel_matrix(Atr, cfg).entries
    assert np.abs(K[i, j] - amp ** 2).max() <= 1e-12
    assert sv.kernel_entry_oracle(Atr[0], Atr[0], cfg) == 1.0 or \
        abs(sv.kernel_entry_oracle(Atr[0], Atr[0], cfg) - 1.0) <= 1e-14


def test_guards_and_conventions():
    from paper_2405_02630_b200 import CapacityError

    with pytest.raises(CapacityError, match="33 qubits exceeds the 32-qubit guard"):
        sv.zero_amplitude(np.zeros(33), np.zeros(33), FeatureMapConfig(33))
    with pytest.raises(ValueError, match="finite"):
        sv.zero_amplitude([np.nan, 0.0], [0.0, 0.0], FeatureMapConfig(2))
    with pytest.raises(ValueError, match="unknown kernel convention"):
        sv.kernel_entry_oracle([0.1], [0.2], FeatureMapConfig(1), "nope")
    # the reference tests' known answers (test_circuit.py:79-84, test_statevector.py:63-70),
    # as the reference's own kernel_entry_oracle returned them (tests/golden/known_answers)
    rows = load_golden("known_answers")["rows"]
    for k, (n, L, a, b, val) in enumerate(rows):
        conv = "magnitude" if k < len(rows) - 1 else "probability"
        assert sv.kernel_entry_oracle([a], [b], FeatureMapConfig(int(n), int(L)), conv) == val
