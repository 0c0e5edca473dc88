"""layers 5..8 on the GPU (the shared-memory deep sweep, bond 4^(L-1) = 256..16384 per pair)
and the factored register sweep of layers 3, 4, against the oracle (pinned to the reference's
own contract_batch output in tests/golden/*_L5..L8) — Gram, cross, packed tiles + unpack,
the pair-list kernel behind contract_batch, and the host pipeline."""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import oracle
from paper_2405_02630_b200 import (CapacityError, FeatureMapConfig, SweepPlan,
                                   compute_cross_kernel, compute_kernel_matrices,
                                   compute_kernel_matrix, contract_batch)
from paper_2405_02630_b200 import device as dev

pytestmark = pytest.mark.gpu

K_ABS = 1e-12
AMP_REL = 1e-9


def _clustered(rng, N, n, spread):
    centre = rng.uniform(0, np.pi, n)
    return centre + rng.normal(0, spread, (N, n))


@pytest.mark.parametrize("L,n,N", [(5, 1, 4), (5, 5, 70), (5, 17, 40), (6, 4, 66), (6, 9, 20),
                                   (7, 6, 12), (8, 3, 9), (8, 5, 5)])
def test_gram_and_cross_vs_oracle(L, n, N, rng):
    X = _clustered(rng, N, n, 0.5 / np.sqrt(n))
    T = _clustered(rng, 3, n, 0.5 / np.sqrt(n))
    cfg = FeatureMapConfig(n, layers=L)
    K = compute_kernel_matrix(X, cfg).entries
    Kx = compute_cross_kernel(T, X, cfg).entries
    assert np.all(np.diag(K) == 1.0) and np.array_equal(K, K.T)
    assert np.abs(K - oracle.kernel_matrix(X, L)).max() <= K_ABS
    assert np.abs(Kx - oracle.cross_kernel(T, X, L)).max() <= K_ABS


@pytest.mark.parametrize("L", [5, 6])
def test_joint_pipeline_and_packed_tiles(L, rng):
    n = 7
    X = _clustered(rng, 130, n, 0.3)
    T = _clustered(rng, 20, n, 0.3)
    cfg = FeatureMapConfig(n, layers=L)
    K, Kx = compute_kernel_matrices(X, T, cfg)  # host pipeline: progress-counted drain
    assert np.array_equal(K.entries, compute_kernel_matrix(X, cfg).entries)
    assert np.array_equal(Kx.entries, compute_cross_kernel(T, X, cfg).entries)
    plan = SweepPlan(n, L)
    planes = dev.gate_build(plan, torch.as_tensor(X, device="cuda"))
    nt = plan.gram_tile_count(130)
    packed = dev.gram(planes, packed=True, tile_begin=0, tile_end=nt)
    Ku = dev.unpack_gram(plan, packed, 130, 0, nt,
                         torch.empty((130, 130), dtype=torch.float64, device="cuda"))
    Ku = Ku.cpu().numpy()
    assert np.array_equal(Ku, K.entries)


def test_contract_batch_and_pair_kernel_deep():
    for name in ("pairs_n24_L5", "pairs_n10_L6", "pairs_n8_L7", "pairs_n6_L8"):
        g = load_golden(name)
        L = int(g["layers"])
        ops = [(g["A"][p], g["B"][q]) for p, q in g["pairs"]]
        amps = np.array([a.real for a in contract_batch(FeatureMapConfig(g["A"].shape[1], L),
                                                        ops)])
        ref = g["amp_re"]
        assert np.all(np.abs(amps - ref) <= AMP_REL * np.abs(ref) + 1e-300), name
    # pair-list kernel == tile sweep bit for bit (same deep_sweep, same reduction order)
    rng = np.random.default_rng(5)
    X = _clustered(rng, 20, 9, 0.3)
    plan = SweepPlan(9, 5)
    planes = dev.gate_build(plan, torch.as_tensor(X, device="cuda"))
    K = dev.gram(planes).cpu().numpy()
    i, j = np.triu_indices(20, 1)
    amp = dev.pair_amplitudes(planes, planes,
                              torch.as_tensor(np.stack([i, j], 1), device="cuda")).cpu().numpy()
    assert np.array_equal(K[i, j], amp * amp)


def test_wide_chain_layers5_vs_oracle(rng):
    """784 qubits at L = 5 (the MNIST width): sampled pairs against the oracle."""
    n = 784
    X = _clustered(rng, 6, n, 0.02)
    pairs = np.array([[0, 1], [2, 3], [4, 5], [1, 4]])
    plan = SweepPlan(n, 5)
    planes = dev.gate_build(plan, torch.as_tensor(X, device="cuda"))
    amp = dev.pair_amplitudes(planes, planes, torch.as_tensor(pairs, device="cuda")).cpu().numpy()
    ref = oracle.amplitudes(X, X, pairs, 5).real
    assert np.all(np.abs(amp - ref) <= AMP_REL * np.abs(ref) + 1e-300)
    assert np.abs(amp ** 2 - ref ** 2).max() <= K_ABS


def test_layers_above_8_refused():
    with pytest.raises(CapacityError, match="bond-65536"):
        compute_kernel_matrix(np.zeros((3, 4)), FeatureMapConfig(4, layers=9))
