"""In-kernel plane build of the host pipelines (opt-in, pinned angle buffers): the H2D goes up in
chunks of plane blocks on its own stream and the persistent sweep builds each plane block
itself as soon as its angles have landed.  It must reproduce the gate-build path (pageable
inputs: upload, gate-build kernel, sweep) bit for bit, for every shape of the chunking."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2405_02630_b200 import (FeatureMapConfig, RebindError, compute_cross_kernel,
                                   compute_kernel_matrices, compute_kernel_matrix)

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fused_build_on():
    """The in-kernel plane build is opt-in (QK_FUSED_BUILD=1, read on every call)."""
    old = os.environ.get("QK_FUSED_BUILD")
    os.environ["QK_FUSED_BUILD"] = "1"
    yield
    if old is None:
        del os.environ["QK_FUSED_BUILD"]
    else:
        os.environ["QK_FUSED_BUILD"] = old


def _pinned(a: np.ndarray) -> np.ndarray:
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    out = t.numpy()
    out[...] = a
    return out


@pytest.mark.parametrize("L,n,n_train,n_test", [
    (2, 40, 1300, 150), (2, 17, 600, 7), (2, 784, 700, 65), (1, 33, 1025, 64),
    (2, 5, 64, 0), (2, 9, 65, 1), (2, 3, 5, 3), (2, 20, 1, 4), (1, 8, 2, 0)])
def test_pinned_inputs_match_pageable_bit_for_bit(L, n, n_train, n_test, rng):
    X = rng.uniform(0, np.pi, n) + rng.normal(0, 0.4 / np.sqrt(n), (n_train, n))
    T = rng.uniform(0, np.pi, n) + rng.normal(0, 0.4 / np.sqrt(n), (n_test, n))
    cfg = FeatureMapConfig(n, layers=L)
    K, Kx = compute_kernel_matrices(X, T, cfg)                      # pageable: gate-build path
    Kp, Kxp = compute_kernel_matrices(_pinned(X), _pinned(T), cfg)  # pinned: in-kernel build
    assert np.array_equal(K.entries, Kp.entries)
    assert np.array_equal(Kx.entries, Kxp.entries)
    if n_train >= 2:
        assert np.array_equal(compute_kernel_matrix(_pinned(X), cfg).entries, K.entries)
    if n_test:
        assert np.array_equal(compute_cross_kernel(_pinned(T), _pinned(X), cfg).entries,
                              Kx.entries)
    if n_train * n <= 40000:
        assert np.abs(Kp.entries - oracle.kernel_matrix(X, L)).max() <= 1e-12


def test_repeated_calls_and_growing_sizes(rng):
    """Arrival marks carry a per-call epoch: repeated and growing calls reuse them safely."""
    cfg = FeatureMapConfig(12)
    for N in (70, 70, 900, 130, 2000):
        X = _pinned(rng.uniform(0, 1, (N, 12)))
        T = _pinned(rng.uniform(0, 1, (33, 12)))
        K, Kx = compute_kernel_matrices(X, T, cfg)
        K2, Kx2 = compute_kernel_matrices(np.array(X), np.array(T), cfg)
        assert np.array_equal(K.entries, K2.entries) and np.array_equal(Kx.entries, Kx2.entries)


def test_non_finite_pinned_input_names_the_operand_set():
    cfg = FeatureMapConfig(4)
    X = _pinned(np.zeros((6, 4)))
    X[3, 2] = np.nan
    with pytest.raises(RebindError, match="operand set 2: feature angles must be finite"):
        compute_kernel_matrix(X, cfg)
    T = _pinned(np.zeros((2, 4)))
    T[1, 0] = np.inf
    with pytest.raises(RebindError, match="operand set 6: feature angles must be finite"):
        compute_cross_kernel(T, _pinned(np.zeros((6, 4))), cfg)
    # the pipeline is healthy afterwards
    Y = _pinned(np.random.default_rng(1).uniform(0, 1, (9, 4)))
    assert np.array_equal(compute_kernel_matrix(Y, cfg).entries,
                          compute_kernel_matrix(np.array(Y), cfg).entries)
