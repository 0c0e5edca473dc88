"""Kernel container / shard partial / CSV round trips — host-only."""
import numpy as np
import pytest

from paper_2405_02630_b200 import DataFormatError, KernelMatrix, ShardMergeError, enumerate_pairs
from paper_2405_02630_b200.container import (enumeration_pairs, export_csv, load_kernel,
                                             merge_partials, save_kernel, save_partial,
                                             shard_pair_range)


def _gram(n, rng):
    U = np.triu(rng.uniform(0, 1, (n, n)), 1)
    return U + U.T + np.eye(n)


def test_enumeration_pairs_matches_enumerate_pairs():
    for n in (2, 3, 7, 64, 65):
        ref = np.array(enumerate_pairs(n, n, True)) - 1
        assert np.array_equal(enumeration_pairs(n, n, True, 0, len(ref)), ref)
        lo, hi = len(ref) // 3, 2 * len(ref) // 3
        assert np.array_equal(enumeration_pairs(n, n, True, lo, hi), ref[lo:hi])
    ref = np.array(enumerate_pairs(4, 5, False)) - 1
    assert np.array_equal(enumeration_pairs(4, 5, False, 3, 17), ref[3:17])


def test_container_round_trip_and_csv(tmp_path, rng):
    K = _gram(9, rng)
    km = KernelMatrix(9, 9, K, "probability", {"kind": "gram", "qubits": 8, "layers": 2,
                                               "config_hash": "abc", "dataset": "syn"})
    save_kernel(tmp_path / "k.qkk", km)
    back = load_kernel(tmp_path / "k.qkk")
    assert np.array_equal(back.entries, K) and back.metadata["qubits"] == 8
    export_csv(tmp_path / "k.csv", km)
    assert np.array_equal(np.loadtxt(tmp_path / "k.csv", delimiter=","), K)
    (tmp_path / "bad.qkk").write_bytes(b"NOTAKERNEL")
    with pytest.raises(DataFormatError, match="magic"):
        load_kernel(tmp_path / "bad.qkk")
    raw = (tmp_path / "k.qkk").read_bytes()
    (tmp_path / "trunc.qkk").write_bytes(raw[:-8])
    with pytest.raises(DataFormatError, match="truncated"):
        load_kernel(tmp_path / "trunc.qkk")


def test_shard_run_then_merge_is_byte_identical(tmp_path, rng):
    n = 11
    K = _gram(n, rng)
    meta = {"config_hash": "h", "qubits": 3, "layers": 2, "dataset": None, "kind": "gram"}
    save_kernel(tmp_path / "full.qkk", KernelMatrix(n, n, K, "probability", meta))
    paths = []
    for k in range(3):
        lo, hi = shard_pair_range(n, n, True, k, 3)
        ij = enumeration_pairs(n, n, True, lo, hi)
        save_partial(tmp_path / f"p{k}.qkk", K[ij[:, 0], ij[:, 1]], (lo, hi), n, n, True,
                     metadata=meta)
        paths.append(tmp_path / f"p{k}.qkk")
    merged = merge_partials(paths)
    save_kernel(tmp_path / "merged.qkk", merged)
    assert (tmp_path / "merged.qkk").read_bytes() == (tmp_path / "full.qkk").read_bytes()
    with pytest.raises(ShardMergeError, match="gap"):
        merge_partials(paths[:2])
