"""Host-side logic of the SPEC kernel_pipeline boundary: pair enumeration,
symmetrisation, sharding and merge, KernelMatrix, configs and error hierarchy."""
import numpy as np
import pytest

from paper_2405_02630_b200 import (FeatureMapConfig, KernelMatrix, RebindError, ShardMergeError,
                                   StructuralError, TnkernelError, enumerate_pairs, shard_merge,
                                   shard_range, symmetrize)
from paper_2405_02630_b200 import errors as E
from paper_2405_02630_b200.config import as_config


def test_enumerate_pairs_spec_examples():
    assert enumerate_pairs(3, 3, True) == [(1, 2), (1, 3), (2, 3)]
    assert len(enumerate_pairs(1000, 1000, True)) == 499_500
    assert enumerate_pairs(2, 3, False) == [(1, 1), (1, 2), (1, 3), (2, 1), (2, 2), (2, 3)]
    with pytest.raises(ValueError):
        enumerate_pairs(0, 3, True)


def test_symmetrize_spec_examples():
    U = np.zeros((3, 3))
    U[0, 1] = 0.5
    K = symmetrize(KernelMatrix(3, 3, U)).entries
    assert K[0, 1] == K[1, 0] == 0.5 and np.all(np.diag(K) == 1.0)
    assert np.array_equal(symmetrize(KernelMatrix(3, 3, np.zeros((3, 3)))).entries, np.eye(3))
    with pytest.raises(StructuralError, match="precondition"):
        symmetrize(KernelMatrix(3, 3, K))  # already symmetrised
    with pytest.raises(StructuralError):
        symmetrize(KernelMatrix(2, 3, np.zeros((2, 3))))


def _values(pairs):
    return [0.01 * i + 0.001 * j for i, j in pairs]


def test_shard_merge_is_bit_exact_and_checks_coverage():
    pairs = enumerate_pairs(4, 4, True)
    full = shard_merge([(pairs, _values(pairs))], n_a=4)
    parts = []
    for k in range(2):
        lo, hi = shard_range(len(pairs), k, 2)
        parts.append((pairs[lo:hi], _values(pairs[lo:hi])))
    assert np.array_equal(shard_merge(parts, n_a=4).entries, full.entries)
    assert np.array_equal(full.entries, full.entries.T)
    with pytest.raises(ShardMergeError, match="gap at pair \\(1, 3\\)"):
        shard_merge([(pairs[:1] + pairs[2:], _values(pairs[:1] + pairs[2:]))], n_a=4)
    with pytest.raises(ShardMergeError, match="overlap"):
        shard_merge([(pairs, _values(pairs)), (pairs[:1], [0.3])], n_a=4)
    cross = enumerate_pairs(2, 3, False)
    km = shard_merge([(cross, _values(cross))], n_a=2, n_b=3, symmetric=False)
    assert km.entries.shape == (2, 3) and km.entries[1, 2] == pytest.approx(0.023)


def test_shard_range_contiguous_ceil():
    assert [shard_range(10, k, 3) for k in range(3)] == [(0, 4), (4, 8), (8, 10)]
    assert shard_range(0, 0, 4) == (0, 0)
    with pytest.raises(ValueError):
        shard_range(10, 3, 3)


def test_feature_map_config_mirrors_reference():
    assert FeatureMapConfig(8).layers == 2
    for kw, msg in [({"width": 0}, "width must be >= 1"), ({"width": 2, "layers": 0},
                    "layers must be >= 1"), ({"width": 2, "entanglement": "full"},
                    "unsupported entanglement"), ({"width": 2, "embedding": "zz"},
                    "unsupported embedding")]:
        with pytest.raises(ValueError, match=msg):
            FeatureMapConfig(**kw)

    class RefLike:  # duck-typed reference FeatureMapConfig / TensorNetwork
        width, layers, entanglement, embedding = 5, 3, "linear", "ry_angle"

    assert as_config(RefLike()) == FeatureMapConfig(5, 3)
    assert FeatureMapConfig(8).config_hash() != FeatureMapConfig(8, 3).config_hash()


def test_kernel_matrix_checks_shape_and_convention():
    with pytest.raises(StructuralError):
        KernelMatrix(2, 2, np.zeros((2, 3)))
    with pytest.raises(ValueError):
        KernelMatrix(1, 1, np.zeros((1, 1)), convention="amplitude")


def test_error_hierarchy_matches_reference():
    assert issubclass(RebindError, StructuralError)
    assert issubclass(E.ShardMergeError, StructuralError)
    for cls in (E.ConfigError, E.DataFormatError, E.CapacityError, E.StructuralError,
                E.SliceInfeasibleError, E.ConvergenceError, E.NativeLibraryError):
        assert issubclass(cls, TnkernelError)
    err = E.ConvergenceError("cap", alphas=[1], bias=0.5, kkt_residual=1e-3)
    assert err.bias == 0.5


def test_host_result_mappings_are_recycled_only_after_every_view_is_gone():
    from paper_2405_02630_b200.kernel_pipeline import _host_cache, host_empty

    shape = (9000, 1000)  # 72 MB: above the mapping threshold
    before = _host_cache.bytes
    a = host_empty(shape)
    a[:] = 2.0
    addr = a.ctypes.data
    view = a[10:20, 5]
    del a
    assert _host_cache.bytes == before  # a view still holds the mapping
    assert float(view[0]) == 2.0
    del view
    assert _host_cache.bytes == before + 72_000_000
    b = host_empty(shape)  # same size: the cached mapping, already faulted in
    assert b.ctypes.data == addr and b.shape == shape and b.flags.c_contiguous
    c = host_empty(shape)  # cache empty for this size again: a new mapping
    assert c.ctypes.data != addr
    small = host_empty((10, 10))  # small results are plain numpy arrays
    assert small.base is None or not hasattr(small.base, "__buffer__")
    del b, c


def test_result_mappings_page_locked_once_and_unlocked_before_unmap(monkeypatch):
    """Host logic of the page-locked result cache (no GPU: libqk's register entry points are
    replaced by counters): a mapping is registered once when created, handed back registered
    when recycled, and unregistered before it is unmapped (cache overflow, drop_all)."""
    from paper_2405_02630_b200 import kernel_pipeline as kp

    calls = []

    class FakeLib:
        def qk_host_register(self, ptr, n):
            calls.append(("reg", ptr.value, n.value))
            return 0

        def qk_host_unregister(self, ptr):
            calls.append(("unreg", ptr.value))
            return 0

    monkeypatch.setattr(kp._native, "lib", lambda: FakeLib())
    monkeypatch.setattr(kp._native, "bind_current_device", lambda: None)
    cache = kp._HostCache()
    cache.pin, cache.limit = True, 3 << 20
    a = cache.get(2 << 20)
    assert len(calls) == 1 and calls[0][0] == "reg" and calls[0][2] == 2 << 20
    addr = calls[0][1]
    assert cache.pinned == {id(a): addr}
    cache.put(a)  # fits the 3 MB limit: kept, still registered
    assert cache.get(2 << 20) is a and len(calls) == 1
    b = cache.get(2 << 20)  # a new mapping: registered
    assert len(calls) == 2 and calls[1][0] == "reg"
    cache.put(a)
    cache.put(b)  # over the limit: unregistered, then unmapped
    assert calls[2] == ("unreg", calls[1][1]) and b.closed and id(b) not in cache.pinned
    cache.drop_all()  # the cached one too
    assert calls[3] == ("unreg", addr) and a.closed and cache.pinned == {} and cache.bytes == 0
