"""The C ABI (include/qk.h) — loads, exports every declared symbol, validates like the reference
(FeatureMapConfig checks, circuit.py:86-91) without a GPU, and fails loudly (no CPU fallback)
when no CUDA device is present."""
import ctypes

import numpy as np
import pytest

from paper_2405_02630_b200 import (CapacityError, DeviceError, FeatureMapConfig, SweepPlan,
                                   compute_cross_kernel, compute_kernel_matrix)
from paper_2405_02630_b200 import _native


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = _native.declared_symbols()
    assert len(declared) >= 17
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native._SIGNATURES)
    assert lib.qk_abi_version() == 2


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("width,layers,conv,exc,msg", [
    (0, 2, 0, ValueError, "width must be >= 1"),
    (4, 0, 0, ValueError, "layers must be >= 1"),
    (4, 2, 7, ValueError, "unknown kernel convention"),
    (4, 9, 0, CapacityError, "bond-65536"),
])
def test_plan_validation_through_the_abi(width, layers, conv, exc, msg):
    lib = _native.lib()
    h = ctypes.c_void_p()
    status = lib.qk_plan_create(width, layers, conv, ctypes.byref(h))
    assert status != 0 and not h.value
    with pytest.raises(exc, match=msg):
        _native.check(status)


def test_plan_geometry_and_costs():
    p = SweepPlan(784, 2)
    i = p.info
    assert (i["bond"], i["tile_edge"], i["chunk"], i["width_padded"]) == (4, 64, 16, 784)
    assert i["algorithmic_flops_per_entry"] == 34 * 784 + 4
    assert i["dp_instr_per_entry"] == 16 * 784 + 3
    assert i["reference_cmacs_per_entry"] == 1056 * 784 - 3912  # reference planner (probe1)
    assert p.gram_tile_count(10000) == 157 * 158 // 2
    assert p.cross_tile_count(2000, 10000) == 32 * 157
    assert p.planes_bytes(10000) == 157 * 784 * 64 * 16
    q = SweepPlan(17, 2)
    assert q.info["width_padded"] == 32  # 15 identity qubits in front
    assert SweepPlan(5, 1).info["bond"] == 1
    assert SweepPlan(5, 3).info["bond"] == 16
    for L in (5, 6, 7, 8):  # factored level passes
        M, D = L - 1, 2 ** (L - 1)
        E = D * D
        info = SweepPlan(5, L).info
        assert info["bond"] == E
        assert info["algorithmic_flops_per_entry"] == (6 * M * E + E + 6) * 5 + E
        if L == 5:  # rotated blocked form over D / 2 threads per pair
            assert info["dp_instr_per_entry"] == (4 * (M - 1) * E + 2 * E + 9 * D) * 5 + E // 2 + D // 2
        elif L <= 7:  # register-resident: mask folded into level 0, per-thread coefficients
            assert info["dp_instr_per_entry"] == (4 * M * E + 8 * D) * 5 + 2 * E
        else:
            assert info["dp_instr_per_entry"] == (4 * M * E + E + 4) * 5 + E
    assert SweepPlan(5, 3).info["dp_instr_per_entry"] == 112 * 5 + 9  # rotated blocked bond 16
    assert SweepPlan(5, 4).info["dp_instr_per_entry"] == 656 * 5 + 33  # rotated blocked bond 64
    assert SweepPlan(5, 4).info["bond"] == 64


def test_null_and_range_arguments_are_rejected():
    lib = _native.lib()
    p = SweepPlan(8, 2)
    assert lib.qk_gram_tiles(p.handle, None, 100, 0, 10**6, None, 0, None) == _native.QK_ERR_VALUE
    assert "tile range" in _native.last_error()
    assert lib.qk_gram_tiles(None, None, 1, 0, 1, None, 0, None) == _native.QK_ERR_VALUE
    assert lib.qk_cross_tiles(p.handle, None, 10, None, 10, 0, 1, None, 5, 0, None) == \
        _native.QK_ERR_VALUE  # ld_out < n_cols


def _has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except ImportError:  # pragma: no cover
        return False


@pytest.mark.skipif(_has_cuda(), reason="checks the no-device failure mode")
def test_compute_fails_loudly_without_a_device():
    X = np.random.default_rng(0).uniform(0, 1, (5, 4))
    with pytest.raises(DeviceError):
        compute_kernel_matrix(X, FeatureMapConfig(4))
    with pytest.raises(DeviceError):
        compute_cross_kernel(X, X, FeatureMapConfig(4))


def test_missing_library_is_a_hard_error(tmp_path, monkeypatch):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "absent.so")
    from paper_2405_02630_b200 import NativeLibraryError

    with pytest.raises(NativeLibraryError, match="no CPU fallback"):
        _native.lib()


def test_statevector_entry_points_validate_before_touching_the_device():
    lib = _native.lib()
    assert lib.qk_statevector_bytes(30) == 8 << 30 and lib.qk_statevector_bytes(0) == 0
    A = np.zeros((2, 4))
    out = np.empty(1)
    bad = np.array([[0, 2]], dtype=np.int64)
    assert lib.qk_statevector_pairs(4, 2, A.ctypes.data, 2, A.ctypes.data, 2, bad.ctypes.data,
                                    1, out.ctypes.data) == _native.QK_ERR_VALUE
    assert "indexes outside" in _native.last_error()
    assert lib.qk_statevector_pairs(14, 2, A.ctypes.data, 0, A.ctypes.data, 0, bad.ctypes.data,
                                    1, out.ctypes.data) == _native.QK_ERR_CAPACITY
    A[1, 2] = np.inf
    ok = np.array([[0, 1]], dtype=np.int64)
    assert lib.qk_statevector_pairs(4, 2, A.ctypes.data, 2, A.ctypes.data, 2, ok.ctypes.data,
                                    1, out.ctypes.data) == _native.QK_ERR_REBIND
