"""ctypes binding of libqk.so — the C ABI declared in include/qk.h.

The library is the only compute path of this package.  If it is missing or fails to load,
every entry point raises :class:`NativeLibraryError`; nothing falls back to the CPU.
"""
from __future__ import annotations

import ctypes
import re
import threading
from pathlib import Path

from .errors import CapacityError, DeviceError, NativeLibraryError, RebindError, StructuralError

import os

# QK_LIB_PATH selects an alternative in-tree build (kernel-variant tuning); default libqk.so.
LIB_PATH = Path(os.environ.get("QK_LIB_PATH") or
                Path(__file__).resolve().parent / "_lib" / "libqk.so")
HEADER = Path(__file__).resolve().parent.parent / "include" / "qk.h"

QK_OK, QK_ERR_VALUE, QK_ERR_REBIND, QK_ERR_CAPACITY, QK_ERR_STRUCTURAL, QK_ERR_CUDA = range(6)
QK_PROBABILITY, QK_MAGNITUDE = 0, 1
QK_OUT_DENSE, QK_OUT_PACKED = 0, 1

_c_i32, _c_i64, _c_vp, _c_sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32), ("layers", ctypes.c_int32), ("convention", ctypes.c_int32),
        ("bond", ctypes.c_int32), ("tile_edge", ctypes.c_int32), ("chunk", ctypes.c_int32),
        ("width_padded", ctypes.c_int32), ("stages", ctypes.c_int32),
        ("dp_instr_per_entry", ctypes.c_int64), ("flops_per_entry", ctypes.c_int64),
        ("algorithmic_flops_per_entry", ctypes.c_int64),
        ("reference_cmacs_per_entry", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


_SIGNATURES = {
    "qk_abi_version": (ctypes.c_int, []),
    "qk_last_error": (ctypes.c_char_p, []),
    "qk_set_device": (ctypes.c_int, [_c_i32]),
    "qk_plan_create": (ctypes.c_int, [_c_i32, _c_i32, _c_i32, ctypes.POINTER(_c_vp)]),
    "qk_plan_destroy": (ctypes.c_int, [_c_vp]),
    "qk_plan_get_info": (ctypes.c_int, [_c_vp, ctypes.POINTER(PlanInfo)]),
    "qk_planes_bytes": (_c_sz, [_c_vp, _c_i64]),
    "qk_gram_tile_count": (_c_i64, [_c_vp, _c_i64]),
    "qk_cross_tile_count": (_c_i64, [_c_vp, _c_i64, _c_i64]),
    "qk_gate_build": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "qk_gram_tiles": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_i32, _c_vp]),
    "qk_unpack_gram": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp]),
    "qk_cross_tiles": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp,
                                      _c_i64, _c_i32, _c_vp]),
    "qk_unpack_cross": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp,
                                       _c_i64, _c_vp]),
    "qk_pair_amplitudes": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_i64,
                                          _c_vp, _c_vp]),
    "qk_pair_kernel_values": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp,
                                             _c_i64, _c_vp, _c_vp]),
    "qk_kernel_matrix_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp]),
    "qk_cross_kernel_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp]),
    "qk_dfma_peak": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double), _c_vp]),
    "qk_job_tile_count": (_c_i64, [_c_vp, _c_i64, _c_i64]),
    "qk_job_tiles": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp,
                                    _c_vp, _c_vp]),
    "qk_job_run": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp, _c_vp, _c_vp,
                                  _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "qk_kernel_matrices_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp,
                                               _c_vp]),
    "qk_shared_alloc": (ctypes.c_int, [_c_sz, ctypes.POINTER(_c_vp)]),
    "qk_shared_free": (ctypes.c_int, [_c_vp]),
    "qk_ipc_export": (ctypes.c_int, [_c_vp, ctypes.c_char_p]),
    "qk_ipc_import": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_c_vp)]),
    "qk_ipc_close": (ctypes.c_int, [_c_vp]),
    "qk_device_bus_id": (ctypes.c_int, [ctypes.c_char_p]),
    "qk_can_reach": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32)]),
    "qk_host_register": (ctypes.c_int, [_c_vp, _c_sz]),
    "qk_host_unregister": (ctypes.c_int, [_c_vp]),
    "qk_copy_d2h": (ctypes.c_int, [_c_vp, _c_vp, _c_sz, _c_vp]),
    "qk_copy_h2d": (ctypes.c_int, [_c_vp, _c_vp, _c_sz, _c_vp]),
    "qk_copy_d2d": (ctypes.c_int, [_c_vp, _c_vp, _c_sz, _c_vp]),
    "qk_statevector_bytes": (_c_sz, [ctypes.c_int32]),
    "qk_statevector_amplitude": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _c_vp, _c_vp,
                                                _c_vp, ctypes.POINTER(ctypes.c_double), _c_vp]),
    "qk_statevector_pairs": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _c_vp, _c_i64,
                                            _c_vp, _c_i64, _c_vp, _c_i64, _c_vp]),
}

_lib = None


def declared_symbols() -> list[str]:
    """Function names declared in include/qk.h (the ABI contract)."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*]+\s*\**\s*(qk_\w+)\s*\(", text, re.M)))


def lib() -> ctypes.CDLL:
    """Load libqk.so once; raise NativeLibraryError if it is absent or incomplete."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a); there is no CPU fallback")
    try:
        handle = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (restype, argtypes) in _SIGNATURES.items():
        try:
            fn = getattr(handle, name)
        except AttributeError as exc:
            raise NativeLibraryError(f"{LIB_PATH} does not export {name}") from exc
        fn.restype = restype
        fn.argtypes = argtypes
    if handle.qk_abi_version() != 2:  # QK_ABI_VERSION
        raise NativeLibraryError("libqk ABI version mismatch")
    _lib = handle
    return _lib


_bound = threading.local()


def bind_current_device() -> None:
    """Point libqk's CUDA runtime (linked statically) at the device torch considers current on
    this thread, so multi-GPU processes launch on the device that owns their streams."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return
    if not torch.cuda.is_available():
        return
    dev = torch.cuda.current_device()
    if getattr(_bound, "device", None) != dev:
        check(lib().qk_set_device(dev))
        _bound.device = dev


def last_error() -> str:
    msg = lib().qk_last_error()
    return msg.decode() if msg else ""


def check(status: int, context: str | None = None) -> None:
    """Map a qk_status onto the reference's exception hierarchy (errors.py:8-47)."""
    if status == QK_OK:
        return
    msg = last_error()
    if context:
        msg = f"{context}: {msg}"
    if status == QK_ERR_VALUE:
        raise ValueError(msg)
    if status == QK_ERR_REBIND:
        raise RebindError(msg)
    if status == QK_ERR_CAPACITY:
        raise CapacityError(msg)
    if status == QK_ERR_STRUCTURAL:
        raise StructuralError(msg)
    raise DeviceError(msg)
