"""Dense state-vector ground truth on the GPU (reference: statevector.py:1-70).

The reference's brute-force simulator applies the pair circuit ``compose_kernel_circuit(x_i,
x_j, cfg)`` (circuit.py:150-157) gate by gate to |0...0> and reads the zero amplitude; it is
guarded at 24 qubits (statevector.py:14,43-46).  This module runs the same simulation in libqk
(``qk_statevector_*``, csrc/qk_statevector.cu): every gate in the reference's order on a real
fp64 state (the family's gates are real), so its amplitudes are bit-identical to the
reference's, and device memory moves the guard to ``MAX_WIDTH`` qubits (2^32 doubles = 32 GB).
It shares nothing with the tile sweep's closed form, which makes it the independent check of
the sweep at widths the CPU oracle cannot reach.

``MAX_BATCH_WIDTH``: up to this width ``amplitudes`` simulates many pairs at once (one CTA per
pair, the state in shared memory); wider pairs run one at a time over the whole GPU.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native
from .config import FeatureMapConfig, as_config
from .errors import CapacityError, DeviceError

MAX_WIDTH = 32
MAX_BATCH_WIDTH = 13


def _check_width(cfg: FeatureMapConfig) -> None:
    if cfg.width > MAX_WIDTH:
        raise CapacityError(
            f"state vector for {cfg.width} qubits exceeds the {MAX_WIDTH}-qubit guard")


def _angles(x, width: int) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.ndim != 1 or x.shape[0] != width:
        raise ValueError(f"feature vector has length {x.size}, circuit width is {width}")
    if not np.all(np.isfinite(x)):
        raise ValueError("feature angles must be finite")
    return x


def zero_amplitude(x_i, x_j, cfg: FeatureMapConfig) -> float:
    """<0...0| U(x_i)^dag U(x_j) |0...0> of the pair circuit (reference zero_amplitude of
    compose_kernel_circuit(x_i, x_j, cfg), statevector.py:57-59).  Real: the family's gates
    are real."""
    cfg = as_config(cfg)
    _check_width(cfg)
    xi, xj = _angles(x_i, cfg.width), _angles(x_j, cfg.width)
    if not torch.cuda.is_available():
        raise DeviceError("the state-vector simulator runs on the GPU (no CPU path)")
    lib = _native.lib()
    _native.bind_current_device()
    state = torch.empty(int(lib.qk_statevector_bytes(cfg.width)) // 8, dtype=torch.float64,
                        device="cuda")
    out = ctypes.c_double()
    _native.check(lib.qk_statevector_amplitude(
        cfg.width, cfg.layers, xi.ctypes.data, xj.ctypes.data, state.data_ptr(),
        ctypes.byref(out), torch.cuda.current_stream().cuda_stream))
    return out.value


def kernel_entry_oracle(x_i, x_j, cfg: FeatureMapConfig,
                        convention: str = "probability") -> float:
    """Kernel entry by brute force: |amp| or |amp|^2 (reference statevector.py:62-70)."""
    amp = zero_amplitude(x_i, x_j, cfg)
    mag = abs(amp)
    if convention == "magnitude":
        return mag
    if convention == "probability":
        return mag * mag
    raise ValueError(f"unknown kernel convention {convention!r}")


def amplitudes(A, B, pairs, cfg: FeatureMapConfig) -> np.ndarray:
    """Zero amplitudes of the pair circuits (A[p], B[q]) for 0-based index pairs (p, q)."""
    cfg = as_config(cfg)
    _check_width(cfg)
    A = np.ascontiguousarray(np.asarray(A, dtype=np.float64).reshape(-1, cfg.width))
    B = np.ascontiguousarray(np.asarray(B, dtype=np.float64).reshape(-1, cfg.width))
    P = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))
    if cfg.width > MAX_BATCH_WIDTH:
        return np.array([zero_amplitude(A[p], B[q], cfg) for p, q in P], dtype=np.float64)
    if not torch.cuda.is_available():
        raise DeviceError("the state-vector simulator runs on the GPU (no CPU path)")
    out = np.empty(len(P), dtype=np.float64)
    lib = _native.lib()
    _native.bind_current_device()
    _native.check(lib.qk_statevector_pairs(cfg.width, cfg.layers, A.ctypes.data, len(A),
                                           B.ctypes.data, len(B), P.ctypes.data, len(P),
                                           out.ctypes.data))
    return out
