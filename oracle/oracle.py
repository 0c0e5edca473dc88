"""oracle — TEST INFRASTRUCTURE ONLY: the CPU checker for the QSVM kernel hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
the ``--impl reference`` arm) may import this module, and only as the checker / the timed
CPU baseline — never as a compute path of the product package.

Contents
  * ``amplitudes`` / ``kernel_matrix`` / ``cross_kernel`` — ctypes front end of
    ``qk_oracle.c``: a complex128 restatement of the reference's tensor-network contraction
    of the kernel circuit (reference: pkg/src/tnkernel/circuit.py:121-157,
    network.py:125-302, engine.py:52-166), multi-threaded over pairs like contract_batch's
    worker pool (engine.py:159-166).  Pair enumeration and symmetrisation follow SPEC.md:389-415.
  * ``statevector_amplitude`` — the brute-force dense simulator of statevector.py:17-59
    restated in numpy (n <= 20), an independent third check for small widths.

Pinning: tests/test_oracle.py checks both against tests/golden/*.npz, which
tests/golden/make_golden.py produced by running the reference package itself.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libqk_oracle.so"


def build(force: bool = False) -> Path:
    """Compile qk_oracle.c with gcc into oracle/_build/ (idempotent)."""
    src = _HERE / "qk_oracle.c"
    if _SO.exists() and not force and _SO.stat().st_mtime >= src.stat().st_mtime:
        return _SO
    _SO.parent.mkdir(parents=True, exist_ok=True)
    # -fcx-limited-range: complex products by the plain (ac - bd, ad + bc) formula, as numpy's
    # einsum computes them, without libgcc's __muldc3 call (identical values for finite
    # operands); -ffp-contract=off keeps every product and sum separately rounded (no FMA), so
    # the vector build is bit-identical to the scalar -O2 one and ~1.9x faster.
    cmd = ["gcc", "-O3", "-fcx-limited-range", "-ffp-contract=off", "-mavx2", "-mfma", "-fPIC",
           "-shared", "-std=c11", "-o", str(_SO), str(src), "-lm", "-lpthread"]
    subprocess.run(cmd, check=True)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_SO))
        lib.qko_amplitudes.restype = ctypes.c_int
        lib.qko_amplitudes.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
        ]
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def amplitudes(A, B, pairs, layers: int = 2, threads: int | None = None) -> np.ndarray:
    """Complex amplitudes <0|U(A[p])^dag U(B[q])|0> for pairs (p, q), in input order."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[1]:
        raise ValueError("A and B must be 2-D with equal widths")
    n = A.shape[1]
    P = pairs.shape[0]
    re = np.empty(P, dtype=np.float64)
    im = np.empty(P, dtype=np.float64)
    if P == 0:
        return re.astype(np.complex128)
    if pairs.min() < 0 or pairs[:, 0].max() >= A.shape[0] or pairs[:, 1].max() >= B.shape[0]:
        raise IndexError("pair index out of range")
    rc = _load().qko_amplitudes(n, int(layers), A.ctypes.data, B.ctypes.data, pairs.ctypes.data,
                                P, re.ctypes.data, im.ctypes.data,
                                int(threads or default_threads()))
    if rc != 0:
        raise ValueError(f"oracle rejected (n={n}, layers={layers})")
    return re + 1j * im


def _value(amp: np.ndarray, convention: str) -> np.ndarray:
    mag = np.abs(amp)
    if convention == "magnitude":
        return mag
    if convention == "probability":
        return mag * mag
    raise ValueError(f"unknown kernel convention {convention!r}")


def upper_pairs(n: int) -> np.ndarray:
    """Strict upper triangle, row-major, 0-based."""
    i, j = np.triu_indices(n, k=1)
    return np.stack([i, j], axis=1).astype(np.int64)


def kernel_matrix(X, layers: int = 2, convention: str = "probability",
                  threads: int | None = None) -> np.ndarray:
    """Train Gram: contract the strict upper triangle, then K + K^T + I."""
    X = np.asarray(X, dtype=np.float64)
    N = X.shape[0]
    pairs = upper_pairs(N)
    vals = _value(amplitudes(X, X, pairs, layers, threads), convention)
    K = np.zeros((N, N))
    K[pairs[:, 0], pairs[:, 1]] = vals
    return K + K.T + np.eye(N)


def cross_kernel(test, train, layers: int = 2, convention: str = "probability",
                 threads: int | None = None) -> np.ndarray:
    """Full rectangle, rows = test, diagonal computed."""
    test = np.asarray(test, dtype=np.float64)
    train = np.asarray(train, dtype=np.float64)
    r, c = np.meshgrid(np.arange(test.shape[0]), np.arange(train.shape[0]), indexing="ij")
    pairs = np.stack([r.ravel(), c.ravel()], axis=1)
    vals = _value(amplitudes(test, train, pairs, layers, threads), convention)
    return vals.reshape(test.shape[0], train.shape[0])


# ---------------------------------------------------------------------------------------
# Dense state-vector restatement (statevector.py:17-59): little-endian, qubit q at stride 2^q.
# ---------------------------------------------------------------------------------------
def _ry(theta: float) -> np.ndarray:
    c, s = np.cos(theta / 2), np.sin(theta / 2)
    return np.array([[c, -s], [s, c]], dtype=complex)


def _apply_single(state, m, q):
    view = state.reshape(-1, 2, 1 << q)
    a = view[:, 0, :].copy()
    b = view[:, 1, :].copy()
    view[:, 0, :] = m[0, 0] * a + m[0, 1] * b
    view[:, 1, :] = m[1, 0] * a + m[1, 1] * b


def _apply_cnot(state, c, t):
    idx = np.arange(state.size)
    sel = ((idx >> c) & 1) == 1
    src = idx[sel]
    dst = src ^ (1 << t)
    tmp = state[src].copy()
    state[dst] = tmp


def statevector_amplitude(xi, xj, layers: int = 2) -> complex:
    """<0|U(x_i)^dag U(x_j)|0> by dense simulation of the composed circuit (n <= 20)."""
    xi = np.asarray(xi, dtype=float)
    xj = np.asarray(xj, dtype=float)
    n = xi.size
    if n > 20:
        raise ValueError("statevector oracle limited to 20 qubits")
    state = np.zeros(1 << n, dtype=complex)
    state[0] = 1.0
    for _ in range(layers):  # U(x_j)
        for q in range(n):
            _apply_single(state, _ry(xj[q]), q)
        for q in range(n - 1):
            _apply_cnot(state, q, q + 1)
    for _ in range(layers):  # U(x_i)^dag: reversed gates, negated angles
        for q in reversed(range(n - 1)):
            _apply_cnot(state, q, q + 1)
        for q in reversed(range(n)):
            _apply_single(state, _ry(-xi[q]), q)
    return complex(state[0])
