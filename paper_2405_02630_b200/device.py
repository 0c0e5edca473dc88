"""Device-resident engine calls: torch CUDA tensors in, torch CUDA tensors out.

Thin stream-ordered wrappers over the C ABI (include/qk.h).  torch supplies device memory,
the current stream and the process group; every FLOP runs in libqk's sm_100a kernels.
Non-CUDA inputs are rejected — there is no CPU path.
"""
from __future__ import annotations

import torch

from . import _native
from .errors import DeviceError, RebindError
from .planner import SweepPlan


def _stream() -> int:
    _native.bind_current_device()
    return torch.cuda.current_stream().cuda_stream


def _require(t: torch.Tensor, name: str, dtype=None) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DeviceError(f"{name} must be a CUDA tensor (the engine has no CPU path)")
    _on_current(t, name)
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _on_current(t: torch.Tensor, name: str) -> None:
    """Launches go to torch's current stream on the current device: a tensor on another GPU
    would be read by the wrong device's kernels, so it is refused (torch.cuda.set_device or
    ``with torch.cuda.device(...)`` selects the device)."""
    cur = torch.cuda.current_device()
    if t.device.index != cur:
        raise DeviceError(f"{name} is on {t.device} but the current device is cuda:{cur}")


def angles_to_device(x, device=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(device=device or x.device, dtype=torch.float64)
    else:
        t = torch.as_tensor(x, dtype=torch.float64).to(device or "cuda")
    return t.contiguous()


class Planes:
    """Per-sample rotation planes in HBM (output of the gate-build kernel)."""

    def __init__(self, plan: SweepPlan, n_samples: int, buf: torch.Tensor, bad: torch.Tensor):
        self.plan = plan
        self.n = int(n_samples)
        self.buf = buf
        self.bad = bad

    def ptr(self) -> int:
        return self.buf.data_ptr()

    def bad_sample(self) -> int | None:
        """Smallest sample index holding a non-finite angle, or None (synchronises)."""
        v = int(self.bad.item())
        return None if v == -1 else v


def gate_build(plan: SweepPlan, angles: torch.Tensor, out: torch.Tensor | None = None,
               bad: torch.Tensor | None = None) -> Planes:
    """angles [N, width] fp64 (CUDA) -> planes (network.py:283-302 per sample).

    ``bad``: optional one-element int64 CUDA tensor already holding -1, the non-finite
    sentinel to use (callers that build several plane sets reset theirs in one fill)."""
    _require(angles, "angles", torch.float64)
    if angles.dim() != 2 or angles.shape[1] != plan.width:
        raise RebindError(f"feature vectors of length {angles.shape[-1]} do not match width "
                          f"{plan.width}")
    n = angles.shape[0]
    nbytes = plan.planes_bytes(n)
    if out is None or out.numel() < nbytes:
        out = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=angles.device)
    if bad is None:
        bad = torch.full((1,), -1, dtype=torch.int64, device=angles.device)
    _native.check(_native.lib().qk_gate_build(plan.handle, angles.data_ptr(), n, plan.width,
                                              out.data_ptr(), bad.data_ptr(), _stream()))
    return Planes(plan, n, out, bad)


def gram(planes: Planes, out: torch.Tensor | None = None, tile_begin: int = 0,
         tile_end: int | None = None, packed: bool = False) -> torch.Tensor:
    """Train Gram over upper-triangle tiles [tile_begin, tile_end).

    Dense: writes an N x N fp64 matrix (strict upper computed, mirrored, unit diagonal).
    Packed: returns the tile-major buffer of the range (edge^2 doubles per tile)."""
    plan, n = planes.plan, planes.n
    _on_current(planes.buf, "planes")
    nt = plan.gram_tile_count(n)
    tile_end = nt if tile_end is None else tile_end
    edge = plan.tile_edge
    if out is None:
        shape = ((tile_end - tile_begin) * edge * edge,) if packed else (n, n)
        out = torch.empty(shape, dtype=torch.float64, device=planes.buf.device)
    _require(out, "out", torch.float64)
    mode = _native.QK_OUT_PACKED if packed else _native.QK_OUT_DENSE
    _native.check(_native.lib().qk_gram_tiles(plan.handle, planes.ptr(), n, tile_begin,
                                              tile_end, out.data_ptr(), mode, _stream()))
    return out


def cross(rows: Planes, cols: Planes, out: torch.Tensor | None = None, tile_begin: int = 0,
          tile_end: int | None = None, packed: bool = False) -> torch.Tensor:
    """Test-versus-train block K[r][c] over rectangle tiles [tile_begin, tile_end)."""
    plan = rows.plan
    _on_current(rows.buf, "row planes")
    _on_current(cols.buf, "column planes")
    nt = plan.cross_tile_count(rows.n, cols.n)
    tile_end = nt if tile_end is None else tile_end
    edge = plan.tile_edge
    if out is None:
        shape = ((tile_end - tile_begin) * edge * edge,) if packed else (rows.n, cols.n)
        out = torch.empty(shape, dtype=torch.float64, device=rows.buf.device)
    _require(out, "out", torch.float64)
    mode = _native.QK_OUT_PACKED if packed else _native.QK_OUT_DENSE
    ld = cols.n if not packed else 0
    _native.check(_native.lib().qk_cross_tiles(plan.handle, rows.ptr(), rows.n, cols.ptr(),
                                               cols.n, tile_begin, tile_end, out.data_ptr(), ld,
                                               mode, _stream()))
    return out


def gram_into(planes: Planes, out_ptr: int, tile_begin: int, tile_end: int) -> None:
    """Dense Gram tiles [tile_begin, tile_end) stored at a raw device address (e.g. a peer
    rank's matrix imported over CUDA IPC; row-major N x N)."""
    _on_current(planes.buf, "planes")
    _native.check(_native.lib().qk_gram_tiles(planes.plan.handle, planes.ptr(), planes.n,
                                              tile_begin, tile_end, out_ptr,
                                              _native.QK_OUT_DENSE, _stream()))


def cross_into(rows: Planes, cols: Planes, out_ptr: int, tile_begin: int, tile_end: int) -> None:
    """Dense cross tiles stored at a raw device address (row-major n_rows x n_cols)."""
    _on_current(rows.buf, "row planes")
    _on_current(cols.buf, "column planes")
    _native.check(_native.lib().qk_cross_tiles(rows.plan.handle, rows.ptr(), rows.n, cols.ptr(),
                                               cols.n, tile_begin, tile_end, out_ptr, cols.n,
                                               _native.QK_OUT_DENSE, _stream()))


def job_into(train: Planes, test: Planes | None, K_train_ptr: int, K_cross_ptr: int,
             tile_begin: int = 0, tile_end: int | None = None) -> None:
    """Train Gram + test x train block as one tile list, one persistent launch, dense outputs
    at raw device addresses (row-major N_train x N_train and N_test x N_train)."""
    plan = train.plan
    _on_current(train.buf, "train planes")
    if test is not None:
        _on_current(test.buf, "test planes")
    n_test = test.n if test is not None else 0
    nt = int(_native.lib().qk_job_tile_count(plan.handle, train.n, n_test))
    tile_end = nt if tile_end is None else tile_end
    _native.check(_native.lib().qk_job_tiles(plan.handle, train.ptr(), train.n,
                                             test.ptr() if test is not None else None, n_test,
                                             tile_begin, tile_end, K_train_ptr,
                                             K_cross_ptr if n_test else None, _stream()))


def unpack_gram(plan: SweepPlan, packed: torch.Tensor, n: int, tile_begin: int, tile_end: int,
                K: torch.Tensor) -> torch.Tensor:
    _require(packed, "packed", torch.float64)
    _require(K, "K", torch.float64)
    _native.check(_native.lib().qk_unpack_gram(plan.handle, packed.data_ptr(), n, tile_begin,
                                               tile_end, K.data_ptr(), _stream()))
    return K


def unpack_cross(plan: SweepPlan, packed: torch.Tensor, n_rows: int, n_cols: int,
                 tile_begin: int, tile_end: int, K: torch.Tensor) -> torch.Tensor:
    _require(packed, "packed", torch.float64)
    _require(K, "K", torch.float64)
    _native.check(_native.lib().qk_unpack_cross(plan.handle, packed.data_ptr(), n_rows, n_cols,
                                                tile_begin, tile_end, K.data_ptr(), n_cols,
                                                _stream()))
    return K


def pair_amplitudes(a: Planes, b: Planes, pairs: torch.Tensor) -> torch.Tensor:
    """Signed real amplitudes for explicit (p, q) index pairs, input order (engine.py:132)."""
    _require(pairs, "pairs", torch.int64)
    _on_current(a.buf, "planes")
    _on_current(b.buf, "planes")
    pairs = pairs.reshape(-1, 2).contiguous()
    out = torch.empty(pairs.shape[0], dtype=torch.float64, device=a.buf.device)
    _native.check(_native.lib().qk_pair_amplitudes(a.plan.handle, a.ptr(), a.n, b.ptr(), b.n,
                                                   pairs.data_ptr(), pairs.shape[0],
                                                   out.data_ptr(), _stream()))
    return out


def pair_kernel_values(a: Planes, b: Planes, pairs: torch.Tensor) -> torch.Tensor:
    """Kernel values K(a_p, b_q) under the plan's convention for explicit (p, q) pairs, input
    order, computed in the pair kernel's epilogue (the SPEC's shard partial)."""
    _require(pairs, "pairs", torch.int64)
    _on_current(a.buf, "planes")
    _on_current(b.buf, "planes")
    pairs = pairs.reshape(-1, 2).contiguous()
    out = torch.empty(pairs.shape[0], dtype=torch.float64, device=a.buf.device)
    _native.check(_native.lib().qk_pair_kernel_values(a.plan.handle, a.ptr(), a.n, b.ptr(), b.n,
                                                      pairs.data_ptr(), pairs.shape[0],
                                                      out.data_ptr(), _stream()))
    return out


def dfma_peak_flops() -> float:
    """Measured FP64 FMA issue rate of the current device (FLOP/s, FMA = 2)."""
    import ctypes

    v = ctypes.c_double(0.0)
    _native.check(_native.lib().qk_dfma_peak(ctypes.byref(v), _stream()))
    torch.cuda.synchronize()
    return float(v.value)
