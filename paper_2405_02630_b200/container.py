"""Kernel container files, shard partials and CSV export (resumable pipelines).

Format (little-endian):

    8 B   magic  b"QKKMAT01"
    4 B   u32    header length H
    H B   JSON   {"rows", "cols", "convention", "kind": "gram"|"cross"|"partial",
                  "config_hash", "qubits", "layers", "dataset", "symmetric",
                  "pair_range": [lo, hi]  (partials only; 0-based, half-open, of the
                                           row-major enumeration of SPEC.md:389-397)}
    pad   zero bytes to an 8-byte boundary
    8 B * count   float64 payload: rows*cols row-major (full) or hi-lo pair values (partial)

The header is serialised with sorted keys so identical matrices produce identical files
(shard-run-then-merge equals the unsharded file byte for byte).  CSV export
writes 17 significant digits, which round-trips float64 exactly.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .errors import DataFormatError, ShardMergeError
from .kernel_pipeline import KernelMatrix, shard_merge, shard_range

MAGIC = b"QKKMAT01"


def _header(km_rows, km_cols, convention, meta: dict, kind: str, symmetric: bool,
            pair_range=None) -> dict:
    h = {"rows": int(km_rows), "cols": int(km_cols), "convention": convention, "kind": kind,
         "config_hash": meta.get("config_hash"), "qubits": meta.get("qubits"),
         "layers": meta.get("layers"), "dataset": meta.get("dataset"),
         "symmetric": bool(symmetric)}
    if pair_range is not None:
        h["pair_range"] = [int(pair_range[0]), int(pair_range[1])]
    return h


def _write(path, header: dict, payload: np.ndarray) -> None:
    hb = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    pad = (-(len(MAGIC) + 4 + len(hb))) % 8
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(hb)))
        f.write(hb)
        f.write(b"\0" * pad)
        f.write(np.ascontiguousarray(payload, dtype="<f8").tobytes())


def _read(path) -> tuple[dict, np.ndarray]:
    data = Path(path).read_bytes()
    if len(data) < 12 or data[:8] != MAGIC:
        raise DataFormatError(f"{path}: not a kernel container (bad magic)")
    (hl,) = struct.unpack("<I", data[8:12])
    try:
        header = json.loads(data[12:12 + hl].decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise DataFormatError(f"{path}: corrupt header") from exc
    off = 12 + hl
    off += (-off) % 8
    payload = np.frombuffer(data[off:], dtype="<f8")
    if header.get("kind") == "partial":
        lo, hi = header["pair_range"]
        expect = hi - lo
    else:
        expect = header["rows"] * header["cols"]
    if payload.size != expect:
        raise DataFormatError(f"{path}: payload has {payload.size} values, header implies "
                              f"{expect} (truncated?)")
    return header, payload


def save_kernel(path, km: KernelMatrix) -> None:
    """Write a full kernel matrix container."""
    entries = np.asarray(km.to_numpy(), dtype=np.float64)
    kind = km.metadata.get("kind", "gram" if km.rows == km.cols else "cross")
    _write(path, _header(km.rows, km.cols, km.convention, km.metadata, kind,
                         kind == "gram"), entries.reshape(-1))


def load_kernel(path) -> KernelMatrix:
    h, payload = _read(path)
    if h["kind"] == "partial":
        raise DataFormatError(f"{path}: shard partial — merge it with merge_partials()")
    meta = {k: h.get(k) for k in ("config_hash", "qubits", "layers", "dataset", "kind")}
    return KernelMatrix(h["rows"], h["cols"], payload.reshape(h["rows"], h["cols"]).copy(),
                        h["convention"], meta)


def enumeration_pairs(n_a: int, n_b: int, symmetric: bool, lo: int, hi: int) -> np.ndarray:
    """0-based (i, j) pairs [lo, hi) of the row-major enumeration."""
    k = np.arange(lo, hi, dtype=np.int64)
    if not symmetric:
        return np.stack([k // n_b, k % n_b], axis=1)
    # strict upper triangle, row-major: row i starts at off(i) = i*n - i*(i+1)/2
    n = n_a
    i = np.floor((2 * n - 1 - np.sqrt((2 * n - 1) ** 2 - 8.0 * k)) / 2).astype(np.int64)
    off = lambda r: r * n - r * (r + 1) // 2  # noqa: E731
    i = np.where(off(i + 1) <= k, i + 1, i)
    i = np.where(off(i) > k, i - 1, i)
    j = k - off(i) + i + 1
    return np.stack([i, j], axis=1)


def save_partial(path, values: np.ndarray, pair_range, n_a: int, n_b: int, symmetric: bool,
                 convention: str = "probability", metadata: dict | None = None) -> None:
    """Write one shard partial: the values of pairs [lo, hi) of the enumeration."""
    values = np.asarray(values, dtype=np.float64)
    lo, hi = pair_range
    if values.size != hi - lo:
        raise ShardMergeError(f"partial has {values.size} values for pair range [{lo}, {hi})")
    _write(path, _header(n_a, n_b, convention, metadata or {}, "partial", symmetric,
                         pair_range), values)


def merge_partials(paths) -> KernelMatrix:
    """Merge shard partial files into the full matrix: deterministic
    placement by pair index; gaps/overlaps raise ShardMergeError naming the pair."""
    parts, first = [], None
    for p in paths:
        h, vals = _read(p)
        if h.get("kind") != "partial":
            raise DataFormatError(f"{p}: not a shard partial")
        if first is None:
            first = h
        elif any(h.get(k) != first.get(k) for k in ("rows", "cols", "convention", "symmetric",
                                                     "config_hash")):
            raise ShardMergeError(f"{p}: partial belongs to a different kernel matrix")
        lo, hi = h["pair_range"]
        pairs = enumeration_pairs(h["rows"], h["cols"], h["symmetric"], lo, hi) + 1
        parts.append(([tuple(map(int, ij)) for ij in pairs], vals.tolist()))
    if first is None:
        raise ShardMergeError("no partials to merge")
    meta = {k: first.get(k) for k in ("config_hash", "qubits", "layers", "dataset")}
    meta["kind"] = "gram" if first["symmetric"] else "cross"
    return shard_merge(parts, first["rows"], first["cols"], first["symmetric"],
                       first["convention"], meta)


def export_csv(path, km: KernelMatrix) -> None:
    """Row-major CSV with 17 significant digits (exact float64 round trip)."""
    np.savetxt(path, np.asarray(km.to_numpy()), fmt="%.17g", delimiter=",")


def shard_pair_range(n_a: int, n_b: int, symmetric: bool, shard: int, n_shards: int):
    """Contiguous ceil(P/W) pair range of shard k (0-based)."""
    P = n_a * (n_a - 1) // 2 if symmetric else n_a * n_b
    return shard_range(P, shard, n_shards)
