"""Feature-map configuration (reference: pkg/src/tnkernel/circuit.py:74-91).

Same frozen dataclass, field names, defaults and validation messages as the reference's
``FeatureMapConfig``, so a config built for the reference drops in unchanged.  Also accepts
any object exposing ``width``/``layers``/``entanglement``/``embedding`` (e.g. the reference's
own class) through :func:`as_config`.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

CONVENTIONS = ("probability", "magnitude")


@dataclass(frozen=True)
class FeatureMapConfig:
    """Feature-map family: RY angle embedding with a linear CNOT chain."""

    width: int
    layers: int = 2
    entanglement: str = "linear"
    embedding: str = "ry_angle"

    def __post_init__(self):
        if self.width < 1:
            raise ValueError("width must be >= 1")
        if self.layers < 1:
            raise ValueError("layers must be >= 1")
        if self.entanglement != "linear":
            raise ValueError(f"unsupported entanglement {self.entanglement!r}")
        if self.embedding != "ry_angle":
            raise ValueError(f"unsupported embedding {self.embedding!r}")

    def config_hash(self) -> str:
        """Stable hash of the feature-map structure (KernelMatrix metadata)."""
        key = f"{self.width}|{self.layers}|{self.entanglement}|{self.embedding}"
        return hashlib.sha256(key.encode()).hexdigest()[:16]


def as_config(cfg) -> FeatureMapConfig:
    """Coerce a FeatureMapConfig-like object (ours or the reference's) to ours."""
    if isinstance(cfg, FeatureMapConfig):
        return cfg
    try:
        return FeatureMapConfig(int(cfg.width), int(getattr(cfg, "layers", 2)),
                                str(getattr(cfg, "entanglement", "linear")),
                                str(getattr(cfg, "embedding", "ry_angle")))
    except AttributeError as exc:
        raise TypeError(f"expected a FeatureMapConfig, got {type(cfg).__name__}") from exc


def check_convention(convention: str) -> str:
    if convention not in CONVENTIONS:
        raise ValueError(f"unknown kernel convention {convention!r}")
    return convention
