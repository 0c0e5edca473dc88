"""Host sweep planner (Python face of the C++ ``qk_plan``).

Replaces the reference's plan-once step — ``plan_contraction`` over the simplified network
(reference: pkg/src/tnkernel/paths.py:529-543, network.py:183-280) — whose result every
pair reuses ("path reuse").  For the RY + linear-CNOT feature
map the optimal order is structural (a sweep along the qubit chain with a bond-4 state), so
the plan records that sweep's geometry and its per-entry costs.  One plan per
(width, layers, convention); cached.
"""
from __future__ import annotations

import ctypes
import functools

from . import _native
from .config import FeatureMapConfig, as_config, check_convention

_CONV = {"probability": _native.QK_PROBABILITY, "magnitude": _native.QK_MAGNITUDE}


class SweepPlan:
    """A fixed contraction plan for one circuit structure; immutable, thread-safe."""

    def __init__(self, width: int, layers: int = 2, convention: str = "probability"):
        check_convention(convention)
        lib = _native.lib()
        handle = ctypes.c_void_p()
        _native.check(lib.qk_plan_create(int(width), int(layers), _CONV[convention],
                                         ctypes.byref(handle)))
        self._h = handle
        self.width = int(width)
        self.layers = int(layers)
        self.convention = convention
        info = _native.PlanInfo()
        _native.check(lib.qk_plan_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    @property
    def tile_edge(self) -> int:
        return self.info["tile_edge"]

    def planes_bytes(self, n_samples: int) -> int:
        return int(_native.lib().qk_planes_bytes(self._h, int(n_samples)))

    def gram_tile_count(self, n_samples: int) -> int:
        return int(_native.lib().qk_gram_tile_count(self._h, int(n_samples)))

    def cross_tile_count(self, n_rows: int, n_cols: int) -> int:
        return int(_native.lib().qk_cross_tile_count(self._h, int(n_rows), int(n_cols)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _native._lib is not None:
            _native._lib.qk_plan_destroy(h)
            self._h = None

    def __repr__(self) -> str:
        return (f"SweepPlan(width={self.width}, layers={self.layers}, "
                f"convention={self.convention!r}, bond={self.info['bond']}, "
                f"tile={self.info['tile_edge']}, chunk={self.info['chunk']})")


@functools.lru_cache(maxsize=64)
def _cached(width: int, layers: int, convention: str) -> SweepPlan:
    return SweepPlan(width, layers, convention)


def plan_for(cfg: FeatureMapConfig, convention: str = "probability") -> SweepPlan:
    cfg = as_config(cfg)
    return _cached(cfg.width, cfg.layers, check_convention(convention))
