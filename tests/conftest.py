"""Shared fixtures.  `-m gpu` tests need a CUDA device (B200); everything else runs on CPU."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


def pytest_collection_modifyitems(config, items):
    """A plain `pytest` on a machine without a GPU skips the `gpu` tests instead of erroring."""
    gpu_items = [it for it in items if "gpu" in it.keywords]
    if not gpu_items:
        return
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="needs a CUDA device")
    for it in gpu_items:
        it.add_marker(skip)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


GOLDEN_CASES = sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem != "known_answers")


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(1234)
