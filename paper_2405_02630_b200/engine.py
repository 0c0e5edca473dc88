"""``contract_batch`` drop-in (reference: pkg/src/tnkernel/engine.py:132-166).

Same call shape — ``contract_batch(template, operand_sets, path, workers=1) -> list[complex]``
— and the same error contract: a width mismatch raises ``RebindError("operand set k: ...")``
up front (engine.py:139-144), a non-finite angle raises ``RebindError("operand set k: feature
angles must be finite")`` (network.py:295-296 rewrapped at engine.py:153-155), an empty batch
returns ``[]`` (engine.py:146-147), output order equals input order.

``template`` is anything exposing ``width`` and ``layers`` — the reference's simplified
``TensorNetwork`` (network.py:69-75) or a :class:`FeatureMapConfig`.  ``path`` is accepted and
ignored when it is a reference path (the sweep order is structural) or used when it is a
:class:`SweepPlan`.  Amplitudes are real for this feature map (RY and CNOT are real); they
are returned as ``complex`` with a zero imaginary part, like the reference.

Each call uploads the batch, builds the gate planes per distinct vector slot and runs the
pair-list sm_100a kernel (``qk_pair_amplitudes``); no CPU compute path exists.
"""
from __future__ import annotations

import numpy as np

from .config import FeatureMapConfig
from .errors import RebindError
from .planner import SweepPlan, plan_for


def contract_batch(template, operand_sets, path=None, workers: int = 1) -> list[complex]:
    import torch

    from . import device as dev

    width = int(template.width)
    layers = int(getattr(template, "layers", 2) or 2)
    pairs = [(np.asarray(a, dtype=float), np.asarray(b, dtype=float)) for a, b in operand_sets]
    for k, (a, b) in enumerate(pairs):
        if a.shape != (width,) or b.shape != (width,):
            raise RebindError(f"operand set {k}: vectors of lengths {a.size}/{b.size}"
                              f" do not match width {width}")
    if int(workers) < 1:
        raise ValueError("workers must be >= 1")
    if not pairs:
        return []
    for k, (a, b) in enumerate(pairs):
        if not (np.all(np.isfinite(a)) and np.all(np.isfinite(b))):
            raise RebindError(f"operand set {k}: feature angles must be finite")
    plan = path if isinstance(path, SweepPlan) else plan_for(FeatureMapConfig(width, layers))
    A = torch.as_tensor(np.stack([a for a, _ in pairs]), dtype=torch.float64).cuda()
    B = torch.as_tensor(np.stack([b for _, b in pairs]), dtype=torch.float64).cuda()
    idx = torch.arange(len(pairs), dtype=torch.int64, device=A.device)
    amp = dev.pair_amplitudes(dev.gate_build(plan, A), dev.gate_build(plan, B),
                              torch.stack([idx, idx], dim=1))
    return [complex(v, 0.0) for v in amp.cpu().tolist()]
