"""``contract_batch`` drop-in (reference: pkg/src/tnkernel/engine.py:132-166).

Same call shape — ``contract_batch(template, operand_sets, path, workers=1) -> list[complex]``
— and the same error contract, in the reference's order:

1. a width mismatch raises ``RebindError("operand set k: ...")`` up front (engine.py:139-144);
2. the path is validated once for the batch like ``estimate_cost`` (engine.py:145,
   paths.py:88-130): ``TypeError`` for an object that is not a path, ``StructuralError`` for
   a merge list that does not fit the template's operands;
3. an empty batch returns ``[]`` (engine.py:146-147);
4. per pair, in input order, what ``rebind_operands`` raises (network.py:283-302, rewrapped at
   engine.py:153-155): ``RebindError("operand set k: feature angles must be finite")``, or
   ``RebindError("operand set k: network carries no feature slots; not built from a kernel
   circuit")`` for a template without feature slots (reference test_network.py:141-145).

``template`` is the reference's ``TensorNetwork`` (simplified or not) of a kernel circuit —
its operand graph is walked wire by wire and must be exactly the RY + linear-CNOT feature-map
kernel circuit of ``compose_kernel_circuit`` (circuit.py:121-157) for some width and layers —
or a :class:`FeatureMapConfig` (anything exposing ``width`` and ``layers``).  A network that
carries feature slots but is not that circuit raises ``StructuralError`` (the engine
contracts the feature-map family only; the reference's generic contraction would accept it).
``path`` may also be a :class:`SweepPlan` (checked against the template) or ``None`` (the
cached plan).  ``workers`` is accepted for signature compatibility (one process drives one
GPU).  Amplitudes are real for this feature map (RY and CNOT are real); they are returned as
``complex`` with a zero imaginary part, like the reference.

Each call uploads the batch, builds the gate planes per distinct vector slot and runs the
pair-list sm_100a kernel (``qk_pair_amplitudes``); no CPU compute path exists.
"""
from __future__ import annotations

import numpy as np

from .config import FeatureMapConfig
from .errors import RebindError, StructuralError
from .planner import SweepPlan, plan_for

_NO_SLOTS = "network carries no feature slots; not built from a kernel circuit"


def _kind(f) -> str:
    k = getattr(f, "kind", None)
    return str(getattr(k, "value", k))


def _slots(template) -> list:
    return [f for op in template.operands for f in (getattr(op, "chain", ()) or ())
            if getattr(f, "slot", None) is not None]


def _view_checks(template) -> None:
    """The index-structure checks of the reference's planner view (paths.py:60-79)."""
    ops = template.operands
    if not ops:
        raise StructuralError("network has no operands")
    counts: dict = {}
    for op in ops:
        ix = tuple(op.indices)
        if len(set(ix)) != len(ix):
            raise StructuralError("repeated index within one operand is unsupported")
        for label in ix:
            counts[label] = counts.get(label, 0) + 1
    for label, c in counts.items():
        if c > 2:
            raise StructuralError(f"index {label} appears {c} times; hyperedges unsupported")


def _replay(merges, m: int) -> None:
    """Merge-list validation of paths.py:_replay (88-113), without the cost bookkeeping."""
    merges = list(merges)
    if len(merges) != m - 1:
        raise StructuralError(f"path has {len(merges)} merges for {m} operands")
    alive = set(range(m))
    nxt = m
    for a, b in merges:
        if a == b or a not in alive or b not in alive:
            raise StructuralError(f"merge ({a},{b}) references an unavailable operand")
        alive.discard(a)
        alive.discard(b)
        alive.add(nxt)
        nxt += 1


def _check_path(template, path, width: int, layers: int | None) -> None:
    """estimate_cost(template, path) (paths.py:121-130) for reference paths; a SweepPlan must
    describe the template's circuit."""
    if path is None:
        return
    if isinstance(path, SweepPlan):
        if path.width != width or (layers is not None and path.layers != layers):
            raise StructuralError(f"plan for width {path.width}, layers {path.layers} does not "
                                  f"match the template (width {width}, layers {layers})")
        return
    network = hasattr(template, "operands")
    if hasattr(path, "path") and hasattr(path, "sliced"):  # SlicedPath
        merges = getattr(path.path, "merges", None)
    elif hasattr(path, "merges"):  # ContractionPath
        merges = path.merges
    else:
        raise TypeError(f"expected ContractionPath or SlicedPath, got {type(path).__name__}")
    if network:
        _view_checks(template)
        _replay(merges, len(template.operands))


def kernel_layers(template) -> int | None:
    """Layers of the feature-map kernel circuit the template is, or None when it carries no
    feature slots.  A network with slots that is not exactly the RY + linear-CNOT kernel
    circuit of ``compose_kernel_circuit`` (circuit.py:121-157) raises ``StructuralError``.

    Walks every wire from its start cap through the operand graph (single-wire operands
    data[out, in], CNOTs data[out_c, out_t, in_c, in_t], network.py:125-176; fused and
    cap-absorbed operands of ``simplify`` keep their gate recipe, network.py:183-280) and
    compares each wire's gate sequence and each CNOT's (control, target) wires with the
    circuit's."""
    if not hasattr(template, "operands"):  # a FeatureMapConfig-like template
        layers = int(getattr(template, "layers", 0) or 0)
        return layers if layers >= 1 else None
    width = int(template.width)
    ops = list(template.operands)
    if not _slots(template):
        return None

    def bad(why: str):
        return StructuralError(f"template is not a feature-map kernel network ({why}); the "
                               f"engine contracts RY + linear-CNOT kernel circuits only")

    holders: dict = {}
    for p, op in enumerate(ops):
        for pos, label in enumerate(op.indices):
            holders.setdefault(label, []).append((p, pos))
    visits = [0] * len(ops)
    cnot_legs: dict = {}  # op index -> {"c": wire, "t": wire}
    wires: dict = {}
    for p0, op0 in enumerate(ops):
        if not getattr(op0, "start_cap", False):
            continue
        events = list(op0.chain or ())
        legs = []
        visits[p0] += 1
        rank = len(op0.indices)
        if rank == 0:
            if not getattr(op0, "end_cap", False):
                raise bad("dangling scalar operand")
        elif rank == 1:
            label, prev = op0.indices[0], p0
            for _ in range(len(ops) + 1):
                nxt = [(p, pos) for p, pos in holders.get(label, []) if p != prev]
                if len(nxt) != 1:
                    raise bad(f"index {label} is not a wire segment")
                p, pos = nxt[0]
                op = ops[p]
                visits[p] += 1
                if getattr(op, "two_qubit", False) and len(op.indices) == 4:
                    if pos not in (2, 3):
                        raise bad("a wire enters a CNOT through an output leg")
                    legs.append((p, "c" if pos == 2 else "t"))
                    events.append(("cnot", p, "c" if pos == 2 else "t"))
                    label, prev = op.indices[pos - 2], p
                elif len(op.indices) == 2 and op.chain:
                    if pos != 1:
                        raise bad("a wire enters a gate through its output")
                    events.extend(op.chain)
                    label, prev = op.indices[0], p
                elif len(op.indices) == 1 and getattr(op, "end_cap", False):
                    events.extend(op.chain or ())
                    break
                else:
                    raise bad(f"unexpected operand {getattr(op, 'provenance', p)!r} on a wire")
            else:
                raise bad("a wire does not end in a cap")
        else:
            raise bad("a start cap of rank > 1")
        qs = {f.slot[1] for f in events if not isinstance(f, tuple)
              and getattr(f, "slot", None) is not None}
        if len(qs) != 1:
            raise bad("a wire without exactly one feature qubit")
        q = qs.pop()
        if q in wires:
            raise bad(f"two wires carry qubit {q}")
        wires[q] = events
        for p, role in legs:
            if role in cnot_legs.setdefault(p, {}):
                raise bad("a CNOT with two legs of one role")
            cnot_legs[p][role] = q
    if sorted(wires) != list(range(width)):
        raise bad(f"wires {sorted(wires)[:4]}... do not cover width {width}")
    for p, op in enumerate(ops):
        expect = 2 if getattr(op, "two_qubit", False) else 1
        if visits[p] != expect:
            raise bad(f"operand {getattr(op, 'provenance', p)!r} is not on the wire graph")
    for legs in cnot_legs.values():
        if set(legs) != {"c", "t"} or legs["t"] != legs["c"] + 1:
            raise bad("a CNOT that is not (q, q+1)")
    # per wire: [RY(+x_j) (CNOT target of q-1) (CNOT control of q+1)] x L, then the adjoint:
    # [(control of q+1) (target of q-1) RY(-x_i)] x L
    layers = None
    for q, events in wires.items():
        toks = []
        for e in events:
            if isinstance(e, tuple):
                toks.append(e[2])
            else:
                if _kind(e) != "RY" or e.slot is None:
                    raise bad("a gate other than a feature-slot RY")
                vec, qq, sign = e.slot
                toks.append(("j" if vec == "j" and sign == 1 else
                             "i" if vec == "i" and sign == -1 else "?"))
        fwd = ["j"] + (["t"] if q > 0 else []) + (["c"] if q < width - 1 else [])
        adj = (["c"] if q < width - 1 else []) + (["t"] if q > 0 else []) + ["i"]
        L = len(toks) // (len(fwd) + len(adj)) if toks else 0
        if L < 1 or toks != fwd * L + adj * L:
            raise bad(f"wire {q} gate sequence")
        if layers is None:
            layers = L
        elif L != layers:
            raise bad("wires with different layer counts")
    declared = int(getattr(template, "layers", 0) or 0)
    if declared and declared != layers:
        raise bad(f"declares {declared} layers, its circuit has {layers}")
    return layers


def contract_batch(template, operand_sets, path=None, workers: int = 1) -> list[complex]:
    import torch

    from . import device as dev

    width = int(template.width)
    pairs = [(np.asarray(a, dtype=float), np.asarray(b, dtype=float)) for a, b in operand_sets]
    for k, (a, b) in enumerate(pairs):
        if a.shape != (width,) or b.shape != (width,):
            raise RebindError(f"operand set {k}: vectors of lengths {a.size}/{b.size}"
                              f" do not match width {width}")
    declared = getattr(template, "layers", None)
    _check_path(template, path, width, int(declared) if declared else None)
    if not pairs:
        return []
    layers = kernel_layers(template)
    for k, (a, b) in enumerate(pairs):
        if not (np.all(np.isfinite(a)) and np.all(np.isfinite(b))):
            raise RebindError(f"operand set {k}: feature angles must be finite")
        if layers is None:
            raise RebindError(f"operand set {k}: {_NO_SLOTS}")
    plan = path if isinstance(path, SweepPlan) else plan_for(FeatureMapConfig(width, layers))
    A = torch.as_tensor(np.stack([a for a, _ in pairs]), dtype=torch.float64).cuda()
    B = torch.as_tensor(np.stack([b for _, b in pairs]), dtype=torch.float64).cuda()
    idx = torch.arange(len(pairs), dtype=torch.int64, device=A.device)
    amp = dev.pair_amplitudes(dev.gate_build(plan, A), dev.gate_build(plan, B),
                              torch.stack([idx, idx], dim=1))
    return [complex(v, 0.0) for v in amp.cpu().tolist()]
