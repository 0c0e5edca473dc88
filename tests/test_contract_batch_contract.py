"""contract_batch's error contract and template recognition (CPU: every case raises before
any device work, or calls kernel_layers directly).

Against the reference's own objects when /root/reference is importable (the build
container): its kernel networks — simplified or not, any width / layers — are recognised;
its random-circuit network raises the reference's RebindError (test_network.py:141-145
semantics, rewrapped with the operand-set index as engine.py:153-155 does); bad paths raise
what estimate_cost raises (paths.py:88-130), before the empty-batch return
(engine.py:145-147)."""
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2405_02630_b200 import FeatureMapConfig, RebindError, StructuralError, contract_batch
from paper_2405_02630_b200.engine import kernel_layers

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref():
    if not (REF / "tnkernel").is_dir():
        pytest.skip("reference package not present (only in the build container)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import tnkernel.circuit as circuit
    import tnkernel.network as network
    import tnkernel.paths as paths
    return circuit, network, paths


def _kernel_net(ref, n, L, simplified=True):
    circuit, network, _ = ref
    cfg = circuit.FeatureMapConfig(n, layers=L)
    tn = network.circuit_to_network(circuit.compose_kernel_circuit(np.zeros(n), np.zeros(n), cfg))
    return network.simplify(tn) if simplified else tn


def _random_net(ref, rng, width, n_gates):
    circuit, network, _ = ref
    G, K = circuit.Gate, circuit.GateKind
    gates = []
    for _ in range(n_gates):
        k = [K.H, K.RY, K.RZ, K.CNOT][rng.integers(4)]
        if k is K.CNOT:
            c, t = rng.choice(width, size=2, replace=False)
            gates.append(G(K.CNOT, (int(c), int(t))))
        elif k is K.H:
            gates.append(G(k, (int(rng.integers(width)),)))
        else:
            gates.append(G(k, (int(rng.integers(width)),), float(rng.uniform(-6, 6))))
    return network.circuit_to_network(circuit.Circuit(width, tuple(gates)))


@pytest.mark.parametrize("simplified", [True, False])
@pytest.mark.parametrize("n,L", [(1, 1), (1, 2), (2, 1), (2, 2), (3, 2), (5, 3), (8, 2),
                                 (4, 4), (17, 2)])
def test_reference_kernel_networks_recognised(ref, n, L, simplified):
    assert kernel_layers(_kernel_net(ref, n, L, simplified)) == L


def test_non_kernel_network_raises_no_slots(ref, rng):
    tn = _random_net(ref, rng, 2, 6)
    pairs = [(np.zeros(2), np.zeros(2)), (np.ones(2), np.ones(2))]
    with pytest.raises(RebindError, match=r"^operand set 0: network carries no feature slots; "
                                          r"not built from a kernel circuit$"):
        contract_batch(tn, pairs, None)
    # the reference checks finiteness first (network.py:295-298)
    with pytest.raises(RebindError, match=r"^operand set 0: feature angles must be finite$"):
        contract_batch(tn, [(np.full(2, np.nan), np.zeros(2))] + pairs, None)
    # an empty batch never reaches the rebind
    assert contract_batch(tn, [], None) == []


def test_template_without_layers_raises_no_slots():
    class Template:  # duck-typed: the reference's TensorNetwork.layers defaults to 0
        width, layers = 3, 0

    with pytest.raises(RebindError, match="operand set 0: network carries no feature slots"):
        contract_batch(Template(), [(np.zeros(3), np.zeros(3))])


def test_width_mismatch_first(ref, rng):
    tn = _random_net(ref, rng, 2, 6)
    with pytest.raises(RebindError, match=r"^operand set 1: vectors of lengths 3/2 do not "
                                          r"match width 2$"):
        contract_batch(tn, [(np.zeros(2), np.zeros(2)), (np.zeros(3), np.zeros(2))], "bad")


def test_bad_paths_like_estimate_cost(ref):
    _, _, paths = ref
    tn = _kernel_net(ref, 4, 2)
    pairs = [(np.zeros(4), np.zeros(4))]
    with pytest.raises(TypeError, match="expected ContractionPath or SlicedPath, got str"):
        contract_batch(tn, pairs, "greedy")
    with pytest.raises(TypeError, match="got str"):  # before the empty-batch return
        contract_batch(tn, [], "greedy")
    m = len(tn.operands)
    with pytest.raises(StructuralError, match=f"path has 2 merges for {m} operands"):
        contract_batch(tn, pairs, paths.ContractionPath(((0, 1), (2, 3)), 0, 0))
    merges = tuple((0, 1) for _ in range(m - 1))
    with pytest.raises(StructuralError, match=r"merge \(0,1\) references an unavailable"):
        contract_batch(tn, pairs, paths.ContractionPath(merges, 0, 0))
    with pytest.raises(StructuralError, match="path has 1 merges"):
        contract_batch(tn, [], paths.SlicedPath(paths.ContractionPath(((0, 1),), 0, 0), (), 1,
                                                0, 0))


def test_reference_plan_accepted_by_validation(ref):
    """A real plan_contraction path (sliced or not) passes the validation."""
    _, _, paths = ref
    tn = _kernel_net(ref, 6, 2)
    plan = paths.plan_contraction(tn)
    from paper_2405_02630_b200.engine import _check_path
    _check_path(tn, plan, 6, 2)
    _check_path(tn, plan.path, 6, 2)


@pytest.mark.parametrize("mutate", ["drop_cnot", "reverse_cnot", "wrong_layers", "extra_gate"])
def test_slotted_non_feature_map_networks_rejected(ref, mutate):
    circuit, network, _ = ref
    n, L = 4, 2
    cfg = circuit.FeatureMapConfig(n, layers=L)
    c = circuit.compose_kernel_circuit(np.zeros(n), np.zeros(n), cfg)
    gates = list(c.gates)
    G, K = circuit.Gate, circuit.GateKind
    layers = L
    if mutate == "drop_cnot":
        gates.remove(next(g for g in gates if g.kind is K.CNOT))
    elif mutate == "reverse_cnot":
        k = next(i for i, g in enumerate(gates) if g.kind is K.CNOT)
        gates[k] = G(K.CNOT, tuple(reversed(gates[k].qubits)))
    elif mutate == "wrong_layers":
        layers = 3
    else:
        gates.insert(3, G(K.H, (1,)))
    tn = network.simplify(network.circuit_to_network(circuit.Circuit(n, tuple(gates),
                                                                     layers=layers)))
    with pytest.raises(StructuralError, match="not a feature-map kernel network"):
        kernel_layers(tn)
    with pytest.raises(StructuralError, match="not a feature-map kernel network"):
        contract_batch(tn, [(np.zeros(n), np.zeros(n))])


def test_sweep_plan_must_match_template():
    from paper_2405_02630_b200 import planner
    from paper_2405_02630_b200.engine import _check_path

    p = planner.SweepPlan.__new__(planner.SweepPlan)
    p.width, p.layers = 5, 2
    with pytest.raises(StructuralError, match="does not match the template"):
        _check_path(FeatureMapConfig(6), p, 6, 2)
    _check_path(FeatureMapConfig(5), p, 5, 2)
