"""partial_amplitude / single_amplitude / plan_cut (SURVEY 8(f) row 5,
reference pathsum.hpp:188-459) through the Python facade: the cut method's
branches batched as extra qubits of two half-size GPU states
(qs_partial_amplitude), checked against the C oracle's full state vector."""
import numpy as np
import pytest

import oracle_lib as ol
from paper_2212_14201_b200 import qforge as Q

pytestmark = pytest.mark.gpu


def random_cut_circuit(n, gates, seed, max_two):
    rng = np.random.default_rng(seed)
    p = Q.Program(n, 0)
    two = 0
    kinds = [Q.GateKind.H, Q.GateKind.S, Q.GateKind.T, Q.GateKind.RX, Q.GateKind.RY, Q.GateKind.RZ, Q.GateKind.U3]
    for _ in range(gates):
        if two < max_two and rng.integers(3) == 0:
            a, b = rng.choice(n, 2, replace=False)
            p.add(Q.make_gate(Q.GateKind.CNOT if rng.integers(2) else Q.GateKind.CZ, [int(a), int(b)]))
            two += 1
        else:
            k = kinds[rng.integers(len(kinds))]
            ar = {Q.GateKind.RX: 1, Q.GateKind.RY: 1, Q.GateKind.RZ: 1, Q.GateKind.U3: 3}.get(k, 0)
            p.add(Q.make_gate(k, [int(rng.integers(n))], [float(x) for x in rng.uniform(0, 6.28, ar)]))
    return p


def bits(i, n):
    return format(i, "0%db" % n)


@pytest.mark.parametrize("n,gates,two,seed", [(4, 18, 4, 1), (7, 40, 8, 2), (12, 120, 10, 3), (18, 200, 9, 4),
                                              (22, 300, 7, 5)])
def test_partial_amplitude_matches_full_state(n, gates, two, seed):
    p = random_cut_circuit(n, gates, seed, two)
    plan = Q.plan_cut(p)
    want = ol.run_gates(n, p.gates())
    rng = np.random.default_rng(seed + 100)
    idx = [0, (1 << n) - 1] + [int(x) for x in rng.integers(0, 1 << n, 6)]
    targets = [bits(i, n) for i in idx]
    got = Q.partial_amplitude(p, plan, targets)
    for i, t in zip(idx, targets):
        assert abs(got[t] - want[i]) <= 1e-10, (t, got[t], want[i])


def test_partial_amplitude_branch_chunks():
    """More branch variables than fit the batch: the remaining ones are fixed
    per chunk (batch_qubits small) -- same amplitudes.  A fixed cut (qubits
    0-7 | 8-15) with 4 crossing CZ/CNOTs (each chunk of fixed variables is its
    own plan, so the test keeps the chunk count small)."""
    n = 16
    p = random_cut_circuit(n, 100, 9, 0)
    rng = np.random.default_rng(21)
    body = list(p.body)
    for j in range(4):
        a, b = int(rng.integers(8)), 8 + int(rng.integers(8))
        g = Q.make_gate(Q.GateKind.CZ if j % 2 else Q.GateKind.CNOT, [a, b] if j % 3 else [b, a])
        body.insert(15 * (j + 1), g)
    p.body = body
    cross = [i for i, g in enumerate(p.body) if len(g.targets) == 2 and (g.targets[0] < 8) != (g.targets[1] < 8)]
    plan = Q.CutPlan(list(range(8)), list(range(8, 16)), cross, 1 << len(cross))
    assert len(cross) == 4
    want = ol.run_gates(n, p.gates())
    targets = [bits(i, n) for i in (0, 5, 777, (1 << n) - 3)]
    for bq in (0, 8 + 1, 8 + 2):  # blocks of 8: all 4, 1 or 2 branch qubits batched, the rest chunked
        got = Q.partial_amplitude(p, plan, targets, batch_qubits=bq)
        for t in targets:
            assert abs(got[t] - want[int(t, 2)]) <= 1e-10, (bq, t)


def test_cut_planning_and_errors():
    p = Q.Program(4, 0)
    p.add(Q.make_gate(Q.GateKind.CNOT, [0, 1]))
    p.add(Q.make_gate(Q.GateKind.CNOT, [2, 3]))
    p.add(Q.make_gate(Q.GateKind.CZ, [1, 2]))
    p.add(Q.make_gate(Q.GateKind.CNOT, [0, 1]))
    plan = Q.plan_cut(p)
    assert len(plan.block_a) == 2 and plan.crossing_gates == [2] and plan.branch_count == 2
    with pytest.raises(Q.BudgetExceeded) as e:
        Q.partial_amplitude(p, plan, ["0000"], branch_budget=1)
    assert e.value.estimated_paths == 2
    bad = Q.CutPlan(plan.block_a, plan.block_b, [], plan.branch_count)
    with pytest.raises(Q.ValidationError):
        Q.partial_amplitude(p, bad, ["0000"])
    sw = Q.Program(4, 0)
    sw.add(Q.make_gate(Q.GateKind.SWAP, [0, 2]))
    with pytest.raises(Q.UnsupportedError):
        Q.plan_cut(sw)
    q = Q.Program(3, 0)
    q.add(Q.make_gate(Q.GateKind.H, [0]))
    q.add(Q.make_gate(Q.GateKind.CNOT, [0, 1]))
    q.add(Q.make_gate(Q.GateKind.CZ, [1, 2]))
    q.add(Q.make_gate(Q.GateKind.TOFFOLI, [0, 1, 2]))
    assert Q.path_count_estimate(q) == 16
    with pytest.raises(Q.BudgetExceeded):
        Q.single_amplitude(q, "000", 8)
    want = ol.run_gates(3, q.gates())
    for i in range(8):
        assert abs(Q.single_amplitude(q, bits(i, 3)) - want[i]) <= 1e-12
    with pytest.raises(Q.ValidationError):
        Q.single_amplitude(q, "00")


@pytest.mark.parametrize("c", __import__("golden_io").cases("cut", "manifest_cut.json"), ids=lambda c: c["name"])
def test_partial_amplitude_matches_reference_values(c):
    """The reference's own partial_amplitude values (ref_driver golden_cut: its
    plan_cut + branch loop over StateVector runs) for layered random circuits,
    6-20 qubits, against the batched GPU form with the same cut."""
    import golden_io as gio
    circ = gio.read_circuit(c["name"] + ".circ")
    p = Q.Program(circ.qubits, 0)
    for g in circ.gates:
        q = Q.make_gate(Q.GateKind(g.kind), g.targets, g.params)
        q.controls = list(g.controls)
        q.dagger = g.dagger
        p.add(q)
    plan = Q.CutPlan(c["block_a"], c["block_b"], c["crossing_gates"], c["branch_count"])
    got = Q.partial_amplitude(p, plan, c["targets"])
    for t, re, im in zip(c["targets"], c["re"], c["im"]):
        assert abs(got[t] - complex(re, im)) <= 1e-10, t


def test_partial_amplitude_edge_cases():
    """No crossing gates (one branch), empty target list, duplicate targets,
    one-qubit blocks, an empty program."""
    p = Q.Program(2, 0)
    p.add(Q.make_gate(Q.GateKind.H, [0]))
    p.add(Q.make_gate(Q.GateKind.RY, [1], [0.3]))
    plan = Q.plan_cut(p)
    assert plan.crossing_gates == [] and plan.branch_count == 1
    want = ol.run_gates(2, p.gates())
    got = Q.partial_amplitude(p, plan, ["00", "01", "10", "11", "01"])
    assert set(got) == {"00", "01", "10", "11"}
    for t in got:
        assert abs(got[t] - want[int(t, 2)]) <= 1e-12
    assert Q.partial_amplitude(p, plan, []) == {}
    e = Q.Program(3, 0)
    pe = Q.plan_cut(e)
    got = Q.partial_amplitude(e, pe, ["000", "101"])
    assert abs(got["000"] - 1) <= 1e-15 and abs(got["101"]) <= 1e-15
    c = Q.Program(2, 0)
    c.add(Q.make_gate(Q.GateKind.H, [0]))
    c.add(Q.make_gate(Q.GateKind.CNOT, [0, 1]))
    pc = Q.plan_cut(c)
    assert pc.branch_count == 2
    got = Q.partial_amplitude(c, pc, ["00", "11", "01"])
    assert abs(got["00"] - 2 ** -0.5) <= 1e-12 and abs(got["11"] - 2 ** -0.5) <= 1e-12 and abs(got["01"]) <= 1e-12
