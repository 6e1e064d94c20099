"""CPU checks of the tile planner and micro-program semantics: every plan is
replayed by the host emulator (tests/tile_emu.cpp) and compared with the C
oracle.  The GPU suite repeats the same circuits on the device."""
import numpy as np
import pytest

import emu_lib
import golden_io as gio
import oracle_lib as ol
from paper_2212_14201_b200 import _native as N
from paper_2212_14201_b200 import qforge as Q


def random_unitary(k, rng):
    m = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
    q, r = np.linalg.qr(m)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def mixed_gates(n, count, seed, max_controls=2):
    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(count):
        kind = int(rng.integers(0, 16))
        perm = rng.permutation(n).tolist()
        if kind in (11, 12, 13):
            g = Q.make_gate(Q.GateKind(kind), perm[:2])
        elif kind == 14:
            g = Q.make_gate(Q.GateKind.TOFFOLI, perm[:3])
        elif kind == 15:
            k = int(rng.integers(1, 5))
            g = Q.make_custom_gate(perm[:k], random_unitary(k, rng))
        else:
            g = Q.make_gate(Q.GateKind(kind), perm[:1],
                            rng.uniform(0, 6.3, size={7: 1, 8: 1, 9: 1, 10: 3}.get(kind, 0)))
        if rng.random() < 0.25:
            used = len(g.targets)
            g.controls = perm[used:used + int(rng.integers(1, max_controls + 1))]
        if rng.random() < 0.2:
            g.dagger = True
        gates.append(g)
    return gates


@pytest.mark.parametrize("n,m,low", [(6, 12, 3), (9, 12, 3), (10, 8, 3), (12, 9, 3), (13, 10, 5), (14, 12, 3),
                                     (15, 10, 4)])
def test_emulated_tile_plan_matches_oracle_mixed(n, m, low):
    gates = mixed_gates(n, 300, 1000 + n)
    want = ol.run_gates(n, gates)
    got, passes = emu_lib.run(n, gates, N.QS_PLAN_TILED, tile_m=m, low=low)
    assert np.max(np.abs(got - want)) <= 1e-10


@pytest.mark.parametrize("which", ["random", "qft", "hea", "ghz"])
@pytest.mark.parametrize("n,m", [(14, 9), (16, 12), (18, 12)])
def test_emulated_tile_plan_matches_oracle_workloads(which, n, m):
    p = {"random": lambda: Q.gen_random_circuit(n, 6, 424242), "qft": lambda: Q.gen_qft(n, 0x1234 % (1 << n)),
         "hea": lambda: Q.gen_hea(n, 4, 7), "ghz": lambda: Q.gen_ghz(n)}[which]()
    want = ol.run_gates(n, p.gates())
    got, passes = emu_lib.run(n, p.gates(), N.QS_PLAN_TILED, tile_m=m)
    assert np.max(np.abs(got - want)) <= 1e-10


@pytest.mark.parametrize("plan", [N.QS_PLAN_UNFUSED, N.QS_PLAN_DENSE_FUSION])
def test_emulated_other_plans(plan):
    gates = mixed_gates(7, 120, 7)
    want = ol.run_gates(7, gates)
    got, _ = emu_lib.run(7, gates, plan, maxk=3)
    assert np.max(np.abs(got - want)) <= 1e-10


@pytest.mark.parametrize("c", [c for c in gio.cases("state")], ids=lambda c: c["name"])
def test_emulated_golden_states(c):
    circ = gio.read_circuit(c["name"] + ".circ")
    if circ.qubits < 6:
        pytest.skip("tiles need >= 6 qubits")
    got, _ = emu_lib.run(circ.qubits, circ.gates, N.QS_PLAN_TILED, tile_m=min(12, max(8, circ.qubits - 2)))
    assert np.max(np.abs(got - gio.read_amps(c["name"] + ".amps"))) <= 1e-10


@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("which", ["random", "qft", "mixed", "hea"])
def test_emulated_sharded_plans(which, g):
    # Sharded plans (rank bits never in a tile, SwapSteps before non-diagonal
    # gates on them, identity layout restored) replayed on the full state.
    n = 14
    gates = {"random": lambda: Q.gen_random_circuit(n, 5, 424242).gates(),
             "qft": lambda: Q.gen_qft(n, 0x2345).gates(),
             "mixed": lambda: mixed_gates(n, 250, 77 + g),
             "hea": lambda: Q.gen_hea(n, 3, 9).gates()}[which]()
    want = ol.run_gates(n, gates)
    for remap in (0, 1):
        got, steps = emu_lib.run(n, gates, N.QS_PLAN_TILED, tile_m=9, low=3, global_qubits=g, remap=remap)
        assert np.max(np.abs(got - want)) <= 1e-10, (remap, steps)


@pytest.mark.parametrize("which", ["random", "qft", "mixed", "hea"])
@pytest.mark.parametrize("n", [16, 18])
def test_emulated_13_qubit_plans_with_register_width_choice(which, n):
    """13-qubit tiles: every pass is compiled with 4 and with 5 register bits
    and the cheaper kept (pass_cost); plans mixing both widths replay to the
    oracle's state."""
    gates = {"random": lambda: Q.gen_random_circuit(n, 8, 424242).gates(),
             "qft": lambda: Q.gen_qft(n, 0x2345).gates(),
             "mixed": lambda: mixed_gates(n, 300, 99 + n),
             "hea": lambda: Q.gen_hea(n, 6, 9).gates()}[which]()
    want = ol.run_gates(n, gates)
    got, passes = emu_lib.run(n, gates, N.QS_PLAN_TILED, tile_m=13, low=4)
    assert np.max(np.abs(got - want)) <= 1e-10
