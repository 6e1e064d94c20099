"""Pins the C oracle (oracle/qsim_oracle.c) against golden vectors emitted by
the unmodified reference (oracle/_ref/ref_driver; tests/golden/README.md).

CPU only.  The oracle is trusted as the GPU checker only after these pass.
"""
import numpy as np
import pytest

import golden_io as gio
import oracle_lib as ol


def test_rng_stream_bit_exact():
    # rng.hpp:9-46 -- mt19937_64, uniform=(next()>>11)*2^-53, derive, below
    c = gio.case("rng")
    for s in c["streams"]:
        r = ol.Rng(s["seed"])
        assert [str(r.next()) for _ in range(8)] == s["next"]
        u = ol.Rng(s["seed"])
        assert [u.uniform() for _ in range(8)] == s["uniform"]
        assert str(ol.Rng(s["seed"], derive_index=3).next()) == s["derive3"]
        assert str(ol.lib().qo_splitmix64(s["seed"])) == s["splitmix"]
        assert str(ol.Rng(s["seed"]).below(10)) == s["below10"]


def _same_gates(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert (x.kind, x.targets, x.controls, x.dagger) == (y.kind, y.targets, y.controls, y.dagger)
        assert x.params == y.params  # bit-exact angles


@pytest.mark.parametrize("name", [c["name"] for c in gio.cases("state") if c["name"].startswith("random_")
                                  and not c["name"].endswith("fused")])
def test_random_circuit_generator_bit_exact(name):
    # bench.hpp:72-94
    _, n, d, seed = name.split("_")
    circ = gio.read_circuit(name + ".circ")
    _same_gates(ol.gen("random_circuit", int(n), int(d), int(seed)), circ.gates)


def test_synthetic_generators_match_reference_side():
    _same_gates(ol.gen("ghz", 6), gio.read_circuit("ghz_6.circ").gates)
    _same_gates(ol.gen("qft", 6, 13), gio.read_circuit("qft_6_13.circ").gates)
    _same_gates(ol.gen("qft", 10, 717), gio.read_circuit("qft_10_717.circ").gates)
    _same_gates(ol.gen("hea", 8, 3, 5), gio.read_circuit("hea_8_3_5.circ").gates)
    _same_gates(ol.gen("ghz", 20), gio.read_circuit("ghz_20.circ").gates)
    _same_gates(ol.gen("qft", 20, 0x5A5A5), gio.read_circuit("qft_20.circ").gates)


STATE_CASES = [c for c in gio.cases("state")]


@pytest.mark.parametrize("c", STATE_CASES, ids=[c["name"] for c in STATE_CASES])
def test_oracle_final_state_and_reductions(c):
    circ = gio.read_circuit(c["name"] + ".circ")
    n = circ.qubits
    want = gio.read_amps(c["name"] + ".amps")
    got = ol.run_gates(n, circ.gates)
    # fused reference runs differ from unfused ones only by rounding
    tol = 1e-12 if not c["fusion"] else 1e-11
    assert np.max(np.abs(got - want)) <= tol
    # reductions on the reference's own amplitudes must agree bit for bit
    # where the reduction order is the reference's (chunked_sum, serial loops)
    assert ol.checksum(want, n) == c["checksum"]
    assert ol.norm2(want, n) == c["norm2"]
    assert [ol.prob_one(want, n, q) for q in range(n)] == c["prob_one"]
    assert ol.probs(want, n, c["marginal_qubits"]).tolist() == c["marginal"]
    # and on the oracle's own evolution within |dprob| <= 1e-12
    assert abs(ol.checksum(got, n) - c["checksum"]) <= 1e-12 * (1 << n)
    assert np.max(np.abs(np.array([ol.prob_one(got, n, q) for q in range(n)]) - c["prob_one"])) <= 1e-12


def test_oracle_ulp_level_agreement():
    # The restatement follows the reference's expression structure; it is bit
    # for bit on the RX/RY/RZ/CNOT layers of gen_random_circuit and within a
    # few ulps elsewhere (complex products contract to FMA differently).
    for c in STATE_CASES:
        if c["fusion"] or c["name"].startswith("custom_"):
            continue
        circ = gio.read_circuit(c["name"] + ".circ")
        got = ol.run_gates(circ.qubits, circ.gates)
        want = gio.read_amps(c["name"] + ".amps")
        if c["name"].startswith("random_"):
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), c["name"]
        else:
            assert np.max(np.abs(got - want)) <= 4e-16, c["name"]


@pytest.mark.parametrize("c", gio.cases("sample"), ids=[c["name"] for c in gio.cases("sample")])
def test_oracle_counts_identical(c):
    # simulator.hpp:164-178 + BasisSampler statevector.hpp:542-570
    circ = gio.read_circuit(c["name"] + ".circ")
    a = ol.run_gates(circ.qubits, circ.gates)
    idx = ol.sample_seeded(a, circ.qubits, c["seed"], c["shots"])
    assert gio.counts_from_indices(idx, circ.measures, circ.cbits) == c["counts"]


def test_oracle_collapse_sequence():
    c = gio.case("collapse")
    circ = gio.read_circuit(c["circuit"])
    a = ol.run_gates(circ.qubits, circ.gates)
    for i, step in enumerate(c["steps"]):
        assert ol.measure_collapse(a, circ.qubits, step["q"], step["u"]) == step["outcome"]
        assert abs(ol.norm2(a, circ.qubits) - step["norm2"]) <= 1e-14
        if i == 2:
            assert np.max(np.abs(a - gio.read_amps("collapse_mid.amps"))) <= 1e-14


@pytest.mark.parametrize("c", gio.cases("expectation"), ids=[c["name"] for c in gio.cases("expectation")])
def test_oracle_expectation(c):
    circ = gio.read_circuit(c["name"] + ".circ")
    a = ol.run_gates(circ.qubits, circ.gates)
    terms = ol.parse_hamiltonian(c["hamiltonian"], circ.qubits)
    re, im = ol.expectation(a, circ.qubits, terms)
    assert abs(re - c["value"]) <= 1e-12
    assert abs(im) <= 1e-10


@pytest.mark.parametrize("name", ["ghz_20", "qft_20"])
def test_oracle_config1_digest(name):
    c = gio.case(name)
    circ = gio.read_circuit(name + ".circ")
    a = ol.run_gates(20, circ.gates)
    assert abs(ol.checksum(a, 20) - c["checksum"]) <= 1e-9
    idx = np.array(c["idx"])
    assert np.max(np.abs(a[idx].real - c["re"])) <= 1e-12
    assert np.max(np.abs(a[idx].imag - c["im"])) <= 1e-12
    assert np.max(np.abs(ol.probs_full(a, 20)[:256] - c["probs_head"])) <= 1e-12
    assert np.max(np.abs(ol.probs(a, 20, c["marginal_qubits"]) - c["marginal"])) <= 1e-12


def test_qft_closed_form_small():
    # QFT generator convention pinned against the DFT closed form
    for n, x in ((6, 13), (10, 717)):
        a = ol.run_gates(n, ol.gen("qft", n, x))
        k = np.arange(1 << n)
        want = np.exp(2j * np.pi * x * k / (1 << n)) / np.sqrt(1 << n)
        assert np.max(np.abs(a - want)) <= 1e-12


def test_huge_manifest_is_the_benchmarked_circuits():
    """tests/golden/huge holds the reference's results for exactly the
    circuits bench.py times (generators are bit-exact, see above)."""
    import json
    import os
    from paper_2212_14201_b200 import qforge as Q
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "huge")
    cases = {c["name"]: c for c in json.load(open(os.path.join(here, "manifest_huge.json")))}
    assert set(cases) == {"random28", "random30", "qft30"}
    import bench
    for name, c in cases.items():
        gen, args, n = bench.WORKLOADS[name]
        assert (gen, list(args), n) == (c["gen"], c["args"], c["n"])
        p = {"random": Q.gen_random_circuit, "qft": Q.gen_qft}[gen](*args)
        assert p.gate_count() == c["gates"]
        assert os.path.getsize(os.path.join(here, c["amps"])) == 16 * c["window"] * len(c["starts"])
        assert abs(c["norm2"] - 1) < 1e-12 and len(c["probs_head"]) == 256 and len(c["marginal"]) == 64
        w = np.fromfile(os.path.join(here, c["amps"]), dtype=np.complex128).reshape(8, -1)
        assert np.allclose(np.abs(w[0, :256]) ** 2, c["probs_head"], atol=1e-15, rtol=0)
    # QFT of a basis state: every amplitude is exp(2 pi i x k / 2^n) / sqrt(2^n)
    q = cases["qft30"]
    x, n = q["args"][1], q["n"]
    w = np.fromfile(os.path.join(here, q["amps"]), dtype=np.complex128).reshape(8, -1)
    for s, row in zip(q["starts"], w):
        k = np.arange(s, s + q["window"], dtype=np.uint64)
        ph = ((np.uint64(x) * k) & np.uint64((1 << n) - 1)).astype(np.float64)  # exact: x k < 2^60
        want = np.exp(2j * np.pi * ph / (1 << n)) / np.sqrt(1 << n)
        assert np.max(np.abs(row - want)) <= 1e-10


def test_reference_cpu_arm_steps_and_configs():
    """bench.py's CPU arm: ref_driver bench_steps runs the reference's run()
    body (fuse_circuit + apply_gate) on one resident state, one JSON line per
    step, and its final digest equals the reference's full run() of the same
    gates (a small circuit; the bench uses the 30-qubit workload)."""
    import json
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "ref_driver")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_driver not built (needs /root/reference at build time)")
    env = dict(os.environ, OMP_NUM_THREADS="2")
    n, d = 10, 3
    out = subprocess.run([exe, "bench_steps", "random", str(n), str(d), "424242", str(2 * n), str(d), "1"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    steps = [r for r in rows if "seconds" in r]
    assert len(steps) == d and all(r["gates"] == 2 * n and r["passes"] >= 1 for r in steps)
    assert rows[0]["threads"] == 2 and "alloc_seconds" in rows[0]
    from paper_2212_14201_b200 import qforge as Q
    want = ol.checksum(ol.run_gates(n, Q.gen_random_circuit(n, d, 424242).gates()), n)
    assert abs(rows[-1]["checksum"] - want) <= 1e-9 * want


def _qprogram(circ):
    from paper_2212_14201_b200 import qforge as Q
    p = Q.Program(circ.qubits, 0)
    for g in circ.gates:
        q = Q.make_gate(Q.GateKind(g.kind), g.targets, g.params)
        q.controls = list(g.controls)
        q.dagger = g.dagger
        p.add(q)
    return p


@pytest.mark.parametrize("c", gio.cases("cut", "manifest_cut.json"), ids=lambda c: c["name"])
def test_plan_cut_matches_reference(c):
    """qforge.plan_cut (host combinatorics of the facade) chooses the same cut
    as the reference's plan_cut (pathsum.hpp:232-310), exhaustive and greedy."""
    from paper_2212_14201_b200 import qforge as Q
    p = _qprogram(gio.read_circuit(c["name"] + ".circ"))
    plan = Q.plan_cut(p)
    assert plan.block_a == c["block_a"] and plan.block_b == c["block_b"]
    assert plan.crossing_gates == c["crossing_gates"] and plan.branch_count == c["branch_count"]


def test_qft_closed_form_convention():
    """QFT|b> = 2^(-n/2) sum_k exp(2 pi i b k / 2^n) |k> in the oracle (the
    closed form the GPU tests use beyond 30 qubits)."""
    from paper_2212_14201_b200 import qforge as Q
    n, b = 8, 0xA5
    a = ol.run_gates(n, Q.gen_qft(n, b).gates())
    k = np.arange(1 << n)
    assert np.max(np.abs(a - np.exp(2j * np.pi * b * k / 2 ** n) / 2 ** (n / 2))) <= 1e-12
