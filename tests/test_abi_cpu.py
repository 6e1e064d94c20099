"""CPU-side checks of the product: the C ABI library loads and exports every
symbol include/qsb.h declares; host-only parts (planner, reference-mode
fusion, RNG, generators, validation) match the reference.  No GPU needed.
"""
import os
import re

import numpy as np
import pytest

import golden_io as gio
from paper_2212_14201_b200 import _native as N
from paper_2212_14201_b200 import qforge as Q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "qsb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    declared = header_functions()
    assert len(declared) >= 40
    missing = [f for f in declared if not hasattr(L, f)]
    assert not missing, missing
    assert set(declared) == set(N.EXPORTED)
    assert L.qs_abi_version() == 1


def test_rng_mirror_matches_reference_stream():
    c = gio.case("rng")
    for s in c["streams"]:
        r = Q.Rng(s["seed"])
        assert [str(r.next()) for _ in range(8)] == s["next"]
        u = Q.Rng(s["seed"])
        assert [u.uniform() for _ in range(8)] == s["uniform"]
        assert str(Q.Rng.derive(s["seed"], 3).next()) == s["derive3"]
        assert str(Q.splitmix64(s["seed"])) == s["splitmix"]


def _same(prog, circ):
    gates = prog.gates()
    assert len(gates) == len(circ.gates)
    for a, b in zip(gates, circ.gates):
        assert (int(a.kind), list(a.targets), list(a.controls), bool(a.dagger)) == \
               (b.kind, b.targets, b.controls, b.dagger)
        assert list(a.params) == b.params


def test_generators_match_reference_side():
    _same(Q.gen_random_circuit(8, 6, 42), gio.read_circuit("random_8_6_42.circ"))
    _same(Q.gen_random_circuit(14, 3, 424242), gio.read_circuit("random_14_3_424242.circ"))
    _same(Q.gen_ghz(20), gio.read_circuit("ghz_20.circ"))
    _same(Q.gen_qft(20, 0x5A5A5), gio.read_circuit("qft_20.circ"))
    _same(Q.gen_qft(10, 717), gio.read_circuit("qft_10_717.circ"))
    _same(Q.gen_hea(8, 3, 5), gio.read_circuit("hea_8_3_5.circ"))
    _same(Q.gen_hea(24, 10, 2024), gio.read_circuit("hea_24_10_2024.circ"))


FUSE = gio.cases("fuse")


@pytest.mark.parametrize("c", FUSE, ids=[c["name"] for c in FUSE])
def test_reference_mode_fusion_reproduces_fuse_circuit(c):
    # fusion.hpp:20-133 restated in csrc/fusion.cpp: same blocks, same order,
    # matrices equal up to matmul rounding.
    src = gio.read_circuit(c["name"] + ".in.circ")
    want = gio.read_circuit(c["name"] + ".circ")
    p = Q.Program(src.qubits, 0)
    for g in src.gates:
        p.add(Q.Gate(Q.GateKind(g.kind), g.targets, g.params, g.controls, g.dagger, g.matrix))
    got = Q.fuse_circuit(p, c["k"]).gates()
    assert len(got) == c["blocks"] == len(want.gates)
    for a, b in zip(got, want.gates):
        assert int(a.kind) == b.kind and list(a.targets) == b.targets and list(a.controls) == b.controls
        if b.matrix is not None:
            assert np.max(np.abs(a.matrix - b.matrix)) <= 1e-13
        else:
            assert list(a.params) == b.params


def test_planner_runs_host_side_and_fuses_passes():
    # Planning is pure host C++: passes << gates for the bench workloads.
    p = Q.gen_random_circuit(30, 20, 424242)
    cc = Q.CompiledCircuit(30, p.gates())
    st = cc.stats()
    assert st["gates"] == 1200
    assert st["passes"] < 120, st
    unf = Q.CompiledCircuit(30, p.gates(), plan=N.QS_PLAN_UNFUSED).stats()
    assert unf["passes"] == 1200
    qft = Q.CompiledCircuit(30, Q.gen_qft(30, 12345).gates()).stats()
    assert qft["passes"] <= 8, qft
    dense = Q.CompiledCircuit(28, Q.gen_random_circuit(28, 20, 424242).gates(),
                              plan=N.QS_PLAN_DENSE_FUSION, max_fused_qubits=3).stats()
    assert dense["passes"] < 1120


def test_plan_tile_info_describes_the_random30_passes():
    # qs_plan_tile_info: every pass of the bench plan holds the 4 resident low
    # qubits, 13 tile qubits, 4 or 5 register bits, <= 3 exchanges, and the
    # passes together cover the layer's gates (3 passes per layer)
    L = N.lib()
    cc = Q.CompiledCircuit(30, Q.gen_random_circuit(30, 20, 424242).gates())
    st = cc.stats()
    covered = 0
    for i in range(st["launches"]):
        m, r, tr, nops = N.C.c_uint32(), N.C.c_uint32(), N.C.c_uint32(), N.C.c_uint32()
        gates = N.C.c_uint64()
        qs = (N.C.c_uint32 * 16)()
        N.check(L.qs_plan_tile_info(cc._h, i, N.C.byref(m), qs, N.C.byref(r), N.C.byref(tr), N.C.byref(nops),
                                    N.C.byref(gates)))
        assert m.value == 13
        q = list(qs)[:13]
        assert q == sorted(q) and q[:4] == [0, 1, 2, 3]
        assert r.value in (4, 5) and tr.value <= 3 and nops.value > 0
        covered += gates.value
    assert st["launches"] == 58
    assert 1100 <= covered <= 1200
    with pytest.raises(Q.ValidationError):
        N.check(L.qs_plan_tile_info(cc._h, 10 ** 6, None, None, None, None, None, None))


def test_validation_errors_without_gpu():
    bad = [Q.make_gate(Q.GateKind.H, [7])]
    with pytest.raises(Q.ValidationError):
        Q.CompiledCircuit(4, bad)
    dup = [Q.make_gate(Q.GateKind.CNOT, [1, 1])]
    with pytest.raises(Q.ValidationError):
        Q.CompiledCircuit(4, dup)
    nonu = [Q.make_custom_gate([0, 1], np.ones((4, 4)))]
    with pytest.raises(Q.ValidationError):
        Q.CompiledCircuit(4, nonu)
    with pytest.raises(Q.ValidationError):
        Q.SimOptions(max_fused_qubits=9).validate()
    p = Q.Program(2, 0)
    p.add(Q.make_gate(Q.GateKind.RX, [0]))  # missing parameter
    with pytest.raises(Q.ValidationError):
        Q.validate_or_throw(p)


_JIT_PROBE = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2212_14201_b200 import _native as N, qforge as Q
cc = Q.CompiledCircuit(16, Q.gen_random_circuit(16, 3, 7).gates())
a = [N.C.c_uint64() for _ in range(3)]
N.check(N.lib().qs_jit_stats(*[N.C.byref(x) for x in a]))
print(json.dumps({"stats": cc.stats(), "jit": [x.value for x in a]}))
"""


def test_jit_disk_cache_serves_a_cold_process(tmp_path):
    """NVRTC output is cached on disk (QSB_JIT_CACHE): a second, fresh process
    planning the same circuit shape builds nothing and loads every tile cubin
    from the cache (the cold-start path of run(), VERDICT r1 item 'cold path')."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, QSB_JIT_CACHE=str(tmp_path / "jit"))
    outs = []
    for _ in range(2):
        r = subprocess.run([sys.executable, "-c", _JIT_PROBE % ROOT], capture_output=True, text=True, env=env,
                           timeout=600)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    first, second = outs
    assert first["stats"] == second["stats"]
    assert first["jit"][0] > 0 and first["jit"][2] == 0     # built with NVRTC, nothing on disk yet
    assert second["jit"][0] == 0                            # nothing rebuilt ...
    assert second["jit"][2] == first["jit"][0]              # ... every module came from disk
    assert len(list((tmp_path / "jit").glob("*.qsbcubin"))) == first["jit"][0]


def test_run_plan_mode_matches_the_cpp_facade():
    """Python run() picks the plan the C++ facade's run() picks
    (include/qforge/simulator.hpp: dense fusion only when asked for by plan)."""
    assert Q.run_plan_mode(Q.SimOptions()) == N.QS_PLAN_TILED
    assert Q.run_plan_mode(Q.SimOptions(fusion_enabled=True)) == N.QS_PLAN_TILED
    assert Q.run_plan_mode(Q.SimOptions(fusion_enabled=True, plan=N.QS_PLAN_DENSE_FUSION)) == N.QS_PLAN_DENSE_FUSION
    assert Q.run_plan_mode(Q.SimOptions(plan=N.QS_PLAN_UNFUSED)) == N.QS_PLAN_UNFUSED
    src = open(os.path.join(ROOT, "paper_2212_14201_b200", "include", "qforge", "simulator.hpp")).read()
    assert "(opts.fusion_enabled && opts.plan == QS_PLAN_DENSE_FUSION) ? QS_PLAN_DENSE_FUSION" in src
