"""Sharded state vectors on the GPU.

All 2^g shards live on one B200 (ShardedState.local): the plans, tile passes
with rank bits, and half-shard exchanges are exactly those a distributed run
executes, only the exchange transport differs (device-local swap instead of
NCCL/peer-memory transfers; those kernels are covered by
test_distributed_exchange_paths_match_oracle).  Results are compared with the C oracle and
with the unsharded tile path."""
import numpy as np
import pytest

import oracle_lib as ol
from test_planner_emu import mixed_gates
from paper_2212_14201_b200 import _native as N
from paper_2212_14201_b200 import qforge as Q
from paper_2212_14201_b200.sharded import ShardedCircuit, ShardedState

pytestmark = pytest.mark.gpu

TOL = 1e-10


def workload(which, n):
    return {"random": lambda: Q.gen_random_circuit(n, 6, 424242),
            "qft": lambda: Q.gen_qft(n, 0x2d5 % (1 << n)),
            "hea": lambda: Q.gen_hea(n, 3, 11),
            "ghz": lambda: Q.gen_ghz(n)}[which]().gates()


@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("which", ["random", "qft", "hea", "ghz"])
def test_sharded_workloads_match_oracle(which, g):
    n = 16
    gates = workload(which, n)
    want = ol.run_gates(n, gates)
    st = ShardedState.local(n, g)
    circ = ShardedCircuit(n, g, gates)
    st.execute(circ)
    got = st.amplitudes()
    assert np.max(np.abs(got - want)) <= TOL
    assert abs(st.norm_squared() - ol.norm2(want, n)) <= 1e-12
    assert abs(st.checksum() - ol.checksum(want, n)) <= 1e-12 * (1 << n)
    if which in ("random", "hea"):
        assert circ.stats()["exchanges"] > 0


@pytest.mark.parametrize("g", [1, 2, 3])
@pytest.mark.parametrize("n", [13, 15])
def test_sharded_mixed_gates_from_random_state(n, g):
    gates = mixed_gates(n, 250, 77 + n + g)
    rng = np.random.default_rng(n * 10 + g)
    a0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    a0 /= np.linalg.norm(a0)
    want = ol.run_gates(n, gates, state=a0.copy())
    st = ShardedState.local(n, g)
    st.set_amplitudes(a0, 0)
    st.apply_circuit(gates)
    got = st.amplitudes(0, 1 << n)
    assert np.max(np.abs(got - want)) <= TOL


def test_sharded_matches_unsharded_bitwise_close():
    n = 20
    gates = workload("random", n)
    sv = Q.StateVector(n)
    sv.apply_circuit(gates, N.QS_PLAN_TILED)
    ref = sv.amplitudes()
    for g in (1, 3):
        st = ShardedState.local(n, g)
        st.apply_circuit(gates)
        assert np.max(np.abs(st.amplitudes() - ref)) <= 1e-12


def test_basis_state_and_partial_io():
    n, g = 12, 2
    st = ShardedState.local(n, g)
    st.reset(3 << (n - g) | 5)
    a = st.amplitudes()
    assert a[(3 << (n - g)) | 5] == 1 and np.count_nonzero(a) == 1
    # a range spanning a shard boundary
    off = (1 << (n - g)) - 7
    vals = np.arange(20) + 1j
    st.set_amplitudes(vals, off)
    assert np.array_equal(st.amplitudes(off, 20), vals)


def test_sharded_errors():
    n = 12
    gates = workload("qft", n)
    with pytest.raises(Q.ValidationError):
        ShardedState.local(n, 0)
    with pytest.raises(Q.ValidationError):
        ShardedState.local(8, 3)  # fewer than 6 local qubits
    st = ShardedState.local(n, 2)
    with pytest.raises(Q.ValidationError):
        st.execute(ShardedCircuit(n, 1, gates))  # plan for another shape
    plain = Q.StateVector(n)
    sharded_plan = ShardedCircuit(n, 2, gates)
    with pytest.raises(Q.ValidationError):
        N.check(N.lib().qs_plan_execute(plain.handle(), sharded_plan.handle()))
    with pytest.raises(Q.ValidationError):
        st.amplitudes(1 << n, 1)


def qft_closed_form(n, x, idx):
    """QFT|x> amplitude at basis indices idx: exp(2 pi i x k / 2^n) / 2^(n/2)."""
    N_ = np.uint64(1 << n)
    ph = (np.uint64(x) * idx.astype(np.uint64)) % N_
    return np.exp(2j * np.pi * ph.astype(np.float64) / float(1 << n)) / np.sqrt(float(1 << n))


@pytest.mark.parametrize("from_basis", [False, True])
@pytest.mark.parametrize("n,g", [(26, 3), (30, 3)])
def test_sharded_qft_closed_form_large(n, g, from_basis):
    """QFT|x> by X gates + QFT, or QFT run from the basis state x (the leading
    all-to-all folded into the start index, reset fused, zero tiles skipped)."""
    x = 0x2A5A5A5 & ((1 << n) - 1)
    st = ShardedState.local(n, g)
    if from_basis:
        st.execute(ShardedCircuit(n, g, Q.gen_qft(n, 0).gates()), from_basis=x)
    else:
        st.execute(ShardedCircuit(n, g, Q.gen_qft(n, x).gates()))
    assert abs(st.norm_squared() - 1.0) <= 1e-10
    size = 1 << n
    rng = np.random.default_rng(5)
    for off in [0, size // 2 - 4096, size - 8192] + [int(v) for v in rng.integers(0, size - 8192, 5)]:
        got = st.amplitudes(off, 8192)
        want = qft_closed_form(n, x, np.arange(off, off + 8192))
        assert np.max(np.abs(got - want)) <= TOL


@pytest.mark.parametrize("mode", ["staged", "peer"])
@pytest.mark.parametrize("g", [1, 2, 3])
def test_distributed_exchange_paths_match_oracle(monkeypatch, g, mode):
    """The distributed transports' data paths on one GPU.  staged: the NCCL
    fallback's pack -> staging buffer -> unpack kernels (chunked; only the
    send/recv is replaced by a device copy).  peer: the peer-memory scatter
    kernel writing every amplitude into its owner's second buffer (sibling
    shards here, NVLink peers over CUDA IPC in a distributed run)."""
    monkeypatch.setenv("QSB_SHARD_EXCHANGE", mode)
    monkeypatch.setenv("QSB_SHARD_CHUNK", "4096")  # force several chunks per exchange
    n = 15
    gates = mixed_gates(n, 200, 4242 + g)
    rng = np.random.default_rng(3)
    a0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    a0 /= np.linalg.norm(a0)
    want = ol.run_gates(n, gates, state=a0.copy())
    st = ShardedState.local(n, g)
    st.set_amplitudes(a0, 0)
    circ = ShardedCircuit(n, g, gates)
    assert circ.stats()["exchanges"] >= 1
    if g > 1:
        assert max(len(gp) for k, gp, _ in circ.steps() if k == 2) > 1  # multi-bit all-to-all
    st.execute(circ)
    assert np.max(np.abs(st.amplitudes() - want)) <= TOL
    assert abs(st.norm_squared() - 1.0) <= 1e-12


def test_nccl_single_rank_communicator():
    """The distributed handle through NCCL (world 1: no exchanges, but libnccl
    loading, communicator setup and the rank-ordered allgather reductions run)."""
    from paper_2212_14201_b200.sharded import DistComm

    comm = DistComm(DistComm.unique_id(), 1, 0, 0)
    n = 14
    gates = workload("random", n)
    st = ShardedState.distributed(n, comm)
    st.execute(ShardedCircuit(n, 0, gates))
    want = ol.run_gates(n, gates)
    assert np.max(np.abs(st.amplitudes() - want)) <= TOL
    assert abs(st.norm_squared() - 1.0) <= 1e-12
    assert abs(st.checksum() - ol.checksum(want, n)) <= 1e-12 * (1 << n)
    # the host gate-list path plans for shards too (no permutation steps):
    # QFT's final SWAPs on a one-rank world
    qft = workload("qft", n)
    st.reset(0)
    st.apply_circuit(qft)
    assert np.max(np.abs(st.amplitudes() - ol.run_gates(n, qft))) <= TOL
    st.run_circuit(gates, basis=5)  # run() from |5>: reset fused, lazy zeros
    want5 = ol.run_gates(n, gates, state=np.eye(1, 1 << n, 5, dtype=np.complex128)[0])
    assert np.max(np.abs(st.amplitudes() - want5)) <= TOL
    st.close()
    comm.close()


def test_checksum_invariant_across_shard_counts():
    """SURVEY 8(d) config 4 parity: the 30-qubit random circuit's checksum does
    not depend on the number of shards (P = 1, 2, 4, 8), nor on the transport."""
    import os
    n = 30
    gates = Q.gen_random_circuit(n, 20, 424242).gates()
    sv = Q.StateVector(n)
    sv.apply_circuit(gates)
    ref = sv.checksum()
    probe = sv.amplitudes(12345678, 4096)
    del sv
    for g, mode in [(1, "swap"), (2, "peer"), (3, "swap"), (3, "peer")]:
        os.environ["QSB_SHARD_EXCHANGE"] = mode
        try:
            st = ShardedState.local(n, g)
        finally:
            del os.environ["QSB_SHARD_EXCHANGE"]
        st.run_circuit(gates) if mode == "peer" else st.apply_circuit(gates)
        assert abs(st.checksum() - ref) <= 1e-12 * (1 << n)
        assert np.max(np.abs(st.amplitudes(12345678, 4096) - probe)) <= 1e-12
        st.close()


@pytest.mark.parametrize("g", [1, 2, 3])
def test_sharded_reductions_match_oracle(g):
    """Marginals (incl. rank-bit qubits), exact sampling across shard
    boundaries, and Pauli expectations with X/Y on rank bits, all against the
    oracle evaluated on the same amplitudes."""
    n = 16
    st = ShardedState.local(n, g)
    st.apply_circuit(workload("random", n))
    a = st.amplitudes(0, 1 << n)
    rng = np.random.default_rng(40 + g)
    for qs in ([n - 1, 0, 5], [n - 2, n - 1], list(rng.permutation(n)[:7]), [3]):
        want = ol.probs(a, n, list(map(int, qs)))
        assert np.max(np.abs(st.probabilities(qs) - want)) <= 1e-12
    for seed in (0, 7, 123):
        got = st.sample_seeded(seed, 20000, exact=True)
        assert np.array_equal(got, ol.sample_seeded(a, n, seed, 20000))
    words = []
    for _ in range(12):
        words.append("".join(rng.choice(list("IXYZ"), size=n)))
    words.append("I" * (n - 1) + "X")           # X on the top (rank) qubit
    words.append("Z" + "I" * (n - 2) + "Y")
    got = st.expect_pauli(words)
    for w, v in zip(words, got):
        re, im = ol.expectation(a, n, [(w, 1.0)])
        assert abs(v.real - re) <= 1e-12 and abs(v.imag - im) <= 1e-12


def test_sharded_sampling_matches_unsharded_30q():
    """30 qubits, 8 shards: exact sampling over the chained cumulative sum gives
    the same indices as the unsharded GPU sampler (which is pinned to the
    reference's serial loop)."""
    n = 30
    gates = Q.gen_random_circuit(n, 4, 9).gates()
    sv = Q.StateVector(n)
    sv.apply_circuit(gates)
    ref = sv.sample_seeded(5, 100000, exact=True)
    del sv
    st = ShardedState.local(n, 3)
    st.apply_circuit(gates)
    assert np.array_equal(st.sample_seeded(5, 100000, exact=True), ref)


@pytest.mark.parametrize("kind", ["qft", "random", "hea", "ghz"])
@pytest.mark.parametrize("g", [1, 3])
def test_sharded_execute_from_basis(g, kind):
    """Runs from a basis state: exchanges before the first pass are folded
    into the start index, the reset into the first pass, zero tiles skipped."""
    n = 15
    gates = workload(kind, n)
    circ = ShardedCircuit(n, g, gates)
    for b in (0, (1 << n) - 1, 0x2C3A):
        st = ShardedState.local(n, g)
        st.reset(b)
        st.execute(circ)
        want = st.amplitudes()
        st2 = ShardedState.local(n, g)
        st2.set_amplitudes(np.full(1 << n, np.nan + 0.25j), 0)  # stale: must be overwritten (lazy zeros)
        st2.execute(circ, from_basis=b)
        got = st2.amplitudes()
        assert np.all(np.isfinite(got))
        assert np.max(np.abs(got - want)) <= 1e-14
