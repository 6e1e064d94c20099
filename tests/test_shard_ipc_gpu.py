"""The multi-process sharded data path on ONE B200:
2 and 4 processes, each holding one shard of a 16-qubit state on cuda:0,
exchange rank bits through CUDA-IPC peer memory -- the scatter kernel and the
tile pass with the exchange fused into its stores, writing into the OTHER
processes' buffers -- with torch.distributed (gloo) as the host barrier /
all-gather (qs_dist_create_host; NCCL refuses two ranks on one device).
Every rank's shard, reductions, samples and Pauli expectations are checked
against the C oracle.  Kernels never wait on another rank (barriers are on
the host, after each rank drained its stream), so sharing one GPU is safe."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib as ol
from test_planner_emu import mixed_gates
from paper_2212_14201_b200 import qforge as Q

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,fuse", [(2, "1"), (4, "1"), (2, "0")])
def test_ipc_exchanges_across_processes_match_oracle(tmp_path, world, fuse):
    port = str(free_port())
    outs = [str(tmp_path / ("r%d.npz" % r)) for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "shard_ipc_worker.py"), str(r), str(world), port,
                               outs[r], fuse], stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(world)]
    errs = []
    for p in procs:
        try:
            _, e = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        errs.append((p.returncode, e[-2000:]))
    assert all(rc == 0 for rc, _ in errs), errs
    res = [np.load(o) for o in outs]
    n = 16
    cases = {"random": Q.gen_random_circuit(n, 6, 424242).gates(), "qft": Q.gen_qft(n, 0x2D5).gates(),
             "hea": Q.gen_hea(n, 3, 11).gates(), "mixed": mixed_gates(n, 200, 91)}
    words = ["Z" * n, "X" + "I" * (n - 2) + "X", "I" * (n - 1) + "Y", "Y" + "Z" * (n - 2) + "X"]
    for name, gates in cases.items():
        want = ol.run_gates(n, gates)
        got = np.zeros(1 << n, dtype=np.complex128)
        for r in res:
            lo, hi = r[name + "_range"]
            got[lo:hi] = r[name + "_amps"]
        assert np.max(np.abs(got - want)) <= 1e-10, name
        for r in res:  # reductions summed in rank order: identical on every rank
            assert abs(r[name + "_cs"][0] - ol.checksum(want, n)) <= 1e-12 * (1 << n)
            assert abs(r[name + "_cs"][1] - 1.0) <= 1e-12
            assert np.max(np.abs(r[name + "_probs"] - ol.probs(want, n, [n - 1, 3, n - 2, 0]))) <= 1e-12
            assert np.array_equal(r[name + "_samples"], ol.sample_seeded(want, n, 7, 4000))
        ex = np.array([complex(*ol.expectation(want, n, [(w, 1.0)])) for w in words])
        for r in res:
            assert np.max(np.abs(r[name + "_pauli"] - ex)) <= 1e-11, name  # sums of 2^n terms
        for r in res[1:]:
            assert np.array_equal(r[name + "_cs"], res[0][name + "_cs"])

