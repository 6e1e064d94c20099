"""Every non-tile kernel of libqsb on a 2^n state (default n = 28, 4 GiB):
device time from CUDA events on the state's stream (median of `--reps`),
algorithmic bytes per launch, GB/s and the fraction of the measured HBM copy
bandwidth (MEASURED_PEAKS.json).  One JSON line per kernel.

Under ncu (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,...`) the
same script gives the per-launch DRAM traffic of each kernel (VERDICT r1 item
"ncu evidence for every kernel choice"); run it with `--reps 1` there.

    python tools/kernel_probe.py [--n 28] [--reps 5]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2212_14201_b200 import _native as N  # noqa: E402
from paper_2212_14201_b200 import qforge as Q  # noqa: E402
from paper_2212_14201_b200.sharded import ShardedState  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n, reps = a.n, a.reps
A = 1 << n  # amplitudes
try:
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6650.0
L = N.lib()
sv = Q.StateVector(n)
sv.apply_circuit(Q.gen_random_circuit(n, 1, 7).gates())  # a dense state
dev = torch.device("cuda", 0)


def stream_of(h, sharded=False):
    return torch.cuda.ExternalStream(L.qs_shards_stream(h) if sharded else L.qs_stream(h), device=dev)


def timeit(name, fn, bytes_per_launch, launches=1, h=None, sharded=False, note=""):
    st = stream_of(h if h is not None else sv.handle(), sharded)
    fn()  # warm-up (JIT, scratch allocation)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / launches)
    ms = statistics.median(ts)
    gbs = bytes_per_launch / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": name, "n": n, "ms": round(ms, 4), "bytes": bytes_per_launch, "GBps": round(gbs, 1),
                      "frac": round(gbs / PEAK, 3), "note": note}), flush=True)


G = Q.GateKind
rng = np.random.default_rng(1)


def unitary(k):
    z = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def gate(kind, targets, params=(), controls=()):
    g = Q.make_gate(kind, targets, params)
    g.controls = list(controls)
    return g


# --- per-gate kernels (statevector.hpp:268-361): 32 B per touched amplitude
for q in (0, n // 2, n - 1):
    timeit("k_mat1 H q%d" % q, lambda q=q: sv.apply_gate(gate(G.H, [q])), 32 * A,
           note="256-bit pair kernel k_mat1_q0" if q == 0 else "")
os.environ["QSB_NO_PAIR256"] = "1"
timeit("k_mat1 H q0 (QSB_NO_PAIR256)", lambda: sv.apply_gate(gate(G.H, [0])), 32 * A)
os.environ.pop("QSB_NO_PAIR256")
timeit("k_mat1 U3 ctrl", lambda: sv.apply_gate(gate(G.U3, [5], (0.1, 0.2, 0.3), [n - 2])), 16 * A,
       note="one control: half the amplitudes")
timeit("k_diag RZ", lambda: sv.apply_gate(gate(G.RZ, [n // 3], (0.7,))), 32 * A)
timeit("k_diag RZ q0", lambda: sv.apply_gate(gate(G.RZ, [0], (0.7,))), 32 * A, note="256-bit pair kernel k_diag_q0")
timeit("k_diag Z (skip_zero)", lambda: sv.apply_gate(gate(G.Z, [n // 3])), 16 * A, note="bit-set half only")
timeit("k_flip X", lambda: sv.apply_gate(gate(G.X, [n - 3])), 32 * A)
timeit("k_flip CNOT", lambda: sv.apply_gate(gate(G.CNOT, [2, n - 4])), 16 * A, note="control: half")
timeit("k_swap SWAP", lambda: sv.apply_gate(gate(G.SWAP, [1, n - 1])), 16 * A, note="pairs with differing bits: half")
for k in (2, 3, 4, 5):
    m = unitary(k)
    for tg in ([n - 1 - 3 * i for i in range(k)], list(range(k - 1, -1, -1))):
        # default selection, then each form forced (QSB_DENSE_FORM)
        for form in ("", "g", "g-nopair", "lanes"):
            if form:
                os.environ["QSB_DENSE_FORM"] = form.split("-")[0]
            if form.endswith("nopair"):
                os.environ["QSB_NO_PAIR256"] = "1"
            timeit("k_dense K=%d t=%s form=%s" % (k, tg, form or "default"),
                   lambda tg=tg, m=m: sv.apply_matrix(tg, m), 32 * A)
            os.environ.pop("QSB_DENSE_FORM", None)
            os.environ.pop("QSB_NO_PAIR256", None)
m6 = unitary(6)
timeit("k_dense_wide K=6", lambda: sv.apply_matrix([n - 1, n - 3, 7, 5, 3, 1], m6), 32 * A,
       note="correctness path for blocks wider than the fusion cap")

# --- reductions (statevector.hpp:110-215): 16 B per amplitude read
timeit("k_reduce norm2", lambda: sv.norm_squared(), 16 * A)
timeit("k_reduce checksum", lambda: sv.checksum(), 16 * A)
timeit("k_reduce prob_one", lambda: sv.probability_of_one(n - 1), 8 * A, note="reads the bit-set half")
timeit("k_marginal_runs 6 qubits", lambda: sv.probabilities([n - 1, 17, 13, 5, 1, 0]), 16 * A)
os.environ["QSB_MARGINAL_LANES"] = "1"
timeit("k_marginal_lanes 6 qubits (QSB_MARGINAL_LANES)", lambda: sv.probabilities([n - 1, 17, 13, 5, 1, 0]), 16 * A)
os.environ.pop("QSB_MARGINAL_LANES")
cnt = 1 << 24
buf = np.empty(cnt, dtype=np.float64)
timeit("k_probs (2^24 window)", lambda: N.check(L.qs_probs_full(sv.handle(), N.dptr(buf), 0, cnt)), 24 * cnt,
       note="includes the 128 MiB device->host copy")

# --- exact sampler chain (statevector.hpp:542-570): k_probs, k_chunk_sum,
# k_scan_estimate, k_chunk_ints, k_sequential, k_expand, k_search
timeit("sampler chain 1e6 shots (exact)", lambda: sv.sample_seeded(3, 1000000, True), 16 * A + 8 * A * 6,
       note="bytes: state read + ~6 sweeps of the 8 B/amplitude arrays")
timeit("checksum_serial (exact serial digest)", lambda: sv.checksum_serial(), 16 * A + 8 * A * 4)

# --- Pauli expectation (variational.hpp:33-47): one read pass per X-group
words = ["Z" * n, "I" * (n - 2) + "XX", "Y" + "I" * (n - 2) + "Y", "I" * (n // 2) + "ZZ" + "I" * (n - n // 2 - 2)]
timeit("k_pauli_group (4 terms, 3 X-groups)", lambda: sv.expect_pauli(words), 16 * A * 3, note="3 groups")

# --- out-of-place qubit permutation (QFT's absorbed SWAPs, not folded)
os.environ["QSB_FOLD_PERM"] = "0"
qft = Q.gen_qft(n, 0).gates()
cc = Q.CompiledCircuit(n, qft)
steps = cc.stats()["launches"]
os.environ.pop("QSB_FOLD_PERM")
tbuf = (N.C.c_float * steps)()
N.check(L.qs_plan_execute_timed(sv.handle(), cc._h, tbuf))
N.check(L.qs_plan_execute_timed(sv.handle(), cc._h, tbuf))
print(json.dumps({"kernel": "k_permute (QFT final SWAPs, QSB_FOLD_PERM=0)", "n": n, "ms": round(tbuf[steps - 1], 4),
                  "bytes": 32 * A, "GBps": round(32 * A / (tbuf[steps - 1] / 1e3) / 1e9, 1),
                  "frac": round(32 * A / (tbuf[steps - 1] / 1e3) / 1e9 / PEAK, 3),
                  "note": "last step of the plan, CUDA events between steps"}), flush=True)
del cc, sv
torch.cuda.empty_cache()

# --- sharded exchange (peer scatter, 8 local shards): 32 B per amplitude
os.environ["QSB_SHARD_EXCHANGE"] = "peer"
st = ShardedState.local(n, 3)
os.environ.pop("QSB_SHARD_EXCHANGE")
st.apply_circuit(Q.gen_random_circuit(n, 1, 9).gates())
for fuse in ("1", "0"):
    os.environ["QSB_FUSE_EXCHANGE"] = fuse
    for g in (1, 2, 3):
        gl = [gate(G.H, [n - 1 - i]) for i in range(g)]
        timeit("%s %d rank bit(s)" % ("exchange-fused tile pass" if fuse == "1" else "k_scatter_exchange", g),
               lambda gl=gl: st.apply_circuit(gl), 32 * A * (2 if fuse == "1" else 3), h=st.handle(), sharded=True,
               note="one step = exchange + H pass + restore exchange; bytes = its HBM sweeps "
                    "(fused: 2, separate: 3; see the launch list per kernel)")
os.environ.pop("QSB_FUSE_EXCHANGE")
st.close()
