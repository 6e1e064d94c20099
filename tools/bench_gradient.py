"""Times gradient() on the config-5 ansatz (HEA(24, 10): 480 rotation slots,
H = sum Z_i Z_{i+1} + 0.5 sum X_i, 47 terms) on cuda:0: adjoint gradient
(qs_gradient) vs the reference's shift rule evaluated with the GPU
expectation() (two runs per slot; timed on a sample of slots and scaled)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

n, layers = 24, 10
pc = Q.ParamCircuit(n)
for l in range(layers):
    for q in range(n):
        pc.add_param(Q.GateKind.RY, q, "y%d_%d" % (l, q))
        pc.add_param(Q.GateKind.RZ, q, "z%d_%d" % (l, q))
    for q in range(n - 1):
        pc.add(Q.GateKind.CNOT, [q, q + 1])
terms = {"Z%d Z%d" % (i, i + 1): 1.0 for i in range(n - 1)}
terms.update({"X%d" % i: 0.5 for i in range(n)})
H = Q.PauliOperator(terms)
rng = np.random.default_rng(2024)
at = {nm: float(rng.uniform(0, 6.28)) for nm in pc.parameter_names()}

g = Q.gradient(pc, H, at)  # warm-up (planning, JIT)
t0 = time.perf_counter()
reps = 3
for _ in range(reps):
    g = Q.gradient(pc, H, at)
adj = (time.perf_counter() - t0) / reps

sample = 8
t0 = time.perf_counter()
shift = []
for idx, (bi, nm) in enumerate(pc.slots[:sample]):
    acc = 0.0
    for sgn in (1, -1):
        p = pc.bind(at)
        p.body[bi].params = [p.body[bi].params[0] + sgn * np.pi / 2]
        acc += 0.5 * sgn * Q.expectation(p, H)
    shift.append(acc)
per_slot = (time.perf_counter() - t0) / sample
err = max(abs(a - b) for a, b in zip(g[:sample], shift))
print({"slots": len(pc.slots), "terms": len(terms), "adjoint_s": round(adj, 4),
       "shift_rule_gpu_s_est": round(per_slot * len(pc.slots), 2), "speedup": round(per_slot * len(pc.slots) / adj, 1),
       "max_abs_diff_first_%d" % sample: err})

# Config 5's sampling sweep: the bound ansatz with every qubit measured,
# run(p, seed=s, 10^6 shots) for s = 0..9 (trailing measurements: one state
# evolution + the exact serial-equivalent sampler on the device).
prog = Q.Program(n, n)
prog.body.extend(pc.bind(at).body)
for q in range(n):
    prog.measure(q, q)
Q.run(prog, Q.SimOptions(seed=0), 1000)  # warm-up
t0 = time.perf_counter()
keys = 0
for s in range(10):
    r = Q.run(prog, Q.SimOptions(seed=s), 1_000_000)
    keys += len(r.counts)
sweep = time.perf_counter() - t0
print({"sampling_sweep": "10 seeds x 1e6 shots, 24 qubits measured", "seconds": round(sweep, 3),
       "per_run_s": round(sweep / 10, 4), "distinct_keys_total": keys})
