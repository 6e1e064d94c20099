"""Small driver for ncu captures: plans a workload once and executes it
`--reps` times on cuda:0 (no timing; use bench.py for numbers)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import _native as N  # noqa: E402
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=26)
ap.add_argument("--workload", default="random", choices=["random", "qft", "hea"])
ap.add_argument("--plan", default="tiled", choices=["tiled", "dense", "unfused"])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
gen = {"random": lambda n: Q.gen_random_circuit(n, 20, 424242), "qft": lambda n: Q.gen_qft(n, 12345),
       "hea": lambda n: Q.gen_hea(n, 10, 2024)}[a.workload]
plan = {"tiled": N.QS_PLAN_TILED, "dense": N.QS_PLAN_DENSE_FUSION, "unfused": N.QS_PLAN_UNFUSED}[a.plan]
p = gen(a.n)
cc = Q.CompiledCircuit(a.n, p.gates(), plan=plan)
sv = Q.StateVector(a.n)
for _ in range(a.reps):
    sv.reset()
    cc.execute(sv)
print("ok", cc.stats(), "checksum", sv.checksum())
