"""Times the exact-scan chains (serial checksum digest, exact sampler) at n
qubits on a random state; run under ncu for the per-kernel split:
    ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none \
        --csv --log-file out.csv python tools/scan_probe.py --n 28"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
sv = Q.StateVector(a.n)
sv.apply_circuit(Q.gen_random_circuit(a.n, 1, 7).gates())
for name, fn in (("checksum_serial", lambda: sv.checksum_serial()),
                 ("sample_seeded 1e6 exact", lambda: sv.sample_seeded(3, 1000000, True))):
    fn()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(json.dumps({"probe": name, "n": a.n, "wall_ms": [round(t, 3) for t in ts]}), flush=True)
