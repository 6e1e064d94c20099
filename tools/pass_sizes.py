"""Diagnostic: average tile-pass time of the random layered circuit vs state
size (L2-resident at <= 2^22 amplitudes, HBM-bound above), per-pass times from
CUDA events between passes (qs_plan_execute_timed)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import _native as N  # noqa: E402
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

sizes = [int(x) for x in (sys.argv[1:] or ["20", "21", "22", "23", "24", "26", "28", "30"])]
for n in sizes:
    gates = Q.gen_random_circuit(n, 20, 424242).gates()
    cc = Q.CompiledCircuit(n, gates)
    sv = Q.StateVector(n)
    st = cc.stats()
    L = N.lib()
    buf = (N.C.c_float * st["launches"])()
    tot = None
    reps = 3
    for r in range(reps + 1):
        sv.reset()
        N.check(L.qs_plan_execute_timed(sv.handle(), cc._h, buf))
        if r:
            t = list(buf)
            tot = t if tot is None else [a + b for a, b in zip(tot, t)]
    per = [x / reps for x in tot]
    avg = sum(per) / len(per)
    print(json.dumps({"n": n, "m": os.environ.get("QSB_TILE_M", "auto"), "passes": st["passes"],
                      "avg_pass_us": round(avg * 1e3, 2), "GBps_rw": round(32 * 2 ** n / (avg * 1e-3) / 1e9, 1),
                      "min_us": round(min(per) * 1e3, 2), "max_us": round(max(per) * 1e3, 2)}), flush=True)
