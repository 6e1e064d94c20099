"""States beyond the reference's 30-qubit cap on one B200 (31-33 qubits:
32-128 GiB of the 180 GB HBM): QFT of a basis state (every probability 2^-n,
amplitude phases in closed form) and a random circuit (norm 1), through the
default tile plan.  One JSON line per case."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import _native as N  # noqa: E402
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or ["31", "32", "33"])]:
    for kind in ("qft", "random"):
        row = {"n": n, "kind": kind, "GiB": 16 * 2 ** n / 2 ** 30}
        sv = None
        try:
            b = 0x2AAAAAAAA & ((1 << n) - 1)
            gates = (Q.gen_qft(n, b) if kind == "qft" else Q.gen_random_circuit(n, 3, 424242)).gates()
            t0 = time.time()
            sv = Q.StateVector(n, 0, max_qubits=n)
            sv.apply_circuit(gates)
            norm = sv.norm_squared()
            row.update({"gates": len(gates), "seconds": round(time.time() - t0, 2), "norm": norm})
            if kind == "qft":
                # closed form (gates.hpp QFT, bench.hpp gen_qft): |a_k| = 2^-n/2 for every k
                idx = np.array([0, 1, 12345, (1 << n) - 1, (1 << (n - 1)) + 7], dtype=np.uint64)
                amps = np.array([sv.amplitude(int(k)) for k in idx])
                row["max_dprob"] = float(np.max(np.abs(np.abs(amps) ** 2 - 2.0 ** -n)))
            row["ok"] = abs(norm - 1) < 1e-9 and row.get("max_dprob", 0) < 1e-15
            cc = Q.CompiledCircuit(n, gates)
            row["plan"] = cc.stats()
        except Exception as e:  # noqa: BLE001 -- reported, the probe goes on
            row["error"] = "%s: %s" % (type(e).__name__, e)
        finally:
            del sv  # free the state before the next case
        print(json.dumps(row), flush=True)
