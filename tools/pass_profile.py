"""Per-pass profile of one random30 (or other) bench step: CUDA-event time of
every launch on the exact bench path (from |0..0>, zero-tile skipping, fused
checksum), with the tile's qubits, register bits, shared-memory exchanges and
micro-op count.  One JSON line per launch.
    python tools/pass_profile.py [--n 30] [--workload random]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import _native as N  # noqa: E402
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--workload", default="random", choices=["random", "qft"])
a = ap.parse_args()
g = (Q.gen_random_circuit(a.n, 20, 424242) if a.workload == "random" else Q.gen_qft(a.n, 0x2AAAAAAA)).gates()
L = N.lib()
cc = Q.CompiledCircuit(a.n, g)
k = cc.stats()["launches"]
sv = Q.StateVector(a.n)
ms, by = (N.C.c_float * k)(), (N.C.c_double * k)()
cs = N.C.c_double()
for _ in range(3):  # the last one is reported (JIT variants built by the first)
    N.check(L.qs_plan_execute_from_basis_profile(sv.handle(), cc._h, 0, N.C.byref(cs), ms, by))
for i in range(k):
    m, r, tr, nops = N.C.c_uint32(), N.C.c_uint32(), N.C.c_uint32(), N.C.c_uint32()
    gates = N.C.c_uint64()
    qs = (N.C.c_uint32 * 16)()
    N.check(L.qs_plan_tile_info(cc._h, i, N.C.byref(m), qs, N.C.byref(r), N.C.byref(tr), N.C.byref(nops),
                                N.C.byref(gates)))
    row = {"step": i, "ms": round(ms[i], 4), "GB": round(by[i] / 1e9, 3),
           "GBps": round(by[i] / (ms[i] / 1e3) / 1e9, 1) if ms[i] > 0 else None}
    if m.value:
        row.update({"qubits": list(qs)[:m.value], "r": r.value, "transposes": tr.value, "ops": nops.value,
                    "gates": gates.value})
    print(json.dumps(row), flush=True)
