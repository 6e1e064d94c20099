"""Diagnostics: compares the GPU state after each plan step with the host
emulator of the same plan (tests/tile_emu.cpp).  Usage:
    python tools/debug_passes.py qft 20 [tile_m]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import emu_lib  # noqa: E402
from paper_2212_14201_b200 import _native as N  # noqa: E402
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

kind, n = sys.argv[1], int(sys.argv[2])
m = int(sys.argv[3]) if len(sys.argv) > 3 else 12
os.environ["QSB_TILE_M"] = str(m)
g = {"qft": lambda: Q.gen_qft(n, 0x5A5A5 % (1 << n)), "random": lambda: Q.gen_random_circuit(n, 6, 424242),
     "hea": lambda: Q.gen_hea(n, 4, 7)}[kind]().gates()
cc = Q.CompiledCircuit(n, g)
st = cc.stats()
print("plan", st)
sv = Q.StateVector(n)
for i in range(st["launches"]):
    N.check(N.lib().qs_plan_execute_range(sv.handle(), cc._h, i, 1))
    os.environ["TE_MAX_STEPS"] = str(i + 1)
    want, _ = emu_lib.run(n, g, N.QS_PLAN_TILED, tile_m=m)
    err = np.max(np.abs(sv.amplitudes() - want))
    print("step", i, "err", err)
    if err > 1e-10:
        sv.set_amplitudes(want)
