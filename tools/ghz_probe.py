"""config 1 breakdown: run() and probabilities() of GHZ(20) / QFT(20), 20 reps each (wall ms)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_14201_b200 import qforge as Q  # noqa: E402

for name, p in (("ghz20", Q.gen_ghz(20)), ("qft20", Q.gen_qft(20, 0x5A5A5))):
    Q.run(p).final_state.probabilities()
    tr, tp = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        r = Q.run(p)
        t1 = time.perf_counter()
        r.final_state.probabilities()
        t2 = time.perf_counter()
        tr.append((t1 - t0) * 1e3)
        tp.append((t2 - t1) * 1e3)
    print(name, "run ms min/med", round(min(tr), 3), round(sorted(tr)[10], 3), "probs ms min/med", round(min(tp), 3),
          round(sorted(tp)[10], 3))
