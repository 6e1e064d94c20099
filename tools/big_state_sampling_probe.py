import sys, time
sys.path.insert(0, '/root/repo')
from paper_2212_14201_b200 import qforge as Q
for n in (32, 33):
    sv = Q.StateVector(n, 0, max_qubits=n)
    sv.apply_circuit(Q.gen_random_circuit(n, 1, 5).gates())
    try:
        t = time.time(); idx = sv.sample_seeded(1, 1000, True); print(n, 'sampled', idx[:3], round(time.time() - t, 2), 's')
    except Exception as e:
        print(n, type(e).__name__, e)
    print(n, 'checksum_serial', end=' ')
    try:
        print(sv.checksum_serial())
    except Exception as e:
        print(type(e).__name__, e)
    del sv
