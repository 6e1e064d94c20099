"""ctypes binding of the C oracle (oracle/_ref/liboracle.so).

TEST INFRASTRUCTURE: the oracle is the checker, never the thing measured or
shipped.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
load it.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref", "liboracle.so")


class QoGate(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dagger", C.c_int32),
        ("num_targets", C.c_uint32),
        ("num_controls", C.c_uint32),
        ("targets", C.c_uint32 * 8),
        ("controls", C.c_uint32 * 40),
        ("params", C.c_double * 3),
        ("matrix", C.POINTER(C.c_double)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), LIB])
    L = C.CDLL(LIB)
    dp = C.POINTER(C.c_double)
    up = C.POINTER(C.c_uint32)
    u64p = C.POINTER(C.c_uint64)
    gp = C.POINTER(QoGate)
    L.qo_splitmix64.restype = C.c_uint64
    L.qo_splitmix64.argtypes = [C.c_uint64]
    L.qo_rng_next.restype = C.c_uint64
    L.qo_rng_uniform.restype = C.c_double
    L.qo_rng_below.restype = C.c_uint64
    L.qo_rng_below.argtypes = [C.c_void_p, C.c_uint64]
    L.qo_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
    L.qo_rng_derive.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
    L.qo_uniforms.argtypes = [C.c_uint64, C.c_uint64, dp]
    L.qo_init_zero.argtypes = [dp, C.c_uint32]
    L.qo_apply_gate.argtypes = [dp, C.c_uint32, gp]
    L.qo_apply_gates.argtypes = [dp, C.c_uint32, gp, C.c_uint64]
    L.qo_norm2.restype = C.c_double
    L.qo_norm2.argtypes = [dp, C.c_uint32]
    L.qo_prob_one.restype = C.c_double
    L.qo_prob_one.argtypes = [dp, C.c_uint32, C.c_uint32]
    L.qo_probs.argtypes = [dp, C.c_uint32, up, C.c_uint32, dp]
    L.qo_probs_full.argtypes = [dp, C.c_uint32, dp]
    L.qo_collapse.argtypes = [dp, C.c_uint32, C.c_uint32, C.c_int, C.c_double]
    L.qo_measure_collapse.argtypes = [dp, C.c_uint32, C.c_uint32, C.c_double]
    L.qo_checksum.restype = C.c_double
    L.qo_checksum.argtypes = [dp, C.c_uint32]
    L.qo_sample_seeded.argtypes = [dp, C.c_uint32, C.c_uint64, C.c_uint64, u64p]
    L.qo_expectation.restype = C.c_double
    L.qo_expectation.argtypes = [dp, C.c_uint32, C.c_char_p, dp, C.c_uint32, dp]
    for fn in ("qo_gen_random_circuit", "qo_gen_ghz", "qo_gen_qft", "qo_gen_hea"):
        getattr(L, fn).restype = C.c_uint64
    L.qo_gen_random_circuit.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, gp]
    L.qo_gen_ghz.argtypes = [C.c_uint32, gp]
    L.qo_gen_qft.argtypes = [C.c_uint32, C.c_uint64, gp]
    L.qo_gen_hea.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, gp]
    L.qo_base_matrix.argtypes = [gp, dp]
    _lib = L
    return L


class Rng:
    """Rng (rng.hpp:20-46) through the oracle."""

    def __init__(self, seed, derive_index=None):
        self._buf = C.create_string_buffer(312 * 8 + 16)
        if derive_index is None:
            lib().qo_rng_seed(self._buf, seed)
        else:
            lib().qo_rng_derive(self._buf, seed, derive_index)

    def next(self):
        return lib().qo_rng_next(self._buf)

    def uniform(self):
        return lib().qo_rng_uniform(self._buf)

    def below(self, k):
        return lib().qo_rng_below(self._buf, k)


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def gate_array(gates):
    """List of golden_io.GateRec -> (ctypes array, keepalive)."""
    arr = (QoGate * max(1, len(gates)))()
    keep = []
    for i, g in enumerate(gates):
        s = arr[i]
        s.kind = g.kind
        s.dagger = 1 if g.dagger else 0
        s.num_targets = len(g.targets)
        s.num_controls = len(g.controls)
        for j, t in enumerate(g.targets):
            s.targets[j] = t
        for j, c in enumerate(g.controls):
            s.controls[j] = c
        for j, p in enumerate(g.params):
            s.params[j] = p
        if g.matrix is not None:
            m = np.ascontiguousarray(g.matrix, dtype=np.complex128).view(np.float64)
            keep.append(m)
            s.matrix = _dptr(m)
    return arr, keep


def gates_from_array(arr, count):
    from golden_io import GateRec
    out = []
    for i in range(count):
        s = arr[i]
        out.append(GateRec(s.kind, list(s.targets[: s.num_targets]),
                           list(s.params[: {7: 1, 8: 1, 9: 1, 10: 3}.get(s.kind, 0)]),
                           list(s.controls[: s.num_controls]), bool(s.dagger)))
    return out


def zero_state(n):
    a = np.zeros(1 << n, dtype=np.complex128)
    a[0] = 1
    return a


def run_gates(n, gates, state=None):
    a = zero_state(n) if state is None else np.array(state, dtype=np.complex128)
    arr, keep = gate_array(gates)
    rc = lib().qo_apply_gates(_dptr(a.view(np.float64)), n, arr, len(gates))
    if rc != 0:
        raise ValueError("oracle rejected the circuit")
    return a


def apply_gate(a, n, g):
    arr, keep = gate_array([g])
    rc = lib().qo_apply_gate(_dptr(a.view(np.float64)), n, arr)
    if rc != 0:
        raise ValueError("oracle rejected the gate")


def gen(name, *args):
    L = lib()
    fn = getattr(L, "qo_gen_" + name)
    count = fn(*args, None)
    arr = (QoGate * count)()
    fn(*args, arr)
    return gates_from_array(arr, count)


def norm2(a, n):
    return lib().qo_norm2(_dptr(a.view(np.float64)), n)


def prob_one(a, n, q):
    return lib().qo_prob_one(_dptr(a.view(np.float64)), n, q)


def probs(a, n, qubits):
    out = np.zeros(1 << len(qubits), dtype=np.float64)
    qs = (C.c_uint32 * len(qubits))(*qubits)
    lib().qo_probs(_dptr(a.view(np.float64)), n, qs, len(qubits), _dptr(out))
    return out


def probs_full(a, n):
    out = np.zeros(1 << n, dtype=np.float64)
    lib().qo_probs_full(_dptr(a.view(np.float64)), n, _dptr(out))
    return out


def checksum(a, n):
    return lib().qo_checksum(_dptr(a.view(np.float64)), n)


def measure_collapse(a, n, q, u):
    r = lib().qo_measure_collapse(_dptr(a.view(np.float64)), n, q, u)
    if r < 0:
        raise RuntimeError("collapse onto zero-probability outcome")
    return r


def sample_seeded(a, n, seed, shots):
    out = np.zeros(shots, dtype=np.uint64)
    lib().qo_sample_seeded(_dptr(a.view(np.float64)), n, seed, shots,
                           out.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out


def uniforms(seed, count):
    out = np.zeros(count, dtype=np.float64)
    lib().qo_uniforms(seed, count, _dptr(out))
    return out


def expectation(a, n, terms):
    """terms: list of (letters-by-qubit string of length n, coeff)."""
    letters = "".join(t for t, _ in terms).encode()
    coeffs = np.array([c for _, c in terms], dtype=np.float64)
    im = C.c_double(0)
    re = lib().qo_expectation(_dptr(a.view(np.float64)), n, letters, _dptr(coeffs), len(terms), C.byref(im))
    return re, im.value


def parse_hamiltonian(text, n):
    """PauliOperator::to_string() text (pauli.hpp:105-128) -> [(letters, coeff)]."""
    terms = []
    for part in text.split(" + "):
        tok = part.split()
        coeff = float(tok[0])
        letters = ["I"] * n
        for f in tok[1:]:
            if f == "I":
                continue
            letters[int(f[1:])] = f[0]
        terms.append(("".join(letters), coeff))
    return terms
