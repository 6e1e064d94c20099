"""Python mirror of the reference's simulation API (qforge), backed by libqsb.

Same names, argument meaning and error behaviour as the C++ headers under
/root/reference/proj/include/qforge (cited per item); the C++ drop-in facade
with identical signatures lives in paper_2212_14201_b200/include/qforge/.
Everything amplitude-touching runs in libqsb.so on the GPU; this module only
builds gate records and moves results.
"""
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import QforgeError, UnsupportedError, ValidationError  # noqa: F401  (re-exported)


class GateKind(enum.IntEnum):
    """circuit.hpp:22-27"""
    I = 0
    X = 1
    Y = 2
    Z = 3
    H = 4
    S = 5
    T = 6
    RX = 7
    RY = 8
    RZ = 9
    U3 = 10
    CNOT = 11
    CZ = 12
    SWAP = 13
    TOFFOLI = 14
    Custom = 15


_TARGET_ARITY = {GateKind.CNOT: 2, GateKind.CZ: 2, GateKind.SWAP: 2, GateKind.TOFFOLI: 3}
_PARAM_ARITY = {GateKind.RX: 1, GateKind.RY: 1, GateKind.RZ: 1, GateKind.U3: 3}


@dataclass
class Gate:
    """circuit.hpp:115-139: targets most-significant first, controls extra."""
    kind: GateKind = GateKind.I
    targets: list = field(default_factory=list)
    params: list = field(default_factory=list)
    controls: list = field(default_factory=list)
    dagger: bool = False
    matrix: object = None  # Custom: 2^t x 2^t complex ndarray

    def qubits(self):
        return list(self.controls) + list(self.targets)


def make_gate(kind, targets, params=()):
    return Gate(GateKind(kind), list(targets), list(params))


def make_custom_gate(targets, matrix):
    return Gate(GateKind.Custom, list(targets), [], [], False, np.asarray(matrix, dtype=np.complex128))


@dataclass
class Measure:
    """MeasureOp (circuit.hpp:307-311)."""
    qubit: int
    cbit: int


class Program:
    """circuit.hpp:337-406 (flat subset: gates and measurements)."""

    def __init__(self, qubit_count=0, cbit_count=0):
        self.qubit_count = qubit_count
        self.cbit_count = cbit_count
        self.body = []

    def add(self, g, targets=None, params=()):
        if targets is not None:
            g = make_gate(g, targets, params)
        self.body.append(g)
        return self

    def measure(self, qubit, cbit):
        self.body.append(Measure(qubit, cbit))
        return self

    def gates(self):
        return [g for g in self.body if isinstance(g, Gate)]

    def gate_count(self):
        return sum(1 for g in self.body if isinstance(g, Gate))


def validate_or_throw(p):
    """circuit.hpp:427-529 (gate arity and range checks; custom unitarity is
    re-checked by the library)."""
    diags = []
    for i, ins in enumerate(p.body):
        here = "instruction %d: " % i
        if isinstance(ins, Measure):
            if ins.qubit >= p.qubit_count:
                diags.append(here + "measured qubit q[%d] out of range" % ins.qubit)
            if ins.cbit >= p.cbit_count:
                diags.append(here + "classical bit c[%d] out of range" % ins.cbit)
            continue
        g = ins
        if g.kind == GateKind.Custom:
            if g.matrix is None:
                diags.append(here + "custom gate has no matrix")
            elif np.asarray(g.matrix).shape != (1 << len(g.targets),) * 2:
                diags.append(here + "custom matrix does not match its targets")
            if g.params:
                diags.append(here + "custom gate takes no parameters")
        else:
            if len(g.targets) != _TARGET_ARITY.get(g.kind, 1):
                diags.append(here + "%s expects %d target(s), got %d" % (g.kind.name, _TARGET_ARITY.get(g.kind, 1),
                                                                       len(g.targets)))
            if len(g.params) != _PARAM_ARITY.get(g.kind, 0):
                diags.append(here + "%s expects %d parameter(s), got %d" % (g.kind.name, _PARAM_ARITY.get(g.kind, 0),
                                                                          len(g.params)))
        qs = g.qubits()
        for q in qs:
            if q >= p.qubit_count:
                diags.append(here + "qubit q[%d] out of range (program has %d)" % (q, p.qubit_count))
        if len(set(qs)) != len(qs):
            diags.append(here + "duplicate qubit operand")
    if diags:
        raise ValidationError("invalid program:\n  " + "\n  ".join(diags))


@dataclass
class SimOptions:
    """simulator.hpp:18-36 plus the B200 planner knobs (plan, device)."""
    parallel_threshold: int = 1 << 14   # accepted, no effect on the GPU
    fusion_enabled: bool = False        # accepted; gate runs are always fused into tile passes
    max_fused_qubits: int = 3
    seed: int = 0
    workers: int = 0                    # accepted, no effect on the GPU
    max_while_iterations: int = 1_000_000
    plan: int = N.QS_PLAN_DEFAULT       # default: shared-memory tile passes
    device: int = 0
    exact_sampling: bool = True

    def validate(self):
        if self.parallel_threshold < 1:
            raise ValidationError("parallel_threshold must be at least 1")
        if self.max_fused_qubits < 1 or self.max_fused_qubits > 5:
            raise ValidationError("max_fused_qubits must be in [1, 5]")
        if self.workers < 0:
            raise ValidationError("workers must be non-negative")

    def plan_mode(self):
        if self.plan != N.QS_PLAN_DEFAULT:
            return self.plan
        return N.QS_PLAN_TILED


class StateVector:
    """statevector.hpp:134-264, device-resident (complex128 in HBM)."""

    def __init__(self, num_qubits, device=0, max_qubits=30, _handle=None):
        L = N.lib()
        if _handle is None:
            h = N.C.c_void_p()
            N.check(L.qs_create(num_qubits, device, max_qubits, N.C.byref(h)))
            _handle = h
        self._h = _handle
        self.n = L.qs_num_qubits(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.qs_destroy(h)
            self._h = None

    @classmethod
    def from_amplitudes(cls, n, amps, device=0, max_qubits=30):
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        if amps.size != (1 << n):
            raise ValidationError("amplitude count does not match qubit count")
        sv = cls(n, device, max_qubits)
        N.check(N.lib().qs_set_amplitudes(sv._h, N.dptr(amps.view(np.float64)), 0, amps.size))
        return sv

    def copy(self):
        h = N.C.c_void_p()
        N.check(N.lib().qs_clone(self._h, N.C.byref(h)))
        return StateVector(0, _handle=h)

    __copy__ = copy

    def num_qubits(self):
        return self.n

    def dimension(self):
        return 1 << self.n

    def handle(self):
        return self._h

    def amplitudes(self, offset=0, count=None):
        count = (1 << self.n) - offset if count is None else count
        out = np.empty(count, dtype=np.complex128)
        N.check(N.lib().qs_get_amplitudes(self._h, N.dptr(out.view(np.float64)), offset, count))
        return out

    def amplitude(self, i):
        return complex(self.amplitudes(i, 1)[0])

    def set_amplitudes(self, amps, offset=0):
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        N.check(N.lib().qs_set_amplitudes(self._h, N.dptr(amps.view(np.float64)), offset, amps.size))

    def reset(self, basis=0):
        N.check(N.lib().qs_set_basis_state(self._h, basis))

    def norm_squared(self):
        out = N.C.c_double()
        N.check(N.lib().qs_norm2(self._h, N.C.byref(out)))
        return out.value

    def scale(self, f):
        f = complex(f)
        N.check(N.lib().qs_scale(self._h, f.real, f.imag))

    def apply_gate(self, g):
        arr, keep = N.gate_array([g])
        N.check(N.lib().qs_apply_gate(self._h, arr))

    def apply_matrix(self, targets, m, controls=()):
        m = np.ascontiguousarray(m, dtype=np.complex128)
        t, nt = N.uarr(targets)
        c, nc = N.uarr(controls)
        N.check(N.lib().qs_apply_matrix(self._h, t, nt, N.dptr(m.view(np.float64)), c, nc))

    def apply_circuit(self, gates, plan=N.QS_PLAN_DEFAULT, max_fused_qubits=3):
        arr, keep = N.gate_array(gates)
        N.check(N.lib().qs_apply_circuit(self._h, arr, len(gates), plan, max_fused_qubits))

    def probability_of_one(self, q):
        out = N.C.c_double()
        N.check(N.lib().qs_prob_one(self._h, q, N.C.byref(out)))
        return out.value

    def probabilities(self, qubits=None):
        if qubits is None:
            out = np.empty(1 << self.n, dtype=np.float64)
            N.check(N.lib().qs_probs_full(self._h, N.dptr(out), 0, out.size))
            return out
        qubits = list(qubits)
        if not qubits:
            raise ValidationError("probabilities: empty qubit subset")
        out = np.empty(1 << len(qubits), dtype=np.float64)
        q, m = N.uarr(qubits)
        N.check(N.lib().qs_probs(self._h, q, m, N.dptr(out)))
        return out

    def measure_collapse(self, q, u):
        o = N.C.c_int()
        N.check(N.lib().qs_measure_collapse(self._h, q, u, N.C.byref(o)))
        return o.value

    def collapse(self, q, outcome, prob):
        N.check(N.lib().qs_collapse(self._h, q, outcome, prob))

    def sample(self, uniforms, exact=True):
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        out = np.empty(u.size, dtype=np.uint64)
        N.check(N.lib().qs_sample(self._h, N.dptr(u), u.size, 1 if exact else 0,
                                  out.ctypes.data_as(N._U64P)))
        return out

    def sample_seeded(self, seed, shots, exact=True):
        out = np.empty(shots, dtype=np.uint64)
        N.check(N.lib().qs_sample_seeded(self._h, seed, shots, 1 if exact else 0, out.ctypes.data_as(N._U64P)))
        return out

    def checksum(self):
        out = N.C.c_double()
        N.check(N.lib().qs_checksum(self._h, N.C.byref(out)))
        return out.value

    def checksum_serial(self):
        """probability_checksum with the reference's serial rounding (bench.hpp:141-148)."""
        out = N.C.c_double()
        N.check(N.lib().qs_checksum_serial(self._h, N.C.byref(out)))
        return out.value

    def expect_pauli(self, words):
        """words: list of per-qubit letter strings of length n -> complex array."""
        letters = "".join(words).encode()
        out = np.empty(2 * len(words), dtype=np.float64)
        N.check(N.lib().qs_expect_pauli(self._h, letters, len(words), N.dptr(out)))
        return out.view(np.complex128)


def probability_checksum(state):
    """bench.hpp:141-148"""
    return state.checksum()


class CompiledCircuit:
    """A gate list planned once (qs_plan_create) and executed many times."""

    def __init__(self, n, gates, plan=N.QS_PLAN_DEFAULT, max_fused_qubits=3):
        arr, keep = N.gate_array(gates)
        h = N.C.c_void_p()
        N.check(N.lib().qs_plan_create(n, arr, len(gates), plan, max_fused_qubits, N.C.byref(h)))
        self._h = h
        self.n = n

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.qs_plan_destroy(h)

    def execute(self, state, from_basis=None):
        """Runs the plan on `state`; with from_basis=b the state is first reset to
        |b> (fused into the first pass)."""
        if from_basis is None:
            N.check(N.lib().qs_plan_execute(state.handle(), self._h))
        else:
            N.check(N.lib().qs_plan_execute_from_basis(state.handle(), self._h, from_basis))

    def execute_checksum(self, state, from_basis=0):
        """Runs the plan from |from_basis> and returns probability_checksum of the
        result (bench.hpp:141-148), summed by the last pass as it stores."""
        cs = N.C.c_double()
        N.check(N.lib().qs_plan_execute_from_basis_checksum(state.handle(), self._h, from_basis, N.C.byref(cs)))
        return cs.value

    def stats(self):
        a, b, c = N.C.c_uint64(), N.C.c_uint64(), N.C.c_uint64()
        N.check(N.lib().qs_plan_stats(self._h, N.C.byref(a), N.C.byref(b), N.C.byref(c)))
        return {"passes": a.value, "launches": b.value, "gates": c.value}


def fuse_circuit(p, max_fused_qubits=3):
    """fusion.hpp:108-133: runs between measurements fused into Custom blocks."""
    if max_fused_qubits < 1:
        raise ValidationError("max_fused_qubits must be at least 1")
    out = Program(p.qubit_count, p.cbit_count)
    run = []

    def flush():
        if not run:
            return
        arr, keep = N.gate_array(run)
        h = N.C.c_void_p()
        N.check(N.lib().qs_fuse(arr, len(run), p.qubit_count, max_fused_qubits, N.C.byref(h)))
        try:
            for i in range(N.lib().qs_fused_count(h)):
                g = N.QsGate()
                N.check(N.lib().qs_fused_get(h, i, N.C.byref(g)))
                out.body.append(_gate_from_struct(g))
        finally:
            N.lib().qs_fused_free(h)
        run.clear()

    for ins in p.body:
        if isinstance(ins, Gate):
            run.append(ins)
        else:
            flush()
            out.body.append(ins)
    flush()
    return out


def _gate_from_struct(s):
    kind = GateKind(s.kind)
    targets = list(s.targets[: s.num_targets])
    controls = list(s.controls[: s.num_controls])
    params = list(s.params[: _PARAM_ARITY.get(kind, 0)])
    m = None
    if kind == GateKind.Custom:
        dim = 1 << s.num_targets
        m = np.ctypeslib.as_array(s.matrix, shape=(2 * dim * dim,)).copy().view(np.complex128).reshape(dim, dim)
    return Gate(kind, targets, params, controls, bool(s.dagger), m)


@dataclass
class RunResult:
    """simulator.hpp:38-42: keys are register contents, c[0] rightmost."""
    counts: dict = field(default_factory=dict)
    final_state: object = None


def _trailing_measure_form(p):
    seen = False
    for ins in p.body:
        if isinstance(ins, Gate):
            if seen:
                return False
        else:
            seen = True
    return True


_KEY_BITS = 12
_KEY_TABLE = {}


def _key_table(width):
    t = _KEY_TABLE.get(width)
    if t is None:
        t = _KEY_TABLE[width] = [format(i, "0%db" % width) for i in range(1 << width)]
    return t


def counts_from_indices(indices, measures, cbits):
    """Key construction of run() (simulator.hpp:170-177): c[0] rightmost.
    Keys are assembled from 12-bit string tables (one lookup per 12 classical
    bits) instead of one format() per distinct outcome."""
    idx = np.asarray(indices, dtype=np.uint64)
    keyint = np.zeros(idx.shape, dtype=np.uint64)
    for m in measures:
        keyint |= ((idx >> np.uint64(m.qubit)) & np.uint64(1)) << np.uint64(m.cbit)
    vals, cnt = np.unique(keyint, return_counts=True)
    if not cbits:
        return {"": int(cnt.sum())} if len(vals) else {}
    parts = []  # most significant chunk first
    for lo in range(0, cbits, _KEY_BITS):
        w = min(_KEY_BITS, cbits - lo)
        tab = _key_table(w)
        parts.insert(0, [tab[v] for v in ((vals >> np.uint64(lo)) & np.uint64((1 << w) - 1)).astype(np.int64).tolist()])
    keys = parts[0] if len(parts) == 1 else ["".join(k) for k in zip(*parts)]
    return dict(zip(keys, cnt.tolist()))


def run_plan_mode(opts):
    """The plan run() executes, as in the C++ facade (include/qforge/simulator.hpp
    run()): fusion_enabled keeps the default tile passes -- they already fuse
    every gate run, far beyond fuse_circuit's k <= 5 blocks -- and the
    reference's dense-block plan runs only when asked for explicitly
    (plan=QS_PLAN_DENSE_FUSION)."""
    return opts.plan_mode()


def run(p, opts=None, shots=0):
    """simulator.hpp:142-194."""
    opts = opts or SimOptions()
    opts.validate()
    validate_or_throw(p)
    mode = run_plan_mode(opts)
    result = RunResult()
    if _trailing_measure_form(p):
        sv = StateVector(p.qubit_count, opts.device)
        gates = p.gates()
        if gates:
            sv.apply_circuit(gates, mode, opts.max_fused_qubits)
        measures = [m for m in p.body if isinstance(m, Measure)]
        result.final_state = sv
        if shots > 0:
            if not measures:
                result.counts["0" * p.cbit_count] = shots
            else:
                idx = sv.sample_seeded(opts.seed, shots, opts.exact_sampling)
                result.counts = counts_from_indices(idx, measures, p.cbit_count)
        return result
    # general path: re-execute per shot with Rng::derive(seed, s) (rng.hpp:26-28)
    runs = shots if shots > 0 else 1
    counts = {}
    sv = None
    for s in range(runs):
        rng = Rng.derive(opts.seed, s)
        sv = StateVector(p.qubit_count, opts.device)
        cbits = [0] * p.cbit_count
        pending = []
        for ins in p.body:
            if isinstance(ins, Gate):
                pending.append(ins)
                continue
            if pending:
                sv.apply_circuit(pending, mode, opts.max_fused_qubits)
                pending = []
            cbits[ins.cbit] = sv.measure_collapse(ins.qubit, rng.uniform())
        if pending:
            sv.apply_circuit(pending, mode, opts.max_fused_qubits)
        if shots > 0:
            key = "".join("1" if cbits[len(cbits) - 1 - i] else "0" for i in range(len(cbits)))
            counts[key] = counts.get(key, 0) + 1
    result.counts = counts
    result.final_state = sv
    return result


# ------------------------------------------------------------------ rng.hpp

_MASK64 = (1 << 64) - 1


def splitmix64(x):
    """rng.hpp:9-14"""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


class Rng:
    """rng.hpp:20-46: std::mt19937_64 with uniform() = (next() >> 11) * 2^-53."""

    def __init__(self, seed):
        mt = [0] * 312
        mt[0] = seed & _MASK64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK64
        self._mt = mt
        self._i = 312

    @staticmethod
    def derive(seed, index):
        return Rng(splitmix64(seed ^ splitmix64(index + 1)))

    def next(self):
        if self._i >= 312:
            mt = self._mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self._i = 0
        y = self._mt[self._i]
        self._i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform(self, hi=None):
        u = (self.next() >> 11) * 2.0 ** -53
        return u if hi is None else u * hi

    def below(self, k):
        return self.next() % k


# ------------------------------------------------------------ generators

def gen_random_circuit(n, d, seed):
    """bench.hpp:72-94"""
    if n < 1:
        raise ValidationError("random circuit requires n >= 1")
    if d < 1:
        raise ValidationError("random circuit requires d >= 1")
    p = Program(n, 0)
    rng = Rng(seed)
    for _ in range(d):
        for q in range(n):
            axis = rng.below(3)
            angle = rng.uniform(2.0 * math.pi)
            p.add(make_gate((GateKind.RX, GateKind.RY, GateKind.RZ)[axis], [q], [angle]))
        if n > 1:
            for i in range(n):
                p.add(make_gate(GateKind.CNOT, [(i + 1) % n, i]))
    return p


def gen_ghz(n):
    """GHZ(n): H(0), CNOT(i, i+1) (oracle/circuits.hpp mirror)."""
    p = Program(n, 0)
    p.add(make_gate(GateKind.H, [0]))
    for i in range(n - 1):
        p.add(make_gate(GateKind.CNOT, [i, i + 1]))
    return p


def gen_qft(n, basis_input=0):
    """QFT(n) on |basis_input>: X prep, H(j) + controlled U3(0,0,pi/2^(j-k)), swaps."""
    p = Program(n, 0)
    for q in range(n):
        if (basis_input >> q) & 1:
            p.add(make_gate(GateKind.X, [q]))
    for j in range(n - 1, -1, -1):
        p.add(make_gate(GateKind.H, [j]))
        for k in range(j - 1, -1, -1):
            g = make_gate(GateKind.U3, [j], [0.0, 0.0, math.pi / float(1 << (j - k))])
            g.controls = [k]
            p.add(g)
    for i in range(n // 2):
        p.add(make_gate(GateKind.SWAP, [i, n - 1 - i]))
    return p


def gen_hea(n, layers, seed):
    """Hardware-efficient ansatz: RY, RZ per qubit then CNOT(q, q+1); Rng(seed) angles."""
    p = Program(n, 0)
    rng = Rng(seed)
    for _ in range(layers):
        for q in range(n):
            a = rng.uniform(2.0 * math.pi)
            p.add(make_gate(GateKind.RY, [q], [a]))
            b = rng.uniform(2.0 * math.pi)
            p.add(make_gate(GateKind.RZ, [q], [b]))
        for q in range(n - 1):
            p.add(make_gate(GateKind.CNOT, [q, q + 1]))
    return p


# ------------------------------------------------------------ variational

class PauliOperator:
    """pauli.hpp:21-252 (subset): sum of real-or-complex weighted Pauli words."""

    def __init__(self, terms=None):
        self._terms = {}
        for word, c in (terms or {}).items():
            key = self._parse(word)
            self._terms[key] = self._terms.get(key, 0) + complex(c)
        self._prune()

    @staticmethod
    def _parse(word):
        t = []
        i = 0
        w = word.strip()
        toks = w.replace(",", " ").split()
        for tok in toks:
            p = tok[0].upper()
            if p == "I":
                continue
            if p not in "XYZ":
                raise ValidationError("Pauli term '%s': expected X/Y/Z/I" % word)
            q = int(tok[1:])
            if any(q == x for x, _ in t):
                raise ValidationError("Pauli term '%s': qubit %d repeated" % (word, q))
            t.append((q, p))
            i += 1
        return tuple(sorted(t))

    def _prune(self):
        self._terms = {k: v for k, v in self._terms.items() if abs(v) >= 1e-14}

    def terms(self):
        return dict(self._terms)

    def num_qubits(self):
        return max((t[-1][0] + 1 for t in self._terms if t), default=0)

    def is_hermitian(self, tol=1e-10):
        return all(abs(c.imag) <= tol for c in self._terms.values())


def expectation(p, H, opts=None):
    """variational.hpp:19-54: <psi|H|psi>, one read pass per term on the GPU."""
    opts = opts or SimOptions()
    opts.validate()
    if not H.is_hermitian():
        raise ValidationError("expectation requires a Hermitian operator")
    if H.num_qubits() > p.qubit_count:
        raise ValidationError("operator touches qubits beyond the program")
    if any(not isinstance(ins, Gate) for ins in p.body):
        raise ValidationError("expectation requires a measurement-free gate program")
    validate_or_throw(p)
    sv = StateVector(p.qubit_count, opts.device)
    if p.body:
        sv.apply_circuit(p.body, opts.plan_mode(), opts.max_fused_qubits)
    terms = list(H.terms().items())
    words = []
    for key, _ in terms:
        letters = ["I"] * p.qubit_count
        for q, l in key:
            letters[q] = l
        words.append("".join(letters))
    vals = sv.expect_pauli(words) if words else np.zeros(0, dtype=np.complex128)
    acc = sum(c * v for (_, c), v in zip(terms, vals))
    acc = complex(acc)
    if abs(acc.imag) > 1e-10:
        raise QforgeError("expectation has a non-real residue of %g; operator or state corrupt" % acc.imag)
    return acc.real


class ParamCircuit:
    """variational.hpp:56-130: a gate template with named rotation slots."""

    def __init__(self, qubits, cbits=0):
        self.tpl = Program(qubits, cbits)
        self.slots = []  # (body index, name)
        self.names = []

    def add(self, g, targets=None, params=()):
        self.tpl.add(g, targets, params)
        return self

    def add_param(self, kind, target, name):
        kind = GateKind(kind)
        if kind not in (GateKind.RX, GateKind.RY, GateKind.RZ):
            raise QforgeError("parameter '%s' used in a non-rotation position (%s)" % (name, kind.name))
        self.slots.append((len(self.tpl.body), name))
        self.tpl.add(kind, [target], [0.0])
        if name not in self.names:
            self.names.append(name)
        return self

    def parameter_names(self):
        return list(self.names)

    def bind(self, values):
        import copy
        p = copy.deepcopy(self.tpl)
        for idx, name in self.slots:
            if name not in values:
                raise ValidationError("parameter '%s' is unbound" % name)
            p.body[idx].params = [float(values[name])]
        return p


def gradient(pc, H, at, opts=None):
    """variational.hpp:139-155 values (shift rule) by adjoint differentiation on
    the GPU: one forward run + one backward sweep for every slot (qs_gradient)."""
    opts = opts or SimOptions()
    opts.validate()
    p = pc.bind(at)
    if not H.is_hermitian():
        raise ValidationError("expectation requires a Hermitian operator")
    if H.num_qubits() > p.qubit_count:
        raise ValidationError("operator touches qubits beyond the program")
    if any(not isinstance(ins, Gate) for ins in p.body):
        raise ValidationError("expectation requires a measurement-free gate program")
    validate_or_throw(p)
    arr, keep = N.gate_array(p.body)
    slots = np.array([idx for idx, _ in pc.slots], dtype=np.uint64)
    terms = list(H.terms().items())
    words, coeffs = [], []
    for key, c in terms:
        letters = ["I"] * p.qubit_count
        for q, l in key:
            letters[q] = l
        words.append("".join(letters))
        coeffs += [complex(c).real, complex(c).imag]
    coeffs = np.array(coeffs if coeffs else [0.0], dtype=np.float64)
    work = StateVector(p.qubit_count, opts.device)
    per = np.zeros(max(1, len(slots)), dtype=np.float64)
    N.check(N.lib().qs_gradient(work.handle(), arr, len(p.body), slots.ctypes.data_as(N._U64P), len(slots),
                                "".join(words).encode(), N.dptr(coeffs), len(terms), N.dptr(per)))
    return [float(sum(per[i] for i, (_, nm) in enumerate(pc.slots) if nm == name)) for name in pc.names]


# ------------------------------------------------------------------ pathsum.hpp

class FlatCircuitRequired(QforgeError):
    """qforge::FlatCircuitRequired (error.hpp:23-26)."""


class BudgetExceeded(QforgeError):
    """qforge::BudgetExceeded (error.hpp:43-48): carries the path / branch estimate."""

    def __init__(self, msg, estimated_paths):
        super().__init__(msg)
        self.estimated_paths = estimated_paths


DEFAULT_PATH_BUDGET = 1 << 22  # pathsum.hpp:183


def _gates_only(p, what):
    for ins in p.body:
        if isinstance(ins, Measure):
            raise UnsupportedError("%s is defined for measurement-free programs" % what)
        if not isinstance(ins, Gate):
            raise FlatCircuitRequired("%s requires a flat program" % what)


def path_count_estimate(p):
    """2^(control count after rewriting each gate as controlled one-target
    operators), as the reference's path evaluator branches (pathsum.hpp:30-101):
    CNOT / CZ one control, TOFFOLI two, SWAP three CNOTs, plus extra controls."""
    bits = 0
    for g in p.body:
        if g.kind == GateKind.I:
            continue
        extra = len(g.controls)
        if g.kind in (GateKind.CNOT, GateKind.CZ):
            bits += extra + 1
        elif g.kind == GateKind.TOFFOLI:
            bits += extra + 2
        elif g.kind == GateKind.SWAP:
            bits += 3 * (extra + 1)
        elif g.kind == GateKind.Custom and len(g.targets) != 1:
            raise UnsupportedError("path-sum evaluation supports custom gates on one target only")
        else:
            bits += extra
    return (1 << bits) if bits <= 62 else (1 << 64) - 1


def _parse_bitstring(bits, n):
    """pathsum.hpp:165-178: rightmost character is qubit 0 -> basis index."""
    if len(bits) != n:
        raise ValidationError("target bitstring length %d does not match %d qubits" % (len(bits), n))
    if any(c not in "01" for c in bits):
        raise ValidationError("target bitstring must contain only 0/1")
    return int(bits, 2) if n else 0


def single_amplitude(p, target, path_budget=DEFAULT_PATH_BUDGET, device=0):
    """<target|U|0...0> (pathsum.hpp:188-202).  Same validation, errors and
    budget as the reference's path evaluator; the value comes from the GPU
    state vector (one tile-pass run, one amplitude read), which the budget does
    not limit -- it is kept only so callers see the reference's behaviour."""
    validate_or_throw(p)
    _gates_only(p, "path-sum evaluation")
    est = path_count_estimate(p)
    idx = _parse_bitstring(target, p.qubit_count)
    if est > path_budget:
        raise BudgetExceeded("path count %s exceeds budget %d" % ("overflows" if est >= (1 << 64) - 1 else est,
                                                                  path_budget), est)
    sv = StateVector(p.qubit_count, device)
    if p.body:
        sv.apply_circuit(p.body)
    return complex(sv.amplitude(idx))


@dataclass
class CutPlan:
    """pathsum.hpp:208-213."""
    block_a: list = field(default_factory=list)
    block_b: list = field(default_factory=list)
    crossing_gates: list = field(default_factory=list)
    branch_count: int = 1


def _check_cuttable(g):
    if g.controls:
        raise UnsupportedError("cut planning expects gates without extra controls")
    if len(g.targets) == 1 or g.kind in (GateKind.CNOT, GateKind.CZ):
        return
    raise UnsupportedError("cut planning cannot handle %s" % g.kind.name)


def plan_cut(p):
    """Balanced bipartition with few crossing 2-qubit gates (pathsum.hpp:232-310):
    exhaustive over the ceil(n/2)-subsets for n <= 12, otherwise first-improving
    pair swaps from the low half.  Host-side combinatorics."""
    validate_or_throw(p)
    _gates_only(p, "cut planning")
    n = p.qubit_count
    if n < 2:
        raise ValidationError("cut planning needs at least 2 qubits")
    pairs = []
    for g in p.body:
        _check_cuttable(g)
        if len(g.targets) == 2:
            pairs.append((g.targets[0], g.targets[1]))
    size_a = (n + 1) // 2

    def cross(mask):
        return sum(((mask >> a) ^ (mask >> b)) & 1 for a, b in pairs)

    if n <= 12:
        best, best_c = 0, None
        for mask in range(1 << n):
            if bin(mask).count("1") != size_a:
                continue
            c = cross(mask)
            if best_c is None or c < best_c:
                best, best_c = mask, c
    else:
        mask = (1 << size_a) - 1
        cur = cross(mask)
        improved = True
        while improved:
            improved = False
            for a in range(n):
                if not (mask >> a) & 1:
                    continue
                for b in range(n):
                    if (mask >> b) & 1:
                        continue
                    m2 = (mask & ~(1 << a)) | (1 << b)
                    c = cross(m2)
                    if c < cur:
                        mask, cur, improved = m2, c, True
                        break
                if improved:
                    break
        best = mask
    plan = CutPlan([q for q in range(n) if (best >> q) & 1], [q for q in range(n) if not (best >> q) & 1])
    for i, g in enumerate(p.body):
        if len(g.targets) == 2 and ((best >> g.targets[0]) & 1) != ((best >> g.targets[1]) & 1):
            plan.crossing_gates.append(i)
    k = len(plan.crossing_gates)
    plan.branch_count = (1 << 64) - 1 if k >= 63 else 1 << k
    return plan


def partial_amplitude(p, plan, targets, branch_budget=DEFAULT_PATH_BUDGET, device=0, batch_qubits=0):
    """pathsum.hpp:317-459: amplitudes of `targets` (bitstrings, qubit 0
    rightmost) summed over the 2^k branches of the cut -- all branches batched
    as extra qubits of two half-size GPU states (qs_partial_amplitude)."""
    validate_or_throw(p)
    n = p.qubit_count
    side = [-1] * n
    for q in plan.block_a:
        if q >= n:
            raise ValidationError("cut plan qubit out of range")
        side[q] = 0
    for q in plan.block_b:
        if q >= n or side[q] != -1:
            raise ValidationError("cut plan blocks must partition the qubits")
        side[q] = 1
    if any(s == -1 for s in side):
        raise ValidationError("cut plan blocks must partition the qubits")
    if plan.branch_count > branch_budget:
        raise BudgetExceeded("branch count %d exceeds budget %d" % (plan.branch_count, branch_budget),
                             plan.branch_count)
    crossing = []
    for i, ins in enumerate(p.body):
        if not isinstance(ins, Gate):
            raise UnsupportedError("partial amplitude expects a gates-only program")
        _check_cuttable(ins)
        if len(ins.targets) == 2 and side[ins.targets[0]] != side[ins.targets[1]]:
            crossing.append(i)
    if crossing != list(plan.crossing_gates):
        raise ValidationError("cut plan does not match the program's gates")
    keys, idx = [], []
    for t in targets:
        b = _parse_bitstring(t, n)
        if t not in keys:
            keys.append(t)
            idx.append(b)
    out = {t: 0j for t in targets}
    if not keys:
        return out
    arr, keep = N.gate_array(p.body)
    ba = np.array(plan.block_a, dtype=np.uint32)
    ti = np.array(idx, dtype=np.uint64)
    res = np.zeros(2 * len(keys), dtype=np.float64)
    N.check(N.lib().qs_partial_amplitude(n, arr, len(p.body), ba.ctypes.data_as(N.C.POINTER(N.C.c_uint32)), len(ba),
                                         ti.ctypes.data_as(N._U64P), len(keys), device, batch_qubits, N.dptr(res)))
    for j, t in enumerate(keys):
        out[t] = complex(res[2 * j], res[2 * j + 1])
    return out
