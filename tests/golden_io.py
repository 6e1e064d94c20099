"""Readers for the golden fixtures in tests/golden/ (written by
oracle/ref_driver.cpp from the unmodified reference; see tests/golden/README.md).

Circuit text format, one instruction per line:
    P <qubits> <cbits>
    G <kind> <dagger> <nt> t.. <nc> c.. <np> p(hex).. <nm> m(hex re, im)..
    M <qubit> <cbit>
Gate kinds are numbered as qforge::GateKind (circuit.hpp:22-27).
"""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class GateRec:
    __slots__ = ("kind", "dagger", "targets", "controls", "params", "matrix")

    def __init__(self, kind, targets, params=(), controls=(), dagger=False, matrix=None):
        self.kind = int(kind)
        self.dagger = bool(dagger)
        self.targets = [int(t) for t in targets]
        self.controls = [int(c) for c in controls]
        self.params = [float(p) for p in params]
        self.matrix = None if matrix is None else np.ascontiguousarray(matrix, dtype=np.complex128)

    def __repr__(self):
        return "GateRec(kind=%d, t=%s, c=%s, p=%s, dag=%s%s)" % (
            self.kind, self.targets, self.controls, self.params, self.dagger,
            "" if self.matrix is None else ", custom %dx%d" % self.matrix.shape)


class CircuitRec:
    def __init__(self, qubits, cbits=0):
        self.qubits = qubits
        self.cbits = cbits
        self.gates = []
        self.measures = []  # (qubit, cbit), only trailing measures are used here


def read_circuit(path):
    if not os.path.isabs(path):
        path = os.path.join(GOLDEN, path)
    circ = None
    with open(path) as f:
        for line in f:
            tok = line.split()
            if not tok:
                continue
            if tok[0] == "P":
                circ = CircuitRec(int(tok[1]), int(tok[2]))
            elif tok[0] == "M":
                circ.measures.append((int(tok[1]), int(tok[2])))
            elif tok[0] == "G":
                i = 1
                kind = int(tok[i]); i += 1
                dagger = tok[i] == "1"; i += 1
                nt = int(tok[i]); i += 1
                targets = [int(x) for x in tok[i:i + nt]]; i += nt
                nc = int(tok[i]); i += 1
                controls = [int(x) for x in tok[i:i + nc]]; i += nc
                np_ = int(tok[i]); i += 1
                params = [float.fromhex(x) for x in tok[i:i + np_]]; i += np_
                nm = int(tok[i]); i += 1
                matrix = None
                if nm:
                    vals = [float.fromhex(x) for x in tok[i:i + 2 * nm]]
                    dim = int(round(nm ** 0.5))
                    arr = np.array(vals, dtype=np.float64).view(np.complex128)
                    matrix = arr.reshape(dim, dim)
                circ.gates.append(GateRec(kind, targets, params, controls, dagger, matrix))
            else:
                raise ValueError("bad circuit line: %r" % line)
    return circ


def read_amps(path):
    if not os.path.isabs(path):
        path = os.path.join(GOLDEN, path)
    return np.fromfile(path, dtype=np.complex128)


def manifest(big=False):
    """manifest.json; big=True: manifest_big.json; a string: that file."""
    name = big if isinstance(big, str) else ("manifest_big.json" if big else "manifest.json")
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def cases(kind, big=False):
    return [c for c in manifest(big) if c["type"] == kind]


def case(name, big=False):
    for c in manifest(big):
        if c["name"] == name:
            return c
    raise KeyError(name)


def counts_from_indices(indices, measures, cbits):
    """run() key construction (simulator.hpp:170-177): c[0] rightmost."""
    out = {}
    idx = np.asarray(indices, dtype=np.uint64)
    keyint = np.zeros(idx.shape, dtype=np.uint64)
    for q, c in measures:
        bit = (idx >> np.uint64(q)) & np.uint64(1)
        keyint |= bit << np.uint64(c)
    vals, cnt = np.unique(keyint, return_counts=True)
    for v, c in zip(vals.tolist(), cnt.tolist()):
        key = "".join("1" if (v >> (cbits - 1 - j)) & 1 else "0" for j in range(cbits))
        out[key] = c
    return out


def fnv_indices(indices):
    """FNV-1a over uint64 LE bytes of the per-shot indices (ref_driver golden_big)."""
    h = 1469598103934665603
    b = np.asarray(indices, dtype="<u8").tobytes()
    # vectorised in chunks would be faster; this is fine for 1e6 shots
    arr = np.frombuffer(b, dtype=np.uint8)
    mask = (1 << 64) - 1
    for x in arr.tolist():
        h ^= x
        h = (h * 1099511628211) & mask
    return h
