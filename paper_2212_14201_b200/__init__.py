"""B200-native state-vector simulator: a drop-in for the gate-application hot
path of qforge (the reference reconstruction of QPanda, arXiv 2212.14201).

libqsb.so (C ABI: include/qsb.h) holds the CUDA kernels for sm_100a and the
C++ planner; `qforge` mirrors the reference API in Python; the C++ drop-in
headers are under include/qforge/.
"""
from . import _native  # noqa: F401
from .qforge import (  # noqa: F401
    CompiledCircuit,
    Gate,
    GateKind,
    Measure,
    PauliOperator,
    Program,
    QforgeError,
    Rng,
    RunResult,
    SimOptions,
    StateVector,
    ValidationError,
    expectation,
    fuse_circuit,
    gen_ghz,
    gen_hea,
    gen_qft,
    gen_random_circuit,
    make_custom_gate,
    make_gate,
    probability_checksum,
    run,
)

__all__ = [n for n in dir() if not n.startswith("_")]
