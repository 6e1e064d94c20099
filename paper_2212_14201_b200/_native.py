"""ctypes binding of libqsb.so (the C ABI declared in include/qsb.h).

The library is built in-tree (paper_2212_14201_b200/libqsb.so) by
__graft_entry__.build() / `make -C paper_2212_14201_b200/csrc`.  There is no
CPU fallback: if the library or a CUDA device is missing, calls raise.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqsb.so")

QS_OK = 0
QS_ERR_VALIDATION = -1
QS_ERR_RUNTIME = -2
QS_ERR_CUDA = -3
QS_ERR_MEMORY = -4
QS_ERR_UNSUPPORTED = -5

QS_PLAN_DEFAULT = 0
QS_PLAN_UNFUSED = 1
QS_PLAN_DENSE_FUSION = 2
QS_PLAN_TILED = 3

MAX_TARGETS = 8
MAX_EXCHANGE_BITS = 16
MAX_CONTROLS = 40


class QforgeError(RuntimeError):
    """qforge::Error (error.hpp:10-13)."""


class ValidationError(QforgeError):
    """qforge::ValidationError (error.hpp:17-20)."""


class CudaError(QforgeError):
    pass


class UnsupportedError(QforgeError):
    """qforge::UnsupportedError (error.hpp:30-33)."""


class QsGate(C.Structure):
    """struct qs_gate (include/qsb.h)."""
    _fields_ = [
        ("kind", C.c_int32),
        ("dagger", C.c_int32),
        ("num_targets", C.c_uint32),
        ("num_controls", C.c_uint32),
        ("targets", C.c_uint32 * MAX_TARGETS),
        ("controls", C.c_uint32 * MAX_CONTROLS),
        ("params", C.c_double * 3),
        ("matrix", C.POINTER(C.c_double)),
    ]


_lib = None

# name -> (restype, argtypes)
_P = C.c_void_p
_DP = C.POINTER(C.c_double)
_UP = C.POINTER(C.c_uint32)
_U64P = C.POINTER(C.c_uint64)
_GP = C.POINTER(QsGate)
HostAllgather = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
HostBarrier = C.CFUNCTYPE(C.c_int, C.c_void_p)


class HostCollectives(C.Structure):
    """qs_host_collectives (include/qsb.h)."""
    _fields_ = [("ctx", C.c_void_p), ("allgather", HostAllgather), ("barrier", HostBarrier)]


_SIGS = {
    "qs_last_error": (C.c_char_p, []),
    "qs_abi_version": (C.c_int, []),
    "qs_kernel_launches": (C.c_uint64, []),
    "qs_jit_stats": (C.c_int, [C.POINTER(C.c_uint64)] * 3),
    "qs_create": (C.c_int, [C.c_uint32, C.c_int, C.c_uint32, C.POINTER(_P)]),
    "qs_destroy": (C.c_int, [_P]),
    "qs_clone": (C.c_int, [_P, C.POINTER(_P)]),
    "qs_num_qubits": (C.c_uint32, [_P]),
    "qs_device": (C.c_int, [_P]),
    "qs_device_ptr": (C.c_void_p, [_P]),
    "qs_reset": (C.c_int, [_P]),
    "qs_set_basis_state": (C.c_int, [_P, C.c_uint64]),
    "qs_sync": (C.c_int, [_P]),
    "qs_set_amplitudes": (C.c_int, [_P, _DP, C.c_uint64, C.c_uint64]),
    "qs_get_amplitudes": (C.c_int, [_P, _DP, C.c_uint64, C.c_uint64]),
    "qs_apply_gate": (C.c_int, [_P, _GP]),
    "qs_apply_1q": (C.c_int, [_P, C.c_uint32, _DP, _UP, C.c_uint32]),
    "qs_apply_diag": (C.c_int, [_P, C.c_uint32, _DP, _UP, C.c_uint32]),
    "qs_apply_flip": (C.c_int, [_P, C.c_uint32, _UP, C.c_uint32]),
    "qs_apply_swap": (C.c_int, [_P, C.c_uint32, C.c_uint32, _UP, C.c_uint32]),
    "qs_apply_matrix": (C.c_int, [_P, _UP, C.c_uint32, _DP, _UP, C.c_uint32]),
    "qs_apply_circuit": (C.c_int, [_P, _GP, C.c_uint64, C.c_uint32, C.c_uint32]),
    "qs_run_circuit": (C.c_int, [_P, C.c_uint64, _GP, C.c_uint64, C.c_uint32, C.c_uint32]),
    "qs_run_circuit_checksum": (C.c_int, [_P, C.c_uint64, _GP, C.c_uint64, C.c_uint32, C.c_uint32,
                                          C.POINTER(C.c_double)]),
    "qs_plan_create": (C.c_int, [C.c_uint32, _GP, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(_P)]),
    "qs_plan_destroy": (C.c_int, [_P]),
    "qs_plan_execute": (C.c_int, [_P, _P]),
    "qs_plan_stats": (C.c_int, [_P, _U64P, _U64P, _U64P]),
    "qs_plan_enqueue": (C.c_int, [_P, _P]),
    "qs_plan_execute_range": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64]),
    "qs_plan_execute_from_basis": (C.c_int, [_P, _P, C.c_uint64]),
    "qs_plan_enqueue_from_basis": (C.c_int, [_P, _P, C.c_uint64]),
    "qs_plan_execute_from_basis_checksum": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_double)]),
    "qs_plan_execute_from_basis_profile": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(C.c_double),
                                                     C.POINTER(C.c_float), C.POINTER(C.c_double)]),
    "qs_plan_execute_timed": (C.c_int, [_P, _P, C.POINTER(C.c_float)]),
    "qs_stream": (C.c_void_p, [_P]),
    "qs_fuse": (C.c_int, [_GP, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(_P)]),
    "qs_fused_count": (C.c_uint64, [_P]),
    "qs_fused_get": (C.c_int, [_P, C.c_uint64, _GP]),
    "qs_fused_free": (C.c_int, [_P]),
    "qs_norm2": (C.c_int, [_P, _DP]),
    "qs_prob_one": (C.c_int, [_P, C.c_uint32, _DP]),
    "qs_probs": (C.c_int, [_P, _UP, C.c_uint32, _DP]),
    "qs_probs_full": (C.c_int, [_P, _DP, C.c_uint64, C.c_uint64]),
    "qs_checksum": (C.c_int, [_P, _DP]),
    "qs_checksum_serial": (C.c_int, [_P, _DP]),
    "qs_collapse": (C.c_int, [_P, C.c_uint32, C.c_int, C.c_double]),
    "qs_measure_collapse": (C.c_int, [_P, C.c_uint32, C.c_double, C.POINTER(C.c_int)]),
    "qs_scale": (C.c_int, [_P, C.c_double, C.c_double]),
    "qs_sample": (C.c_int, [_P, _DP, C.c_uint64, C.c_int, _U64P]),
    "qs_sample_seeded": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_int, _U64P]),
    "qs_expect_pauli": (C.c_int, [_P, C.c_char_p, C.c_uint32, _DP]),
    "qs_cumulative": (C.c_int, [_P, _DP, _DP]),
    "qs_batch_reset": (C.c_int, [_P, C.c_uint32]),
    "qs_batch_measure": (C.c_int, [_P, C.c_uint32, C.c_uint32, _DP, C.c_uint64, C.c_char_p]),
    "qs_batch_kraus": (C.c_int, [_P, C.c_uint32, _UP, C.c_uint32, _DP, C.c_uint32, _DP, C.c_uint64,
                                 C.POINTER(C.c_int32)]),
    "qs_batch_apply": (C.c_int, [_P, C.c_uint32, _UP, C.c_uint32, _DP, C.c_char_p, C.c_uint64]),
    "qs_reduced_density": (C.c_int, [_P, _UP, C.c_uint32, _DP]),
    "qs_gradient": (C.c_int, [_P, _GP, C.c_uint64, _U64P, C.c_uint64, C.c_char_p, _DP, C.c_uint32, _DP]),
    # sharded state vectors
    "qs_dist_unique_id": (C.c_int, [C.c_char_p]),
    "qs_dist_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "qs_partial_amplitude": (C.c_int, [C.c_uint32, C.POINTER(QsGate), C.c_uint64, C.POINTER(C.c_uint32), C.c_uint32,
                                       C.POINTER(C.c_uint64), C.c_uint64, C.c_int, C.c_uint32, C.POINTER(C.c_double)]),
    "qs_dist_create_host": (C.c_int, [C.POINTER(HostCollectives), C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "qs_dist_destroy": (C.c_int, [_P]),
    "qs_shards_create_local": (C.c_int, [C.c_uint32, C.c_uint32, C.c_int, C.POINTER(_P)]),
    "qs_shards_create_dist": (C.c_int, [C.c_uint32, _P, C.POINTER(_P)]),
    "qs_shards_destroy": (C.c_int, [_P]),
    "qs_shards_info": (C.c_int, [_P, _UP, _UP, _UP, _UP]),
    "qs_shards_stream": (C.c_void_p, [_P]),
    "qs_shards_sync": (C.c_int, [_P]),
    "qs_shards_set_basis_state": (C.c_int, [_P, C.c_uint64]),
    "qs_shards_set_amplitudes": (C.c_int, [_P, _DP, C.c_uint64, C.c_uint64]),
    "qs_shards_get_amplitudes": (C.c_int, [_P, _DP, C.c_uint64, C.c_uint64]),
    "qs_plan_create_sharded": (C.c_int, [C.c_uint32, C.c_uint32, _GP, C.c_uint64, C.POINTER(_P)]),
    "qs_plan_exchanges": (C.c_int, [_P, _U64P]),
    "qs_plan_tile_info": (C.c_int, [_P, C.c_uint64, _UP, _UP, _UP, _UP, _UP, C.POINTER(C.c_uint64)]),
    "qs_plan_step_info": (C.c_int, [_P, C.c_uint64, C.POINTER(C.c_int), _UP, _UP, _UP]),
    "qs_shards_plan_enqueue": (C.c_int, [_P, _P]),
    "qs_shards_plan_enqueue_from_basis": (C.c_int, [_P, _P, C.c_uint64]),
    "qs_shards_plan_execute_timed": (C.c_int, [_P, _P, C.POINTER(C.c_float)]),
    "qs_shards_plan_execute": (C.c_int, [_P, _P]),
    "qs_shards_apply_circuit": (C.c_int, [_P, _GP, C.c_uint64]),
    "qs_shards_run_circuit": (C.c_int, [_P, C.c_uint64, _GP, C.c_uint64]),
    "qs_shards_norm2": (C.c_int, [_P, _DP]),
    "qs_shards_probs": (C.c_int, [_P, _UP, C.c_uint32, _DP]),
    "qs_shards_sample": (C.c_int, [_P, _DP, C.c_uint64, C.c_int, _U64P]),
    "qs_shards_sample_seeded": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_int, _U64P]),
    "qs_shards_expect_pauli": (C.c_int, [_P, C.c_char_p, C.c_uint32, _DP]),
    "qs_shards_checksum": (C.c_int, [_P, _DP]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Loads libqsb.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libqsb.so is not built (%s); run __graft_entry__.build()" % LIB_PATH)
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc):
    if rc == QS_OK:
        return
    msg = lib().qs_last_error().decode(errors="replace")
    if rc == QS_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == QS_ERR_CUDA:
        raise CudaError(msg)
    if rc == QS_ERR_MEMORY:
        raise MemoryError(msg)
    if rc == QS_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise QforgeError(msg)


def dptr(a):
    return a.ctypes.data_as(_DP)


def uarr(vals):
    vals = list(vals)
    return (C.c_uint32 * max(1, len(vals)))(*vals), len(vals)


def gate_array(gates):
    """Sequence of objects with kind/targets/controls/params/dagger/matrix -> (QsGate array, keepalive)."""
    arr = (QsGate * max(1, len(gates)))()
    keep = []
    for i, g in enumerate(gates):
        s = arr[i]
        s.kind = int(g.kind)
        s.dagger = 1 if g.dagger else 0
        tg, ct = list(g.targets), list(g.controls)
        if len(tg) > MAX_TARGETS or len(ct) > MAX_CONTROLS:
            raise ValidationError("too many operands for the C ABI")
        s.num_targets = len(tg)
        s.num_controls = len(ct)
        for j, t in enumerate(tg):
            s.targets[j] = t
        for j, c in enumerate(ct):
            s.controls[j] = c
        for j, p in enumerate(list(g.params)[:3]):
            s.params[j] = p
        if g.matrix is not None:
            m = np.ascontiguousarray(np.asarray(g.matrix, dtype=np.complex128)).view(np.float64)
            keep.append(m)
            s.matrix = dptr(m)
    return arr, keep
