"""ctypes binding of oracle/_ref/libtileemu.so (tests/tile_emu.cpp): replays a
libqsb plan on the host.  TEST INFRASTRUCTURE ONLY."""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2212_14201_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "_ref", "libtileemu.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), LIB])
        L = C.CDLL(LIB)
        L.te_run.restype = C.c_int
        L.te_run.argtypes = [C.c_uint32, C.POINTER(N.QsGate), C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                             C.c_uint32, C.POINTER(C.c_double), C.c_char_p, C.POINTER(C.c_uint64)]
        _lib = L
    return _lib


def run(n, gates, plan=N.QS_PLAN_TILED, maxk=3, tile_m=12, low=3, state=None):
    a = np.zeros(1 << n, dtype=np.complex128)
    if state is None:
        a[0] = 1
    else:
        a[:] = state
    arr, keep = N.gate_array(gates)
    err = C.create_string_buffer(256)
    passes = C.c_uint64()
    rc = lib().te_run(n, arr, len(gates), plan, maxk, tile_m, low, N.dptr(a.view(np.float64)), err,
                      C.byref(passes))
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return a, passes.value
