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
                             C.c_uint32, C.POINTER(C.c_double), C.c_char_p, C.POINTER(C.c_uint64), C.c_uint32,
                             C.c_int]
        _lib = L
    return _lib


def run(n, gates, plan=N.QS_PLAN_TILED, maxk=3, tile_m=12, low=3, state=None, global_qubits=0, remap=-1):
    a = np.zeros(1 << n, dtype=np.complex128)
    if state is None:
        a[0] = 1
    else:
        a[:] = state
    arr, keep = N.gate_array(gates)
    err = C.create_string_buffer(256)
    passes = C.c_uint64()
    rc = lib().te_run(n, arr, len(gates), plan, maxk, tile_m, low, N.dptr(a.view(np.float64)), err,
                      C.byref(passes), global_qubits, remap)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return a, passes.value


class Plan:
    """A sharded plan for step-wise replay (te_plan_* in tests/tile_emu.cpp)."""

    OP, TILE, SWAP = 0, 1, 2

    def __init__(self, n, g, gates):
        L = lib()
        L.te_plan_create.restype = C.c_int
        L.te_plan_create.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(N.QsGate), C.c_uint64,
                                     C.POINTER(C.c_void_p), C.c_char_p]
        L.te_plan_free.argtypes = [C.c_void_p]
        L.te_plan_steps.restype = C.c_uint64
        L.te_plan_steps.argtypes = [C.c_void_p]
        L.te_plan_step.restype = C.c_int
        L.te_plan_step.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                   C.POINTER(C.c_uint32)]
        L.te_exec_step.restype = C.c_int
        L.te_exec_step.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_double)]
        arr, keep = N.gate_array(gates)
        err = C.create_string_buffer(256)
        h = C.c_void_p()
        if L.te_plan_create(n, g, arr, len(gates), C.byref(h), err) != 0:
            raise RuntimeError(err.value.decode())
        self._h, self.n, self.g = h, n, g

    def __del__(self):
        if getattr(self, "_h", None):
            lib().te_plan_free(self._h)

    def __len__(self):
        return lib().te_plan_steps(self._h)

    def step(self, i):
        """(kind, gpos tuple, lpos tuple)."""
        nb = C.c_uint32()
        gp, lp = (C.c_uint32 * 16)(), (C.c_uint32 * 16)()
        kind = lib().te_plan_step(self._h, i, C.byref(nb), gp, lp)
        return kind, tuple(gp[:nb.value]), tuple(lp[:nb.value])

    def exec_step(self, i, rank, shard):
        """Runs non-exchange step i on `shard` (complex128, 2^(n-g), in place).
        Returns 0, or -2 if the step moved amplitude across rank bits."""
        return lib().te_exec_step(self._h, i, rank, N.dptr(shard.view(np.float64)))
