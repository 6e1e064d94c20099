"""Sharded state vectors over several GPUs.

The reference has no distributed mode: its StateVector is one host array
(statevector.hpp:111-118).  Here an n-qubit state is split over 2^g shards --
the top g qubits are rank bits -- and a plan compiled for g rank bits runs tile
passes on every shard independently; before a non-diagonal gate on a rank bit
the ranks exchange data so that rank bits and local qubits trade places (one
bit: pairwise half-shard exchange; k bits: all-to-all among 2^k ranks;
paper_2212_14201_b200/csrc/shard.cpp).

  * ``ShardedState.local(n, g)``: all 2^g shards in this process on one GPU
    (exchanges are device-local); validates sharded plans on a single B200.
  * ``ShardedState.distributed(n, comm)``: one shard per process/GPU, exchanges
    over NCCL send/recv.  ``DistComm.from_torch()`` builds the communicator from
    an initialised torch.distributed process group (the NCCL unique id is
    broadcast through it; torch is plumbing only).
"""
import ctypes as C

import numpy as np

from . import _native as N


class DistComm:
    """NCCL communicator over `world` ranks (a power of two), one GPU each."""

    def __init__(self, unique_id, world, rank, device):
        h = C.c_void_p()
        N.check(N.lib().qs_dist_create(bytes(unique_id), world, rank, device, C.byref(h)))
        self._h = h
        self.world = world
        self.rank = rank
        self.device = device

    @staticmethod
    def unique_id():
        buf = C.create_string_buffer(128)
        N.check(N.lib().qs_dist_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch(cls, device=None):
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        if device is None:
            device = torch.cuda.current_device()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(obj[0], world, rank, device)

    @classmethod
    def host_from_torch(cls, device=None, group=None):
        """Communicator whose collectives run through torch.distributed on the
        host (any backend, e.g. gloo) instead of NCCL: qs_dist_create_host.
        Rank-to-rank data then moves only over CUDA-IPC peer memory.  This is
        what lets two processes share one GPU (NCCL refuses duplicate devices),
        so the multi-process IPC data path can be tested on one B200."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        self = cls.__new__(cls)

        def allgather(ctx, send, recv, nbytes):
            try:
                mine = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, mine, group=group)
                C.memmove(recv, b"".join(o.numpy().tobytes() for o in outs), nbytes * world)
                return 0
            except Exception:  # reported to the library as a failed collective
                return 1

        def barrier(ctx):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:
                return 1

        self._cbs = (N.HostAllgather(allgather), N.HostBarrier(barrier))
        coll = N.HostCollectives(None, self._cbs[0], self._cbs[1])
        h = C.c_void_p()
        N.check(N.lib().qs_dist_create_host(C.byref(coll), world, rank, device, C.byref(h)))
        self._h = h
        self.world, self.rank, self.device = world, rank, device
        return self

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.qs_dist_destroy(h)
        self._h = None

    def __del__(self):
        self.close()

    def handle(self):
        return self._h


class ShardedCircuit:
    """A gate list planned for a state with `global_qubits` rank bits."""

    def __init__(self, n, global_qubits, gates):
        arr, keep = N.gate_array(gates)
        h = C.c_void_p()
        N.check(N.lib().qs_plan_create_sharded(n, global_qubits, arr, len(gates), C.byref(h)))
        self._h = h
        self.n = n
        self.g = global_qubits

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.qs_plan_destroy(h)

    def handle(self):
        return self._h

    def steps(self):
        """[(kind, gpos, lpos)] per step; kind 0 per-gate kernel, 1 tile pass,
        2 exchange of rank bits gpos[b] with local qubits lpos[b]."""
        out = []
        k, nb = C.c_int(), C.c_uint32()
        gp, lp = (C.c_uint32 * N.MAX_EXCHANGE_BITS)(), (C.c_uint32 * N.MAX_EXCHANGE_BITS)()
        i = 0
        total = self.stats()["launches"] + self.stats()["exchanges"]
        while i < total:
            N.check(N.lib().qs_plan_step_info(self._h, i, C.byref(k), C.byref(nb), gp, lp))
            out.append((k.value, tuple(gp[:nb.value]), tuple(lp[:nb.value])))
            i += 1
        return out

    def stats(self):
        a, b, c, e = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        N.check(N.lib().qs_plan_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        N.check(N.lib().qs_plan_exchanges(self._h, C.byref(e)))
        return {"passes": a.value, "launches": b.value, "gates": c.value, "exchanges": e.value}


class ShardedState:
    def __init__(self, handle, comm=None):
        self._h = handle
        self._comm = comm  # keeps the communicator alive while the shards exist
        n, g, r, k = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        N.check(N.lib().qs_shards_info(handle, C.byref(n), C.byref(g), C.byref(r), C.byref(k)))
        self.n, self.g, self.first_rank, self.local_count = n.value, g.value, r.value, k.value

    @classmethod
    def local(cls, n, global_qubits, device=0):
        h = C.c_void_p()
        N.check(N.lib().qs_shards_create_local(n, global_qubits, device, C.byref(h)))
        return cls(h)

    @classmethod
    def distributed(cls, n, comm):
        h = C.c_void_p()
        N.check(N.lib().qs_shards_create_dist(n, comm.handle(), C.byref(h)))
        return cls(h, comm)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.qs_shards_destroy(h)
        self._h = None

    def __del__(self):
        self.close()

    def handle(self):
        return self._h

    @property
    def shard_size(self):
        return 1 << (self.n - self.g)

    def local_range(self):
        """Global index range [lo, hi) of the amplitudes held by this handle."""
        lo = self.first_rank * self.shard_size
        return lo, lo + self.local_count * self.shard_size

    def reset(self, basis=0):
        N.check(N.lib().qs_shards_set_basis_state(self._h, basis))

    def amplitudes(self, offset=None, count=None):
        lo, hi = self.local_range()
        offset = lo if offset is None else offset
        count = hi - offset if count is None else count
        out = np.empty(count, dtype=np.complex128)
        N.check(N.lib().qs_shards_get_amplitudes(self._h, N.dptr(out.view(np.float64)), offset, count))
        return out

    def set_amplitudes(self, amps, offset=None):
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        offset = self.local_range()[0] if offset is None else offset
        N.check(N.lib().qs_shards_set_amplitudes(self._h, N.dptr(amps.view(np.float64)), offset, amps.size))

    def apply_circuit(self, gates):
        arr, keep = N.gate_array(gates)
        N.check(N.lib().qs_shards_apply_circuit(self._h, arr, len(gates)))

    def run_circuit(self, gates, basis=0):
        """run(): reset to |basis> fused into the first pass, then `gates`."""
        arr, keep = N.gate_array(gates)
        N.check(N.lib().qs_shards_run_circuit(self._h, basis, arr, len(gates)))

    def execute(self, circuit, sync=True, from_basis=None):
        if from_basis is not None:
            N.check(N.lib().qs_shards_plan_enqueue_from_basis(self._h, circuit.handle(), from_basis))
            if sync:
                self.sync()
            return
        f = N.lib().qs_shards_plan_execute if sync else N.lib().qs_shards_plan_enqueue
        N.check(f(self._h, circuit.handle()))

    def execute_timed(self, circuit):
        """Per-step device times (ms) of one execution, CUDA events on the shard stream."""
        n = len(circuit.steps())
        buf = (C.c_float * max(1, n))()
        N.check(N.lib().qs_shards_plan_execute_timed(self._h, circuit.handle(), buf))
        return list(buf)[:n]

    def stream(self):
        return N.lib().qs_shards_stream(self._h)

    def sync(self):
        N.check(N.lib().qs_shards_sync(self._h))

    def norm_squared(self):
        out = C.c_double()
        N.check(N.lib().qs_shards_norm2(self._h, C.byref(out)))
        return out.value

    def checksum(self):
        out = C.c_double()
        N.check(N.lib().qs_shards_checksum(self._h, C.byref(out)))
        return out.value

    def probabilities(self, qubits):
        qubits = list(qubits)
        out = np.empty(1 << len(qubits), dtype=np.float64)
        q, m = N.uarr(qubits)
        N.check(N.lib().qs_shards_probs(self._h, q, m, N.dptr(out)))
        return out

    def sample(self, uniforms, exact=True):
        u = np.ascontiguousarray(uniforms, dtype=np.float64)
        out = np.empty(u.size, dtype=np.uint64)
        N.check(N.lib().qs_shards_sample(self._h, N.dptr(u), u.size, 1 if exact else 0, out.ctypes.data_as(N._U64P)))
        return out

    def sample_seeded(self, seed, shots, exact=True):
        out = np.empty(shots, dtype=np.uint64)
        N.check(N.lib().qs_shards_sample_seeded(self._h, seed, shots, 1 if exact else 0, out.ctypes.data_as(N._U64P)))
        return out

    def expect_pauli(self, words):
        """words: per-qubit letter strings of length n -> complex array."""
        letters = "".join(words).encode()
        out = np.empty(2 * len(words), dtype=np.float64)
        N.check(N.lib().qs_shards_expect_pauli(self._h, letters, len(words), N.dptr(out)))
        return out.view(np.complex128)
