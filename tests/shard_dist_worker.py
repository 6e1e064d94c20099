"""Per-rank body of the multi-process sharded-plan tests (test_shard_dist_cpu.py).

Each rank holds only its shard (2^(n-g) amplitudes), replays the tile/op steps
of the sharded plan on it with the host emulator, and performs every rank-bit
exchange itself over torch.distributed (gloo) with the protocol of
NcclTransport::exchange (paper_2212_14201_b200/csrc/shard.cpp): for exchanged
rank bits gpos[b] <-> local bits lpos[b], block d (local bits = d) goes to the
peer whose rank bits are d, and that peer's block a (a = our rank bits) lands
in our block d.
TEST INFRASTRUCTURE ONLY."""
import os

import numpy as np


def block_indices(nl, lpos, d):
    """Local indices whose bits lpos[b] equal bit b of d, ordered by the
    remaining bits ascending (block_index in paper_2212_14201_b200/csrc/kernels.cu)."""
    rest = [p for p in range(nl) if p not in lpos]
    e = np.arange(1 << len(rest), dtype=np.int64)
    idx = np.zeros_like(e)
    for t, p in enumerate(rest):
        idx |= ((e >> t) & 1) << p
    for b, p in enumerate(lpos):
        idx |= ((d >> b) & 1) << p
    return idx


def run(rank, world, port, n, which, seed, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import emu_lib
    import oracle_lib as ol
    from test_planner_emu import mixed_gates
    from paper_2212_14201_b200 import qforge as Q

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        gates = {"mixed": lambda: mixed_gates(n, 200, seed),
                 "random": lambda: Q.gen_random_circuit(n, 5, seed).gates(),
                 "qft": lambda: Q.gen_qft(n, seed % (1 << n)).gates(),
                 "hea": lambda: Q.gen_hea(n, 3, seed).gates()}[which]()
        plan = emu_lib.Plan(n, g, gates)
        nl = n - g
        rng = np.random.default_rng(seed)
        full0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        full0 /= np.linalg.norm(full0)
        shard = full0[rank << nl:(rank + 1) << nl].copy()
        exchanges = 0
        leaks = 0
        for i in range(len(plan)):
            kind, gpos, lpos = plan.step(i)
            if kind == emu_lib.Plan.SWAP:
                k = len(gpos)
                a = sum(((rank >> gpos[b]) & 1) << b for b in range(k))
                reqs, recvs = [], {}
                for d in range(1 << k):
                    if d == a:
                        continue
                    peer = rank
                    for b in range(k):
                        peer = (peer & ~(1 << gpos[b])) | (((d >> b) & 1) << gpos[b])
                    send = torch.from_numpy(shard[block_indices(nl, lpos, d)].view(np.float64).copy())
                    recvs[d] = torch.empty_like(send)
                    reqs += [dist.isend(send, peer), dist.irecv(recvs[d], peer)]
                for r in reqs:
                    r.wait()
                for d, buf in recvs.items():
                    shard[block_indices(nl, lpos, d)] = buf.numpy().view(np.complex128)
                exchanges += 1
            else:
                rc = plan.exec_step(i, rank, shard)
                leaks += rc != 0
        # identical plans on every rank
        meta = torch.tensor([len(plan), exchanges], dtype=torch.int64)
        metas = [torch.zeros_like(meta) for _ in range(world)]
        dist.all_gather(metas, meta)
        parts = [torch.zeros(2 << nl, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64)))
        if rank == 0:
            got = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            want = ol.run_gates(n, gates, state=full0.copy())
            out_q.put({"err": float(np.max(np.abs(got - want))), "leaks": int(leaks), "exchanges": exchanges,
                       "same_plan": all(bool(torch.equal(m, metas[0])) for m in metas)})
        else:
            out_q.put({"leaks": int(leaks)})
    finally:
        dist.destroy_process_group()
