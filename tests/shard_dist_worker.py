"""Per-rank body of the multi-process sharded-plan tests (test_shard_dist_cpu.py).

Each rank holds only its shard (2^(n-g) amplitudes), replays the tile/op steps
of the sharded plan on it with the host emulator, and performs every rank-bit
exchange itself over torch.distributed (gloo): partner = rank ^ 2^gpos, the
half with local bit lpos == 1 - (rank bit gpos) changes hands -- the protocol
of NcclTransport::exchange (paper_2212_14201_b200/csrc/shard.cpp).
TEST INFRASTRUCTURE ONLY."""
import os

import numpy as np


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
                partner = rank ^ (1 << gpos)
                v = 1 - ((rank >> gpos) & 1)
                view = shard.reshape(-1, 2, 1 << lpos)
                send = torch.from_numpy(np.ascontiguousarray(view[:, v, :]).view(np.float64).ravel())
                recv = torch.empty_like(send)
                reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
                for r in reqs:
                    r.wait()
                view[:, v, :] = recv.numpy().view(np.complex128).reshape(view[:, v, :].shape)
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
