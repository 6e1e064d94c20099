"""One rank of the multi-process sharded run over CUDA-IPC peer memory with
host (gloo) collectives -- test infrastructure for tests/test_shard_ipc_gpu.py.
Several ranks share cuda:0 (NCCL refuses duplicate devices; the host-collective
communicator does not need NCCL).  No kernel waits on another rank: every
exchange is one scatter kernel (or a tile pass with the exchange fused into
its stores) writing into the other ranks' free buffers, then the stream is
drained and the ranks meet at a host barrier.

    python shard_ipc_worker.py <rank> <world> <port> <out.npz> [fuse0|1]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    if len(sys.argv) > 5:
        os.environ["QSB_FUSE_EXCHANGE"] = sys.argv[5]
    import torch
    import torch.distributed as dist
    from paper_2212_14201_b200 import qforge as Q
    from paper_2212_14201_b200.sharded import DistComm, ShardedState
    from test_planner_emu import mixed_gates

    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%s" % port, rank=rank, world_size=world)
    torch.cuda.set_device(0)
    comm = DistComm.host_from_torch(device=0)
    res = {}
    n = 16
    cases = {"random": Q.gen_random_circuit(n, 6, 424242).gates(), "qft": Q.gen_qft(n, 0x2D5).gates(),
             "hea": Q.gen_hea(n, 3, 11).gates(), "mixed": mixed_gates(n, 200, 91)}
    words = ["Z" * n, "X" + "I" * (n - 2) + "X", "I" * (n - 1) + "Y", "Y" + "Z" * (n - 2) + "X"]
    for name, gates in cases.items():
        st = ShardedState.distributed(n, comm)
        st.run_circuit(gates)  # reset fused, rank-bit exchanges over the IPC mappings
        lo, hi = st.local_range()
        res[name + "_amps"] = st.amplitudes(lo, hi - lo)
        res[name + "_range"] = np.array([lo, hi])
        res[name + "_cs"] = np.array([st.checksum(), st.norm_squared()])
        res[name + "_probs"] = st.probabilities([n - 1, 3, n - 2, 0])
        res[name + "_samples"] = st.sample_seeded(7, 4000, True)
        res[name + "_pauli"] = st.expect_pauli(words)
        st.close()
    np.savez(out, **res)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
