"""Multi-process (gloo, CPU) checks of the sharded execution protocol: every
rank plans independently, replays its shard, exchanges half-shards with its
partner, and the gathered state must equal the oracle's."""
import multiprocessing as mp
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(world, n, which, seed):
    import shard_dist_worker

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=shard_dist_worker.run, args=(r, world, port, n, which, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,which", [(2, "mixed"), (2, "random"), (2, "qft"), (4, "hea"), (4, "mixed"), (8, "random")])
def test_sharded_protocol_gloo(world, which):
    n = 12
    res = _launch(world, n, which, 99 + world)
    head = [r for r in res if "err" in r][0]
    assert head["err"] <= 1e-10
    assert head["same_plan"]
    assert all(r["leaks"] == 0 for r in res)
    if which in ("mixed", "random", "hea"):
        assert head["exchanges"] > 0
