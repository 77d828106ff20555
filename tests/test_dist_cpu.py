"""World-size-2 gloo test of bench.py's replica plumbing (CPU): barrier, max-over-ranks
timing, summed work and the whole-job throughput formula."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    d = bench.Dist()
    try:
        d.barrier()
        t = d.max(10.0 * (rank + 1))           # rank 1 is the slow one: 20 ms
        w = d.sum(1e9 * (rank + 1))            # 1e9 + 2e9 pixel-iterations
        q.put((rank, t, w, bench.throughput(w, t)))
    finally:
        d.close()


def test_replicas_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, w, v in out:
        assert t == 20.0 and w == 3e9
        assert v == pytest.approx(3e9 / 0.020 / 1e9)
