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


def _strip_worker(rank, world, port, q, weighted=False):
    """One rank of a row-strip solve over gloo: torch.distributed point-to-point halo
    exchange, all-reduced max |f|, gathered u (the oracle is every strip's engine).  weighted:
    uneven strips from per-row weights (the balanced partition of restricted solves)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import numpy as np
    import torch.distributed as dist

    from _orc_engine import OracleEngine
    from paper_1807_11534_b200 import strips
    from paper_1807_11534_b200 import workloads as wl

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, W, s, K = 70, 29, 3, 17
        z = wl.gen_voronoi(N=70, seed=5, n_sites=10)[:H, :W].copy()
        wts = np.linspace(1.0, 12.0, H) ** 2 if weighted else None  # heavy bottom rows
        plan = strips.partition(H, world, s, wts)
        me = plan[rank]
        ss = strips.StripSolver(H, W, s, engine=OracleEngine(me.rows, W), weights=wts)
        assert ss.plan == plan
        ss.set_image(z)                       # full image in, the strip's rows used
        ss.set_fitting(0.8, 0.2)
        amax = ss.absmax()
        delta = wl.band_delta(0.3, amax)
        ss.solve(5.0, 0.1, 0.125, delta, K)
        u = ss.gather_u()
        q.put((rank, float(amax), float(delta), None if u is None else u.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,weighted", [(2, False), (3, False), (3, True)])
def test_strips_gloo(orc, world, weighted):
    import numpy as np
    import torch.multiprocessing as mp

    from paper_1807_11534_b200 import workloads as wl

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strip_worker, args=(r, world, port, q, weighted))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=180) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    z = wl.gen_voronoi(N=70, seed=5, n_sites=10)[:70, :29].copy()
    f = orc.fitting(z, 0.8, 0.2)
    amax = orc.absmax(f)
    delta = wl.band_delta(0.3, amax)
    ref = orc.solve(f, delta, 5.0, 0.1, 0.125, 17)
    assert all(o[1] == float(amax) and o[2] == float(delta) for o in out)
    assert np.array_equal(np.array(out[0][3]), ref["u"])


def _strip_tol_worker(rank, world, port, q):
    """One rank: the global q -> q^ (all-reduced radix histograms) and the global stopping rule
    (all-reduced owned-row sums) of a strip-decomposed image, the oracle as every engine."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    from _orc_engine import OracleEngine
    from paper_1807_11534_b200 import strips
    from paper_1807_11534_b200 import workloads as wl

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, W, s = 66, 31, 3
        z = wl.gen_voronoi(N=66, seed=8, n_sites=9)[:H, :W].copy()
        me = strips.partition(H, world, s)[rank]
        ss = strips.StripSolver(H, W, s, engine=OracleEngine(me.rows, W))
        ss.set_image(z)
        ss.set_fitting(0.8, 0.2)
        qh = [float(ss.band_for_fraction(qq)) for qq in (0.0, 1e-3, 0.1, 0.37, 1.0)]
        st = ss.solve_tol(5.0, 0.1, 0.125, ss.band_for_fraction(0.4), 200, 3e-3, 7)
        u = ss.gather_u()
        q.put((rank, qh, st, None if u is None else u.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strips_global_q_and_stop_gloo(orc, world):
    """q^ equals the whole-image oracle's, and the tolerance solve stops at
    the whole-image oracle's iteration with its state."""
    import numpy as np
    import torch.multiprocessing as mp

    from paper_1807_11534_b200 import workloads as wl

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strip_tol_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=180) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    z = wl.gen_voronoi(N=66, seed=8, n_sites=9)[:66, :31].copy()
    f = orc.fitting(z, 0.8, 0.2)
    want = [float(orc.band_for_fraction(f, qq)) for qq in (0.0, 1e-3, 0.1, 0.37, 1.0)]
    ref = orc.solve_tol(f, orc.band_for_fraction(f, 0.4), 5.0, 0.1, 0.125, 200, 3e-3, 7)
    assert 7 < ref["iters"] < 200   # the rule fires inside the run
    for rank, qh, st, _ in out:
        assert qh == want, rank
        assert st["iters"] == ref["iters"] and st["converged"] == 1, (rank, st, ref["iters"])
        assert abs(st["residual"] - ref["residual"]) <= 1e-12 * ref["residual"]
    assert np.array_equal(np.array(out[0][3]), ref["u"])
