"""The persistent K-loop (RDS_OPT_PERSIST, k_loop.cu) runs every block of k_fuse iterations
inside one launch with a barrier between blocks; each item runs the stencil's run_item, so
results must be bit-identical to the launch-per-block form on every shape, k_fuse, K (with
and without a remainder), band, batch, warm start and continuation -- in both barrier forms
(one cluster for <= 16 CTAs, a cooperative grid beyond)."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

pytestmark = pytest.mark.gpu
PAR = (5.0, 0.1, 0.125)


@pytest.fixture(scope="module")
def rds():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_11534_b200 import _build

    _build.build()
    from paper_1807_11534_b200 import rds as _rds

    return _rds


def _solve(rds, z, delta, K, persist, kf=0, warm=None, batch=None, cont=0):
    H, W = z.shape[-2:] if batch else z.shape
    kw = dict(k_fuse=kf, persist=persist, resident=0, grid=0, compact=0)
    s = rds.BatchSolver(batch, H, W, **kw) if batch else rds.Solver(H, W, **kw)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    if warm is not None:
        s.set_state(*warm)
    s.solve(*PAR, delta, K)
    st = s.stats()
    if cont:
        s.solve_continue(cont)
    p1, p2 = s.p()
    out = (s.u(), s.v(), p1, p2, s.mask())
    e = s.energy()
    assert s.check_frame() == 0
    s.close()
    return st, out, e


@pytest.mark.parametrize("H,W,delta_rel,K,kf", [(128, 128, math.inf, 200, 4),
                                                (128, 128, 0.2, 200, 4),
                                                (100, 76, 0.3, 37, 4),
                                                (300, 512, math.inf, 41, 5),
                                                (1024, 1024, 0.2, 30, 6),
                                                (517, 300, 0.05, 50, 7),
                                                (64, 4, 0.4, 23, 4)])
def test_persist_equals_launch_per_block(rds, H, W, delta_rel, K, kf):
    z = wl.gen_voronoi(N=max(H, W), seed=H + W, n_sites=12)[:H, :W].copy()
    z += 0.1 * np.random.default_rng(H).standard_normal(z.shape).astype(np.float32)
    s = rds.Solver(H, W)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    delta = wl.band_delta(delta_rel, s.absmax())
    s.close()
    st0, a, ea = _solve(rds, z, delta, K, 0, kf)
    st1, b, eb = _solve(rds, z, delta, K, 1, kf)
    assert st0["persist"] == 0 and st1["persist"] == 1
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert ea == eb


def test_persist_warm_batch_continue(rds):
    H, W = 160, 200
    z = wl.gen_voronoi(N=200, seed=3, n_sites=9)[:H, :W].copy()
    warm = wl.random_state(H, W, 6)
    a = _solve(rds, z, np.float32(0.3), 29, 0, 4, warm=warm, cont=13)[1]
    b = _solve(rds, z, np.float32(0.3), 29, 1, 4, warm=warm, cont=13)[1]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    zb = np.clip(np.random.default_rng(2).normal(0.5, 0.3, (6, 48, 64)), 0, 1).astype(np.float32)
    a = _solve(rds, zb, np.float32(0.3), 30, 0, 5, batch=6)[1]
    st, b, _ = _solve(rds, zb, np.float32(0.3), 30, 1, 5, batch=6)
    assert st["persist"] == 1
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
