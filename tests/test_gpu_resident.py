"""Small images as one resident cluster (RDS_OPT_RESIDENT, k_small.cu): the whole fixed-K
loop in one launch, the state in the cluster's shared memory.  It runs the stencil's float
operations in the same order, so every result must be bit-identical to the stencil path
(resident = 0) -- on ragged shapes, every slab count, partial last slabs, restricted bands,
batches and warm starts -- and within the north_star tolerances of the fp64 oracle on the
paper's image size (C0)."""
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


def _solve(rds, z, delta, K, resident, warm=None, batch=None, P=None, gamma=0.0):
    H, W = z.shape[-2:] if batch else z.shape
    kw = dict(resident=resident, grid=0 if resident == 0 else None)
    s = rds.BatchSolver(batch, H, W, **kw) if batch else rds.Solver(H, W, **kw)
    s.set_image(z)
    s.set_fitting(0.8, 0.2, gamma, P)
    if warm is not None:
        s.set_state(*warm)
    s.solve(*PAR, delta, K)
    st = s.stats()
    p1, p2 = s.p()
    out = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask())
    e = s.energy()
    assert s.check_frame() == 0
    return s, st, out, e


@pytest.mark.parametrize("H,W,delta_rel,K", [(2, 3, math.inf, 5), (5, 7, 0.4, 9),
                                             (31, 17, 0.3, 30), (33, 129, math.inf, 23),
                                             (100, 77, 0.2, 41), (128, 128, math.inf, 200),
                                             (128, 128, 0.2, 200), (130, 250, 0.3, 17),
                                             (255, 131, math.inf, 12), (250, 250, 0.4, 7),
                                             (40, 350, 0.3, 60)])
def test_resident_equals_stencil(rds, H, W, delta_rel, K):
    z = wl.random_image(H, W, seed=H * 7 + W)
    s = rds.Solver(H, W)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    delta = wl.band_delta(delta_rel, s.absmax())
    s.close()
    sa, st_a, a, ea = _solve(rds, z, delta, K, 0)
    sb, st_b, b, eb = _solve(rds, z, delta, K, 1)
    assert st_a["resident"] == 0 and st_b["resident"] == 1 and st_b["launches"] == 1
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert ea == eb
    # the state left behind continues like the stencil's
    sa.solve_continue(5)
    sb.solve_continue(5)
    assert np.array_equal(sa.u(), sb.u()) and np.array_equal(sa.v(), sb.v())
    sa.close()
    sb.close()


def test_resident_c0_oracle(rds, orc):
    """The paper's image size (C0, 128 x 128, K = 200) against the fp64 oracle."""
    cfg = wl.CONFIGS["C0"]
    z, _ = wl.make_image(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2)
    for dr in cfg.delta_rels:
        delta = wl.band_delta(dr, orc.absmax(f))
        s, st, g, _ = _solve(rds, z, delta, cfg.iters, 2)
        assert st["resident"] == 1
        o = orc.solve(f, delta, cfg.lambdas[0], np.float32(cfg.theta), cfg.tau, cfg.iters)
        for k in ("u", "v", "p1", "p2"):
            assert np.abs(g[k].astype(np.float64) - o[k]).max() <= 5e-4, k
        assert np.mean(g["mask"] != (o["u"] > 0.5)) <= 5e-4
        s.close()


def test_resident_warm_batch_selection(rds):
    """Warm start, a batch of images side by side (per-image Neumann columns), a selection
    term P."""
    rng = np.random.default_rng(4)
    H, W = 96, 120
    z = wl.random_image(H, W, seed=8)
    P = rng.uniform(0, 1, (H, W)).astype(np.float32)
    warm = wl.random_state(H, W, 5)
    res = [_solve(rds, z, np.float32(0.3), 33, r, warm=warm, P=P, gamma=1.5)[2] for r in (0, 1)]
    for k in res[0]:
        assert np.array_equal(res[0][k], res[1][k]), k
    for B, h, w in ((5, 40, 36), (5, 40, 70)):
        zb = np.clip(rng.normal(0.5, 0.3, (B, h, w)), 0, 1).astype(np.float32)
        res = [_solve(rds, zb, np.float32(0.3), 25, r, batch=B) for r in (0, 1)]
        assert res[1][1]["resident"] == 1
        for k in res[0][2]:
            assert np.array_equal(res[0][2][k], res[1][2][k]), (B, h, w, k)


def test_resident_not_taken(rds):
    """Tolerance solves stay on the stencil; images too large for one cluster go to the stencil,
    or resident on the whole GPU with RDS_OPT_GRID on (k_grid, stats resident = 2)."""
    z = wl.random_image(128, 128, seed=1)
    s = rds.Solver(128, 128)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    st = s.solve_tol(*PAR, math.inf, 400, 1e-3, 10)
    assert st["resident"] == 0
    s.solve(*PAR, math.inf, 10)
    assert s.stats()["resident"] == 1
    s.close()
    zb = wl.random_image(300, 300, seed=2)   # more than 16 slabs: no single cluster
    for grid, want in ((None, 0), (1, 2)):
        s = rds.Solver(300, 300, grid=grid)
        s.set_image(zb)
        s.set_fitting(0.8, 0.2)
        s.solve(*PAR, math.inf, 10)
        assert s.stats()["resident"] == want
        s.close()
