"""Mid-size images resident on the whole GPU (RDS_OPT_GRID, k_grid.cu): the whole fixed-K loop
in one cooperative launch, G <= #SM slabs of R rows, halos through an L2 mailbox of
{value, tag} words.  Off by default (slower than the stencil on B200).  It runs the stencil's float operations in the same order, so every result must be
bit-identical to the stencil path (grid = 0) -- on ragged shapes, every slab height R = 2..8,
partial last slabs, odd widths, restricted and empty bands, K = 1, 2, warm starts, batches --
and within the north_star tolerances of the fp64 oracle at C1 (1024 x 1024, K = 500)."""
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


def _solve(rds, z, delta, K, grid, warm=None, batch=None, P=None, gamma=0.0):
    H, W = z.shape[-2:] if batch else z.shape
    kw = dict(resident=0, grid=grid, compact=0)
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


# (H, W): R = ceil(H / #SM) rows per slab from 2 (H <= 296) to 8 (H <= 1184 on 148 SMs)
@pytest.mark.parametrize("H,W,delta_rel,K", [(2, 3, math.inf, 5), (5, 7, 0.4, 9),
                                             (33, 129, math.inf, 23), (300, 1000, 0.3, 17),
                                             (450, 64, math.inf, 12), (600, 333, 0.2, 2),
                                             (740, 1024, 0.3, 1), (1000, 999, math.inf, 11),
                                             (1036, 1000, 0.2, 30), (1184, 1024, math.inf, 6),
                                             (1024, 1024, 0.0, 10)])
def test_grid_equals_stencil(rds, H, W, delta_rel, K):
    z = wl.random_image(H, W, seed=H * 7 + W)
    s = rds.Solver(H, W)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    delta = wl.band_delta(delta_rel, s.absmax()) if delta_rel else np.float32(0.0)
    s.close()
    sa, st_a, a, ea = _solve(rds, z, delta, K, 0)
    sb, st_b, b, eb = _solve(rds, z, delta, K, 1)
    assert st_a["resident"] == 0 and st_b["resident"] == 2 and st_b["launches"] == 1
    for k in a:
        assert np.array_equal(a[k], b[k]), (k, H, W, K)
    assert ea == eb
    # the state left behind continues like the stencil's
    sa.solve_continue(5)
    sb.solve_continue(5)
    assert np.array_equal(sa.u(), sb.u()) and np.array_equal(sa.v(), sb.v())
    sa.close()
    sb.close()


def test_grid_repeat_and_warm_batch(rds):
    """Repeated solves on one handle (the mailbox tags grow across launches), a warm start,
    a batch of images side by side (per-image Neumann columns), a selection term P."""
    rng = np.random.default_rng(4)
    H, W = 500, 600
    z = wl.random_image(H, W, seed=8)
    P = rng.uniform(0, 1, (H, W)).astype(np.float32)
    warm = wl.random_state(H, W, 5)
    res = [_solve(rds, z, np.float32(0.3), 33, g, warm=warm, P=P, gamma=1.5) for g in (0, 1)]
    for k in res[0][2]:
        assert np.array_equal(res[0][2][k], res[1][2][k]), k
    s = res[1][0]
    first = s.u()
    assert res[1][1]["resident"] == 2
    for _ in range(3):
        s.set_state(*warm)
        s.solve(*PAR, np.float32(0.3), 33)
        assert s.stats()["resident"] == 2
        assert np.array_equal(s.u(), first)
    B, h, w = 4, 300, 250
    zb = np.clip(rng.normal(0.5, 0.3, (B, h, w)), 0, 1).astype(np.float32)
    rb = [_solve(rds, zb, np.float32(0.3), 25, g, batch=B) for g in (0, 1)]
    assert rb[1][1]["resident"] == 2
    for k in rb[0][2]:
        assert np.array_equal(rb[0][2][k], rb[1][2][k]), (k,)


def test_grid_not_taken(rds):
    """Tolerance solves and images wider than 1024 columns stay on the stencil."""
    z = wl.random_image(512, 512, seed=1)
    s = rds.Solver(512, 512, grid=1)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    st = s.solve_tol(*PAR, math.inf, 400, 1e-3, 10)
    assert st["resident"] == 0
    s.solve(*PAR, math.inf, 10)
    assert s.stats()["resident"] == 2
    s.close()
    zb = wl.random_image(64, 1100, seed=2)
    s = rds.Solver(64, 1100, grid=1)
    s.set_image(zb)
    s.set_fitting(0.8, 0.2)
    s.solve(*PAR, math.inf, 10)
    assert s.stats()["resident"] == 0
    s.close()


@pytest.mark.parametrize("dr", [0.2, math.inf])
def test_grid_c1_oracle(rds, orc, dr):
    """C1 (1024 x 1024) at its stated K = 500 on the resident grid against the fp64 oracle at
    the north_star tolerances (u, rho within 5e-4; mask disagreement <= 5e-4; labels exact)."""
    cfg = wl.CONFIGS["C1"]
    z, P = wl.make_image(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    delta = wl.band_delta(dr, orc.absmax(f))
    s = rds.Solver(cfg.H, cfg.W, grid=1)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    s.solve(5.0, cfg.theta, cfg.tau, delta, cfg.iters)
    assert s.stats()["resident"] == 2
    o = orc.solve(f, delta, 5.0, np.float32(cfg.theta), cfg.tau, cfg.iters)
    assert np.array_equal(s.labels(), o["labels"])
    p1, p2 = s.p()
    for k, g in (("u", s.u()), ("v", s.v()), ("p1", p1), ("p2", p2)):
        err = np.abs(g.astype(np.float64) - o[k]).max()
        assert err <= 5e-4, (k, err)
    assert np.mean(s.mask() != (o["u"] > 0.5)) <= 5e-4
    s.close()
