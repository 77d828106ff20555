"""The warp-specialised stencil (k_stencil_ws.cu, RDS_OPT_WS) runs the same per-pixel operations
as the single-warp pipeline, split into stage chains on different warps: results must be
bit-identical to RDS_OPT_WS = 0, and within the north_star tolerance of the oracle."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

pytestmark = pytest.mark.gpu

KEYS = ("u", "v", "p1", "p2", "mask")


@pytest.fixture(scope="module")
def rds():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_11534_b200 import _build

    _build.build()
    from paper_1807_11534_b200 import rds as _rds

    return _rds


def _solve(rds, z, P, cfg, delta, iters, tol=None, **opt):
    H, W = z.shape
    s = rds.Solver(H, W, compact=0, grid=0, resident=0, **opt)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    if tol is None:
        s.solve(5.0, cfg.theta, cfg.tau, delta, iters)
    else:
        s.solve_tol(5.0, cfg.theta, cfg.tau, delta, iters, tol, 21)  # blocks of 3 x 7
    p1, p2 = s.p()
    out = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask(), stats=s.stats())
    s.close()
    return out


def _image(H, W, seed):
    rng = np.random.default_rng(seed)
    z = (0.25 + 0.5 * (rng.random((H, W)) < 0.4) + 0.15 * rng.standard_normal((H, W)))
    return z.astype(np.float32), None


@pytest.mark.parametrize("shape", [(300, 260), (517, 700), (64, 128), (1000, 1024), (9, 4)])
@pytest.mark.parametrize("kf", [6, 7, 8])
@pytest.mark.parametrize("dr", [0.2, math.inf])
def test_ws_bitwise(rds, shape, kf, dr):
    cfg = wl.CONFIGS["C1"]
    z, P = _image(*shape, seed=shape[0] * 7 + kf)
    delta = np.float32(np.inf) if math.isinf(dr) else np.float32(dr * 0.5)
    K = 3 * kf + 2  # full-depth launches plus a shorter last one
    a = _solve(rds, z, P, cfg, delta, K, k_fuse=kf, ws=1)
    b = _solve(rds, z, P, cfg, delta, K, k_fuse=kf, ws=0)
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), (k, shape, kf, dr)


@pytest.mark.parametrize("dr", [0.2, math.inf])
def test_ws_bitwise_c3(rds, dr):
    cfg = wl.CONFIGS["C3"]
    z, P = wl.make_image(cfg)
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    delta = wl.band_delta(dr, s.absmax())
    s.close()
    a = _solve(rds, z, P, cfg, delta, 50, ws=1)
    b = _solve(rds, z, P, cfg, delta, 50, ws=0)
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), (k, dr)


def test_ws_tolerance_solve(rds):
    """Tolerance solves run their full-depth PLAIN launches on k_stencil_ws: same stop
    iteration and state as the single-warp kernel."""
    cfg = wl.CONFIGS["C1"]
    z, P = wl.make_image(cfg)
    delta = np.float32(0.3)
    a = _solve(rds, z, P, cfg, delta, 400, tol=1e-2, ws=1)
    b = _solve(rds, z, P, cfg, delta, 400, tol=1e-2, ws=0)
    assert a["stats"]["iters"] == b["stats"]["iters"]
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), k


def test_ws_vs_oracle(rds, orc):
    cfg = wl.CONFIGS["C1"]
    z, P = _image(300, 260, seed=3)
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    delta = wl.band_delta(0.3, orc.absmax(f))
    K = 61
    g = _solve(rds, z, P, cfg, delta, K, k_fuse=7, ws=1)
    o = orc.solve(f, delta, 5.0, np.float32(cfg.theta), cfg.tau, K)
    for k in ("u", "v", "p1", "p2"):
        assert np.abs(g[k].astype(np.float64) - o[k]).max() <= 5e-4, k
    assert np.mean(g["mask"] != (o["u"] > 0.5)) <= 5e-4
