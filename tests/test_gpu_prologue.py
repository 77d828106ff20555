"""The prologue form of the stencil (RDS_OPT_PROLOGUE: the warm-up stages above their
dependency cone elided, k_stencil_impl.cuh Act / Prologue) computes every needed value with the
same operations: results must be bit-identical to the loop form, on ragged shapes, every
k_fuse and tolerance solves; the C1 / C2 parity tests against the oracle run with it on (the
library default for images of at most 2^22 pixels)."""
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


def _solve(rds, z, delta, iters, tol=None, **opt):
    cfg = wl.CONFIGS["C1"]
    H, W = z.shape
    s = rds.Solver(H, W, compact=0, grid=0, resident=0, **opt)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2)
    if tol is None:
        s.solve(5.0, cfg.theta, cfg.tau, delta, iters)
    else:
        s.solve_tol(5.0, cfg.theta, cfg.tau, delta, iters, tol, 14)
    p1, p2 = s.p()
    out = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask(), stats=s.stats())
    s.close()
    return out


def _image(H, W, seed):
    rng = np.random.default_rng(seed)
    z = 0.25 + 0.5 * (rng.random((H, W)) < 0.4) + 0.15 * rng.standard_normal((H, W))
    return z.astype(np.float32)


@pytest.mark.parametrize("shape", [(300, 260), (517, 701), (64, 128), (9, 4), (1000, 1024)])
@pytest.mark.parametrize("kf", [1, 3, 6, 7, 8])
@pytest.mark.parametrize("dr", [0.2, math.inf])
def test_prologue_bitwise(rds, shape, kf, dr):
    z = _image(*shape, seed=shape[0] + 13 * kf)
    delta = np.float32(np.inf) if math.isinf(dr) else np.float32(dr * 0.5)
    K = 3 * kf + 2
    a = _solve(rds, z, delta, K, k_fuse=kf, prologue=1)
    b = _solve(rds, z, delta, K, k_fuse=kf, prologue=0)
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), (k, shape, kf, dr)


@pytest.mark.parametrize("rows", [8, 16, 64])
def test_prologue_short_items(rds, rows):
    """Items of a few rows: the prologue covers most of the march."""
    z = _image(700, 512, seed=rows)
    a = _solve(rds, z, np.float32(0.3), 30, k_fuse=7, item_rows=rows, prologue=1)
    b = _solve(rds, z, np.float32(0.3), 30, k_fuse=7, item_rows=rows, prologue=0)
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), k


def test_prologue_tolerance(rds):
    z = _image(512, 512, seed=5)
    a = _solve(rds, z, np.float32(0.3), 300, tol=1e-2, prologue=1)
    b = _solve(rds, z, np.float32(0.3), 300, tol=1e-2, prologue=0)
    assert a["stats"]["iters"] == b["stats"]["iters"]
    for k in KEYS:
        assert np.array_equal(a[k], b[k]), k
