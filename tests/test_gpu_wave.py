"""The temporal wavefront (RDS_OPT_WAVE, k_wave.cu) runs the same per-pixel operations as the
launch-per-block K-loop, only scheduled differently (blocks of k_fuse iterations chained down
each column strip through progress counters), so every result must be bit-identical to the
non-wave solve -- on ragged shapes, sparse bands with gaps between runs, every supported
k_fuse, K with and without a remainder, batches, continue and warm starts (the launch-per-
block path is pinned to the oracle by tests/test_gpu_parity.py).  The wavefront is off by
default (slower on B200); these tests switch it on explicitly."""
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


def _solve(rds, z, delta, K, wave, kf, warm=None, batch=None, cont=0, skip=True):
    H, W = z.shape[-2:] if batch else z.shape
    s = rds.BatchSolver(batch, H, W, k_fuse=kf, wave=wave, skip=skip, resident=0, grid=0, compact=0) if batch \
        else rds.Solver(H, W, k_fuse=kf, wave=wave, skip=skip, resident=0, grid=0, compact=0)
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
    assert s.check_frame() == 0
    s.close()
    return st, out


def _same(a, b):
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("H,W,delta_rel,K,kf", [(300, 260, math.inf, 40, 6),
                                                (517, 300, 0.2, 37, 6),
                                                (640, 512, 0.05, 50, 4),
                                                (256, 1024, 0.4, 23, 5),
                                                (1000, 132, math.inf, 30, 7),
                                                (96, 96, 0.3, 12, 6)])
def test_wave_equals_launch_per_block(rds, H, W, delta_rel, K, kf):
    z = wl.gen_voronoi(N=max(H, W), seed=H + W, n_sites=12)[:H, :W].copy()
    zz = z + 0.1 * np.random.default_rng(H).standard_normal(z.shape).astype(np.float32)
    s = rds.Solver(H, W)
    s.set_image(zz)
    s.set_fitting(0.8, 0.2)
    delta = wl.band_delta(delta_rel, s.absmax())
    s.close()
    st0, a = _solve(rds, zz, delta, K, 0, kf)
    st1, b = _solve(rds, zz, delta, K, 1, kf)
    assert st0["wave"] == 0 and st1["wave"] == 1
    assert st1["launches"] == st0["launches"] and st1["k_fuse"] == kf
    _same(a, b)


def test_wave_gaps_and_skip_off(rds):
    """A sparse band (runs separated by inactive rows and strips without any run) and the
    same image with skipping off (every row active)."""
    H, W = 700, 600
    z = np.full((H, W), 0.2, np.float32)
    z[100:180, 50:500] = 0.5      # band pixels: |f| small
    z[400:420, 300:350] = 0.5
    z += 0.02 * np.random.default_rng(3).standard_normal(z.shape).astype(np.float32)
    for skip in (True, False):
        _, a = _solve(rds, z, np.float32(0.1), 41, 0, 6, skip=skip)
        st, b = _solve(rds, z, np.float32(0.1), 41, 1, 6, skip=skip)
        assert st["wave"] == 1
        _same(a, b)


def test_wave_continue_and_warm_start(rds):
    H, W = 384, 416
    z = wl.gen_voronoi(N=416, seed=5, n_sites=10)[:H, :W].copy()
    warm = wl.random_state(H, W, 9)
    _, a = _solve(rds, z, np.float32(0.3), 25, 0, 6, warm=warm, cont=19)
    _, b = _solve(rds, z, np.float32(0.3), 25, 1, 6, warm=warm, cont=19)
    _same(a, b)


def test_wave_batch(rds):
    rng = np.random.default_rng(2)
    zb = np.clip(rng.normal(0.5, 0.3, (6, 64, 96)), 0, 1).astype(np.float32)
    _, a = _solve(rds, zb, np.float32(0.3), 30, 0, 6, batch=6)
    st, b = _solve(rds, zb, np.float32(0.3), 30, 1, 6, batch=6)
    assert st["wave"] == 1
    _same(a, b)


def test_wave_not_taken(rds):
    """No wavefront where it does not apply: a tolerance solve, fewer than two full blocks,
    an unsupported k_fuse, a width that is not a multiple of 4."""
    z = wl.gen_voronoi(N=200, seed=1, n_sites=8)[:200, :200].copy()
    s = rds.Solver(200, 200, wave=1, k_fuse=6, resident=0, grid=0, compact=0)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    s.solve(*PAR, np.float32(0.3), 11)
    assert s.stats()["wave"] == 0
    s.solve(*PAR, np.float32(0.3), 12)
    assert s.stats()["wave"] == 1
    st = s.solve_tol(*PAR, np.float32(0.3), 100, 1e-3, 6)
    assert st["wave"] == 0
    s.close()
    s = rds.Solver(200, 198, wave=1, k_fuse=6, resident=0, grid=0, compact=0)
    s.set_image(z[:, :198].copy())
    s.set_fitting(0.8, 0.2)
    s.solve(*PAR, np.float32(0.3), 40)
    assert s.stats()["wave"] == 0
    s.close()
    s = rds.Solver(200, 200, wave=1, k_fuse=3, resident=0, grid=0, compact=0)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    s.solve(*PAR, np.float32(0.3), 40)
    assert s.stats()["wave"] == 0
    s.close()
