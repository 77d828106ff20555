"""GPU parity of batched solves (rds_create_batch): B independent images stacked along
columns, each with its own Neumann last column, must reproduce B independent oracle solves."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rds():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_11534_b200 import _build

    _build.build()
    from paper_1807_11534_b200 import rds as _rds

    return _rds


def _check(g, o, ctx):
    for k in ("u", "v", "p1", "p2"):
        err = np.abs(g[k].astype(np.float64) - o[k]).max()
        assert err <= 5e-4, f"{ctx} {k} {err:.3g}"
    assert np.mean(g["mask"] != (o["u"] > 0.5)) <= 5e-4, ctx
    assert np.array_equal(g["labels"], o["labels"]), ctx


@pytest.mark.parametrize("B,H,W,delta_rel,kf", [(5, 40, 70, 0.3, 0), (3, 33, 129, math.inf, 0),
                                               (7, 45, 64, 0.4, 7), (2, 96, 50, 0.2, 3),
                                               (9, 17, 13, 0.3, 0), (4, 1, 30, math.inf, 5)])
def test_batch_equals_independent_solves(rds, orc, B, H, W, delta_rel, kf):
    rng = np.random.default_rng(B * 1000 + H)
    z = rng.uniform(0, 1, (B, H, W)).astype(np.float32)
    f = np.stack([orc.fitting(z[b], 0.75, 0.25) for b in range(B)])
    delta = wl.band_delta(delta_rel, orc.absmax(f.reshape(B * H, W)))
    s = rds.BatchSolver(B, H, W, k_fuse=kf)
    s.set_image(z)
    s.set_fitting(0.75, 0.25)
    s.solve(4.0, 0.1, 0.125, delta, 60)
    p1, p2 = s.p()
    g = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask(), labels=s.labels())
    e_tot = {k: 0.0 for k in ("E_v", "D_p", "TV_v")}
    for b in range(B):
        o = orc.solve(f[b], delta, 4.0, np.float32(0.1), 0.125, 60)
        _check({k: x[b] for k, x in g.items()}, o, f"image {b}")
        assert not g["p1"][b][-1].any() and not g["p2"][b][:, -1].any()  # own Neumann rows/cols
        e = orc.energy(f[b], 4.0, g["u"][b], g["v"][b], g["p1"][b], g["p2"][b])
        for k in e_tot:
            e_tot[k] += e[k]
    e_g = s.energy()
    for k in e_tot:
        assert abs(e_g[k] - e_tot[k]) <= 1e-5 * max(1.0, abs(e_tot[k])), (k, e_g[k], e_tot[k])
    s.close()


def test_batch_of_paper_size_images(rds, orc):
    """64 images of the paper's size (C0 recipe, seeds 0..63), K = 200, delta = inf."""
    B = 64
    z = np.stack([wl.gen_disk(128, 128, seed=b) for b in range(B)])
    s = rds.BatchSolver(B, 128, 128)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    s.solve(5.0, 0.1, 0.125, np.float32(np.inf), 200)
    u = s.u()
    for b in (0, 17, 63):
        f = orc.fitting(z[b], 0.8, 0.2)
        o = orc.solve(f, np.float32(np.inf), 5.0, np.float32(0.1), 0.125, 200)
        assert np.abs(u[b].astype(np.float64) - o["u"]).max() <= 5e-4, b
    s.close()


def test_batch_errors(rds):
    with pytest.raises(rds.RdsError):
        rds.BatchSolver(0, 64, 16)
    with pytest.raises(rds.RdsError):
        rds.BatchSolver(3, 64, 0)
