"""GPU parity of the 3-D volume path (f4, rds3_*) against the 3-D oracle on seeded inputs, at
the north_star bars: labels bit-exact; u, v, rho within 5e-4 max-abs; mask <= 0.05%."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

pytestmark = pytest.mark.gpu
TAU3 = 1.0 / 12.0


@pytest.fixture(scope="module")
def rds():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_11534_b200 import _build

    _build.build()
    from paper_1807_11534_b200 import rds as _rds

    return _rds


def _solve3(rds, z, c1, c2, lam, delta, K, tau=TAU3):
    s = rds.Solver3(*z.shape)
    s.set_image(z)
    s.set_fitting(c1, c2)
    s.solve(lam, 0.1, tau, delta, K)
    p1, p2, p3 = s.p()
    out = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, p3=p3, mask=s.mask(), labels=s.labels(),
               stats=s.stats(), absmax=s.absmax())
    s.close()
    return out


def _compare(g, o, ctx):
    for k in ("u", "v", "p1", "p2", "p3"):
        err = np.abs(g[k].astype(np.float64) - o[k]).max()
        assert err <= 5e-4, f"{ctx} {k} {err:.3g}"
    dis = np.mean(g["mask"] != (o["u"] > 0.5))
    assert dis <= 5e-4, f"{ctx} mask {dis:.3g}"
    assert np.array_equal(g["labels"], o["labels"]), ctx


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (9, 17, 40), (40, 14, 70),
                                   (20, 30, 33), (1, 37, 61)])
@pytest.mark.parametrize("delta_rel", [0.3, math.inf])
def test_vol_small(rds, orc, shape, delta_rel):
    rng = np.random.default_rng(sum(shape))
    z = rng.uniform(0, 1, shape).astype(np.float32)
    f = orc.fitting(z, 0.75, 0.25)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    g = _solve3(rds, z, 0.75, 0.25, 4.0, delta, 40)
    assert g["absmax"] == orc.absmax(f)
    o = orc.solve3(f, delta, 4.0, np.float32(0.1), TAU3, 40)
    _compare(g, o, f"{shape} d={delta_rel}")
    assert g["stats"]["n_rd"] == int((o["labels"] == 2).sum())


def test_vol_single_plane_matches_2d_oracle(rds, orc):
    z = np.random.default_rng(5).uniform(0, 1, (1, 64, 90)).astype(np.float32)
    f = orc.fitting(z[0], 0.75, 0.25)
    g = _solve3(rds, z, 0.75, 0.25, 4.0, np.float32(0.3), 60, tau=0.125 * 0.6)
    o = orc.solve(f, np.float32(0.3), 4.0, np.float32(0.1), 0.125 * 0.6, 60)
    for k in ("u", "v", "p1", "p2"):
        assert np.abs(g[k][0].astype(np.float64) - o[k]).max() <= 5e-4, k
    assert not g["p3"].any()


@pytest.mark.parametrize("lam_r,want", [(2.5, "empty"), (5.0, "ball")])
def test_vol_ball_cheeger(rds, orc, lam_r, want):
    N, R = 40, 10.0
    k, i, j = np.mgrid[0:N, 0:N, 0:N].astype(np.float64)
    c = (N - 1) / 2
    ball = ((k - c) ** 2 + (i - c) ** 2 + (j - c) ** 2) <= R * R
    # z such that the Chan-Vese f is -1 inside, +1 outside: c1 = 1, c2 = 0 -> f = 1 - 2z
    z = np.where(ball, 1.0, 0.0).astype(np.float32)
    g = _solve3(rds, z, 1.0, 0.0, lam_r / R, np.float32(np.inf), 1500)
    m = g["mask"].astype(bool)
    if want == "empty":
        assert not m.any()
    else:
        assert not (m & ~ball).any() and m.sum() >= 0.95 * ball.sum()


def test_vol_v1_sampled(rds, orc):
    """V1 (256^3) at K = 40: sampled 12^3 blocks against the oracle on cone windows
    (margin 2K+2), plus properties of the whole volume."""
    cfg = wl.VOL_CONFIGS["V1"]
    z = wl.make_volume(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2)
    delta = wl.band_delta(0.2, orc.absmax(f))
    K = 40
    g = _solve3(rds, z, cfg.c1, cfg.c2, cfg.lam, delta, K)
    m = 2 * K + 2
    b = 12
    for (k0, i0, j0) in [(0, 0, 0), (250, 250, 250), (120, 7, 200), (60, 130, 0)]:
        k0, i0, j0 = min(k0, cfg.D - b), min(i0, cfg.H - b), min(j0, cfg.W - b)
        K0, I0, J0 = max(0, k0 - m), max(0, i0 - m), max(0, j0 - m)
        K1, I1, J1 = min(cfg.D, k0 + b + m), min(cfg.H, i0 + b + m), min(cfg.W, j0 + b + m)
        o = orc.solve3(np.ascontiguousarray(f[K0:K1, I0:I1, J0:J1]), delta, cfg.lam,
                       np.float32(cfg.theta), cfg.tau, K)
        sl = (slice(k0 - K0, k0 - K0 + b), slice(i0 - I0, i0 - I0 + b), slice(j0 - J0, j0 - J0 + b))
        gb = {k: g[k][k0:k0 + b, i0:i0 + b, j0:j0 + b] for k in ("u", "v", "p1", "p2", "p3", "mask", "labels")}
        ob = {k: o[k][sl] for k in ("u", "v", "p1", "p2", "p3", "labels")}
        _compare(gb, ob, f"V1 block ({k0},{i0},{j0})")
    pn = np.sqrt(g["p1"].astype(np.float64) ** 2 + g["p2"] ** 2 + g["p3"] ** 2)
    assert pn.max() <= 1 + 1e-5
    off = g["labels"] != 2
    u0 = (f <= 0).astype(np.float32)
    assert np.array_equal(g["u"][off], u0[off]) and np.array_equal(g["v"][off], u0[off])
    assert not g["p3"][-1].any() and not g["p1"][:, -1].any() and not g["p2"][:, :, -1].any()


def test_vol_errors(rds):
    s = rds.Solver3(4, 5, 6)
    z = np.zeros((4, 5, 6), np.float32)
    with pytest.raises(rds.RdsError) as ei:
        s.u()
    assert ei.value.code == rds.RDS_ESTATE
    with pytest.raises(rds.RdsError) as ei:
        s.solve(1.0, 0.1, 1 / 12, 0.5, 10)  # no image yet
    assert ei.value.code == rds.RDS_ESTATE
    z[1, 2, 3] = np.nan
    with pytest.raises(rds.RdsError) as ei:
        s.set_image(z)
    assert ei.value.code == rds.RDS_EINVAL
    z[1, 2, 3] = 0.5
    s.set_image(z)
    s.set_fitting(0.75, 0.25)
    with pytest.raises(rds.RdsError) as ei:
        s.solve(1.0, 0.1, 0.125, 0.5, 10)  # tau > 1/12 in 3-D
    assert ei.value.code == rds.RDS_EINVAL
    with pytest.raises(rds.RdsError):
        s.set_fitting(0.5, 0.5)
    s.solve(1.0, 0.1, 1 / 12, 0.5, 10)
    assert s.u().shape == (4, 5, 6)
    s.close()


@pytest.mark.parametrize("shape", [(3, 5, 7), (9, 17, 40), (40, 14, 70), (33, 61, 29),
                                   (70, 40, 100)])
def test_vol_kfuse_bitwise(rds, shape):
    """k_fuse 1, 2, 3 iterations per pass over the volume (k_vol_step / k_vol_tb) and
    several z-chunk sizes give the same bits: the temporally blocked passes run the same
    per-voxel operations in the same order; K not a multiple of k_fuse exercises the
    remainder pass."""
    rng = np.random.default_rng(sum(shape) + 7)
    z = rng.uniform(0, 1, shape).astype(np.float32)
    res = {}
    for kf, kz in ((1, 0), (2, 0), (3, 0), (2, 5), (3, 8)):
        for K in (1, 2, 5, 7):
            s = rds.Solver3(*shape)
            s.set_kfuse(kf)
            s.set_kz(kz)
            s.set_image(z)
            s.set_fitting(0.75, 0.25)
            d = 0.3 * s.absmax()
            s.solve(4.0, 0.1, TAU3, d, K)
            p1, p2, p3 = s.p()
            out = (s.u(), s.v(), p1, p2, p3, s.mask())
            s.close()
            if K in res:
                for a, b in zip(res[K], out):
                    assert np.array_equal(a, b), (shape, kf, kz, K)
            else:
                res[K] = out


def test_vol_kfuse_errors(rds):
    s = rds.Solver3(4, 5, 6)
    for bad in (-1, 4):
        with pytest.raises(rds.RdsError) as ei:
            s.set_kfuse(bad)
        assert ei.value.code == rds.RDS_EINVAL
    s.close()
