"""CPU pins of the 3-D oracle (f4, reading R-F4): textbook identities of the
3-D operators, the 2-D oracle as the D = 1 special case, the separately written unrestricted
twin, the ball version of the Cheeger argument, invariants."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

TAU3 = 1.0 / 12.0  # ||grad||^2 <= 12 in 3-D (R-F4)


def test_adjointness_3d(orc):
    rng = np.random.default_rng(1)
    for shape in [(1, 1, 1), (2, 3, 4), (5, 1, 7), (6, 9, 4)]:
        u = rng.standard_normal(shape)
        p = [rng.standard_normal(shape) for _ in range(3)]
        g = orc.grad3(u)
        lhs = sum(float((gi * pi).sum()) for gi, pi in zip(g, p))
        rhs = float((u * orc.div3(*p)).sum())
        assert abs(lhs + rhs) <= 1e-12 * max(1.0, abs(lhs)), shape


def test_div3_is_minus_grad_transpose(orc):
    D, H, W = 2, 3, 4
    n = D * H * W
    G = np.zeros((3 * n, n))
    for k in range(n):
        e = np.zeros(n)
        e[k] = 1.0
        g = orc.grad3(e.reshape(D, H, W))
        G[:, k] = np.concatenate([gi.ravel() for gi in g])
    Dm = np.zeros((n, 3 * n))
    for k in range(3 * n):
        e = np.zeros(3 * n)
        e[k] = 1.0
        Dm[:, k] = orc.div3(*(e[c * n:(c + 1) * n].reshape(D, H, W) for c in range(3))).ravel()
    assert np.array_equal(Dm, -G.T)


@pytest.mark.parametrize("delta_rel", [0.3, math.inf])
def test_single_plane_is_the_2d_method(orc, delta_rel):
    rng = np.random.default_rng(2)
    f = rng.uniform(-1, 1, (17, 23)).astype(np.float32)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    o2 = orc.solve(f, delta, 4.0, np.float32(0.1), 0.125, 30)
    o3 = orc.solve3(f[None], delta, 4.0, np.float32(0.1), 0.125, 30)
    for k in ("u", "v", "p1", "p2"):
        assert np.array_equal(o3[k][0], o2[k]), k
    assert not o3["p3"].any()
    assert np.array_equal(o3["labels"][0], o2["labels"])


def test_unrestricted_equals_plain_twin_3d(orc):
    rng = np.random.default_rng(3)
    for shape in [(1, 1, 1), (3, 4, 5), (7, 6, 9)]:
        f = rng.uniform(-1, 1, shape).astype(np.float32)
        a = orc.solve3(f, np.float32(np.inf), 3.0, np.float32(0.1), TAU3, 25)
        b = orc.solve3_plain(f, 3.0, np.float32(0.1), TAU3, 25)
        for k in ("u", "v", "p1", "p2", "p3"):
            assert np.array_equal(a[k], b[k]), (shape, k)


@pytest.mark.parametrize("lam_r,want", [(2.5, "empty"), (5.0, "ball")])
def test_ball_cheeger(orc, lam_r, want):
    """f = -1 in a ball of radius R, +1 outside, delta = inf.  E(r) = 4 pi r^2 - lambda
    (4/3) pi r^3 is concave in r, so the continuous minimiser over centred balls is the
    empty set (lambda R < 3) or the whole ball (lambda R > 3); on the grid (probe at 40^3,
    R = 10, K = 1500): empty up to lambda R = 3.0, the ball less some surface voxels from
    3.5 on."""
    N, R = 40, 10.0
    k, i, j = np.mgrid[0:N, 0:N, 0:N].astype(np.float64)
    c = (N - 1) / 2
    ball = ((k - c) ** 2 + (i - c) ** 2 + (j - c) ** 2) <= R * R
    f = np.where(ball, -1.0, 1.0).astype(np.float32)
    o = orc.solve3(f, np.float32(np.inf), lam_r / R, np.float32(0.1), TAU3, 1500)
    m = o["u"] > 0.5
    if want == "empty":
        assert not m.any()
    else:
        assert not (m & ~ball).any() and m.sum() >= 0.95 * ball.sum()


def test_invariants_3d(orc):
    rng = np.random.default_rng(4)
    f = rng.uniform(-1, 1, (6, 11, 13)).astype(np.float32)
    for delta_rel in (0.0, 0.4, math.inf):
        delta = wl.band_delta(delta_rel, orc.absmax(f))
        o = orc.solve3(f, delta, 4.0, np.float32(0.1), TAU3, 40)
        lab = o["labels"]
        u0 = (f <= 0).astype(np.float64)
        pn = np.sqrt(o["p1"] ** 2 + o["p2"] ** 2 + o["p3"] ** 2)
        assert pn.max() <= 1 + 1e-12
        assert o["v"].min() >= 0 and o["v"].max() <= 1
        off = lab != 2
        assert np.array_equal(o["u"][off], u0[off]) and np.array_equal(o["v"][off], u0[off])
        assert not o["p1"][off].any() and not o["p2"][off].any() and not o["p3"][off].any()
        assert not o["p1"][:, -1].any() and not o["p2"][:, :, -1].any() and not o["p3"][-1].any()
        if delta_rel == 0.0:
            assert np.array_equal(o["u"], u0)
