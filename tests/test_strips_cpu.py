"""Row-strip decomposition on CPU: the partition and halo-exchange plan, and
the protocol run with the oracle as every strip's engine, which must reproduce the
whole-image oracle iterates bit for bit on the owned rows (the dependency-cone argument in
paper_1807_11534_b200/strips.py)."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import strips
from paper_1807_11534_b200 import workloads as wl
from _orc_engine import OracleEngine


@pytest.mark.parametrize("H,G,s", [(100, 1, 3), (100, 2, 3), (101, 3, 5), (64, 4, 2),
                                   (300, 7, 7)])
def test_partition_and_exchange_plan(H, G, s):
    plan = strips.partition(H, G, s)
    owner = np.full(H, -1)
    for st in plan:
        owner[st.lo:st.hi] = st.rank
        assert st.top == (0 if st.rank == 0 else 2 * s)
        assert st.bot == (0 if st.rank == G - 1 else s + 1)
    assert (owner >= 0).all() and (np.diff(owner) >= 0).all()
    sizes = [st.hi - st.lo for st in plan]
    assert max(sizes) - min(sizes) <= 1
    filled = {st.rank: np.zeros(st.rows, bool) for st in plan}
    for src, sr, dst, dr, m in strips.exchange_plan(plan):
        a, b = plan[src], plan[dst]
        for k in range(m):
            g_src, g_dst = a.r0 + sr + k, b.r0 + dr + k
            assert g_src == g_dst                      # the same global row
            assert owner[g_src] == src                 # taken from its owner
            assert not (b.lo <= g_dst < b.hi)          # written into a halo only
            filled[dst][dr + k] = True
    for st in plan:                                    # every halo row refreshed
        halo = np.ones(st.rows, bool)
        halo[st.owned] = False
        assert np.array_equal(filled[st.rank], halo)


def test_partition_rejects_thin_strips():
    with pytest.raises(ValueError):
        strips.partition(30, 4, 5)  # 7-8 rows per strip < the 10-row top halo
    with pytest.raises(ValueError):
        strips.partition(3, 4, 1)
    assert strips.segments(23, 7) == [7, 7, 7, 2]
    assert strips.segments(21, 7) == [7, 7, 7]
    assert strips.segments(0, 7) == []


def _image(H, W, seed):
    return wl.gen_voronoi(N=max(H, W), seed=seed, n_sites=12)[:H, :W].copy()


def _strip_solve(z, plan, c, delta, K, s, par):
    engines = []
    for st in plan:
        e = OracleEngine(st.rows, z.shape[1])
        e.set_image(z[st.r0:st.r0 + st.rows])
        e.set_fitting(*c)
        engines.append(e)
    strips.solve_local(engines, plan, *par, delta, K, s)
    return engines


@pytest.mark.parametrize("H,W,G,s,K,delta_rel", [(60, 37, 2, 3, 14, 0.3),
                                                 (75, 20, 3, 5, 23, math.inf),
                                                 (48, 33, 4, 2, 9, 0.25),
                                                 (40, 16, 2, 1, 6, 0.4)])
def test_strips_reproduce_whole_image_oracle(orc, H, W, G, s, K, delta_rel):
    z = _image(H, W, G * 10 + s)
    c, par = (0.8, 0.2), (5.0, 0.1, 0.125)
    f = orc.fitting(z, *c)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    ref = orc.solve(f, delta, 5.0, 0.1, 0.125, K)
    plan = strips.partition(H, G, s)
    for st, e in zip(plan, _strip_solve(z, plan, c, delta, K, s, par)):
        for k in ("u", "v", "p1", "p2"):
            got = e.st[k][st.owned]
            assert np.array_equal(got, ref[k][st.lo:st.hi]), (st.rank, k)


def test_strips_need_the_halo(orc):
    """With a top halo one segment shorter than 2s the owned rows differ: the halo is not
    a formality (unrestricted band, so every pixel iterates)."""
    H, W, G, s, K = 60, 24, 2, 4, 16
    z = _image(H, W, 7)
    f = orc.fitting(z, 0.8, 0.2)
    ref = orc.solve(f, np.float32(np.inf), 5.0, 0.1, 0.125, K)
    plan = strips.partition(H, G, s)
    short = [strips.Strip(p.rank, p.lo, p.hi, max(0, p.top - s), p.bot) for p in plan]
    engines = _strip_solve(z, short, (0.8, 0.2), np.float32(np.inf), K, s, (5.0, 0.1, 0.125))
    st, e = short[1], engines[1]
    assert not np.array_equal(e.st["u"][st.owned], ref["u"][st.lo:st.hi])


@pytest.mark.parametrize("G,s", [(2, 4), (3, 2), (4, 5)])
def test_local_q_and_tolerance(orc, G, s):
    """One process, G strip engines (the oracle): the summed radix histograms give the whole
    image's q^, and the strip tolerance solve stops where the whole-image oracle does, with
    its state on every owned row."""
    H, W = 61, 27
    z = wl.gen_voronoi(N=61, seed=G * 10 + s, n_sites=8)[:H, :W].copy()
    f = orc.fitting(z, 0.8, 0.2)
    plan = strips.partition(H, G, s)
    engines = []
    for st in plan:
        e = OracleEngine(st.rows, W)
        e.set_image(z[st.r0:st.r0 + st.rows])
        e.set_fitting(0.8, 0.2)
        engines.append(e)
    for q in (0.0, 0.05, 0.5, 0.999, 1.0):
        assert strips.band_for_fraction_local(engines, plan, q, H, W) == \
            orc.band_for_fraction(f, q), q
    delta = orc.band_for_fraction(f, 0.45)
    for m, tol, norm in ((5, 2e-3, "l2"), (3, 1e-4, "rms")):
        st = strips.solve_tol_local(engines, plan, 5.0, 0.1, 0.125, delta, 150, tol, m, s,
                                    norm)
        ref = orc.solve_tol(f, delta, 5.0, 0.1, 0.125, 150, tol, m, norm)
        assert st["iters"] == ref["iters"], (m, st, ref["iters"])
        assert abs(st["residual"] - ref["residual"]) <= 1e-12 * max(ref["residual"], 1e-300)
        for stp, e in zip(plan, engines):
            assert np.array_equal(e.u()[stp.owned], ref["u"][stp.lo:stp.hi])


@pytest.mark.parametrize("H,G,s,seed", [(200, 4, 3, 0), (97, 3, 2, 1), (500, 8, 5, 2),
                                       (64, 2, 1, 3)])
def test_weighted_partition(H, G, s, seed):
    """Balanced cuts: contiguous cover of the rows, every strip owns >= the top halo, and
    without the clamp each strip's weight is within one row's weight of total / G."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0, 1, H) ** 4 * 100 + (np.arange(H) > H // 2) * 50.0
    plan = strips.partition(H, G, s, w)
    top, _ = strips.halo_rows(s)
    assert plan[0].lo == 0 and plan[-1].hi == H
    for a, b in zip(plan, plan[1:]):
        assert a.hi == b.lo
    for p in plan:
        assert p.hi - p.lo >= max(1, top)
    sums = [w[p.lo:p.hi].sum() for p in plan]
    clamped = any(p.hi - p.lo == max(1, top) for p in plan)
    if not clamped:
        assert max(sums) <= w.sum() / G + w.max() + 1e-9
    # skewed weights move the cuts: heavy bottom rows -> shorter bottom strips
    sk = strips.partition(H, G, s, np.linspace(1, 20, H) ** 2)
    assert sk[-1].hi - sk[-1].lo < sk[0].hi - sk[0].lo
    with pytest.raises(ValueError):
        strips.partition(H, G, s, -w)


def test_row_weights_and_weighted_strips_oracle(orc):
    """row_weights of the band labels: RD pixels per row + a floor; a solve on the balanced
    strips reproduces the whole-image oracle bit for bit (owned rows)."""
    H, W, G, s, K = 90, 40, 3, 3, 13
    z = _image(H, W, 11)
    z[: H // 3] = 0.8                     # a flat top third: no RD pixels there
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(0.3, orc.absmax(f))
    labels = orc.labels(f, delta)
    w = strips.row_weights(labels)
    assert np.array_equal(strips.row_weights(labels, cell=None), (labels == 2).sum(axis=1) + 1.0)
    # cells: rows of a band share its count of active 8 x 112 cells
    band = (labels[:8] == 2).any()
    assert w[0] == w[7] == float(band) + 1.0
    plan = strips.partition(H, G, s, w)
    assert plan[0].hi - plan[0].lo > plan[-1].hi - plan[-1].lo   # the empty rows are cheap
    ref = orc.solve(f, delta, 5.0, 0.1, 0.125, K)
    for st, e in zip(plan, _strip_solve(z, plan, (0.8, 0.2), delta, K, s, (5.0, 0.1, 0.125))):
        for k in ("u", "v", "p1", "p2"):
            assert np.array_equal(e.st[k][st.owned], ref[k][st.lo:st.hi]), (st.rank, k)
