"""GPU checks of the row-strip entry points (rds_solve_continue, rds_get/set_state_rows,
rds_set_energy_rows) and of the strip decomposition on one device: G strip handles with
halos, refreshed every s iterations, reproduce the whole-image librds solve bit for bit on
their owned rows (same float operations per pixel; paper_1807_11534_b200/strips.py)."""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import strips
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


def _image(H, W, seed):
    return wl.gen_voronoi(N=max(H, W), seed=seed, n_sites=25)[:H, :W].copy()


def _state(s):
    p1, p2 = s.p()
    return dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask())


@pytest.mark.parametrize("K1,K2,kf", [(10, 11, 4), (7, 7, 7), (1, 20, 0), (13, 0, 3)])
def test_continue_equals_one_solve(rds, K1, K2, kf):
    z = _image(150, 133, 1)
    a, b = rds.Solver(150, 133, k_fuse=kf), rds.Solver(150, 133, k_fuse=kf)
    for s in (a, b):
        s.set_image(z)
        s.set_fitting(0.8, 0.2)
    delta = wl.band_delta(0.3, a.absmax())
    a.solve(*PAR, delta, K1 + K2)
    b.solve(*PAR, delta, K1)
    b.solve_continue(K2)
    sa, sb = _state(a), _state(b)
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k
    assert b.stats()["iters"] == K1 + K2
    assert b.check_frame() == 0


def test_continue_after_tolerance_solve(rds):
    z = _image(96, 96, 2)
    a, b = rds.Solver(96, 96), rds.Solver(96, 96)
    for s in (a, b):
        s.set_image(z)
        s.set_fitting(0.8, 0.2)
    st = a.solve_tol(*PAR, math.inf, 200, 1e-3, 10)
    n = st["iters"]
    assert 0 < n <= 200
    a.solve_continue(9)
    b.solve(*PAR, math.inf, n + 9)
    sa, sb = _state(a), _state(b)
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k


def test_state_rows_roundtrip(rds):
    import torch

    H, W = 70, 45
    s = rds.Solver(H, W)
    s.set_image(_image(H, W, 3))
    s.set_fitting(0.8, 0.2)
    s.solve(*PAR, math.inf, 12)
    p1, p2 = s.p()
    rows = s.state_rows(10, 7)
    assert rows.shape == (3, 7, W)
    assert np.array_equal(rows[0], s.v()[10:17])
    assert np.array_equal(rows[1], p1[10:17]) and np.array_equal(rows[2], p2[10:17])
    dev = torch.empty((3, 7, W), dtype=torch.float32, device="cuda")
    s.state_rows(10, 7, out=dev)
    assert np.array_equal(dev.cpu().numpy(), rows)
    new = np.random.default_rng(0).uniform(-0.5, 0.5, (3, 4, W)).astype(np.float32)
    s.set_state_rows(H - 4, new)
    assert np.array_equal(s.state_rows(H - 4, 4), new)
    s.set_state_rows(0, torch.from_numpy(new).cuda())
    assert np.array_equal(s.state_rows(0, 4), new)
    assert s.check_frame() == 0
    for bad in ((-1, 3), (H - 2, 3)):
        with pytest.raises(rds.RdsError):
            s.state_rows(*bad)
    with pytest.raises(rds.RdsError):
        s.set_energy_rows(5, H + 1)
    fresh = rds.Solver(H, W)
    with pytest.raises(rds.RdsError):
        fresh.solve_continue(3)
    with pytest.raises(rds.RdsError):
        fresh.state_rows(0, 1)


@pytest.mark.parametrize("H,W,G,s,K,delta_rel,kf,compact", [(257, 190, 2, 7, 40, 0.3, 7, 0),
                                                            (300, 129, 3, 5, 33, math.inf, 4, 0),
                                                            (200, 96, 4, 4, 21, 0.2, 0, 0),
                                                            (181, 77, 3, 3, 10, 0.4, 3, 0),
                                                            (240, 200, 3, 6, 30, 0.1, 0, 1)])
def test_strips_bitwise_whole_image(rds, H, W, G, s, K, delta_rel, kf, compact):
    """(compact = 1: every strip's first segment on the compacted RD path, the rest dense --
    the two paths agree value for value, so the strips still equal the whole image)"""
    z = _image(H, W, G * 100 + s)
    ref = rds.Solver(H, W, k_fuse=kf)
    ref.set_image(z)
    ref.set_fitting(0.8, 0.2)
    delta = wl.band_delta(delta_rel, ref.absmax())
    ref.solve(*PAR, delta, K)
    want = _state(ref)
    e_ref = ref.energy()
    plan = strips.partition(H, G, s)
    engines = []
    for st in plan:
        e = rds.Solver(st.rows, W, k_fuse=kf, compact=compact)
        e.set_image(z[st.r0:st.r0 + st.rows])
        e.set_fitting(0.8, 0.2)
        engines.append(e)
    strips.solve_local(engines, plan, *PAR, delta, K, s)
    tot = dict.fromkeys(("TV_v", "fit_v", "E_u", "D_p", "F_rd"), 0.0)
    for st, e in zip(plan, engines):
        got = _state(e)
        stop = st.owned.stop + (1 if st.bot else 0)   # the row below the owned ones too
        for k in got:
            assert np.array_equal(got[k][st.owned.start:stop],
                                  want[k][st.lo:st.lo + stop - st.owned.start]), (st.rank, k)
        e.set_energy_rows(st.owned.start, st.owned.stop)
        en = e.energy()
        for k in tot:
            tot[k] += en[k]
        assert e.check_frame() == 0
    for k in tot:
        assert tot[k] == pytest.approx(e_ref[k], rel=1e-9, abs=1e-9), k


@pytest.mark.parametrize("name,G,seg,dr", [("C1", 3, 7, 0.2), ("C2", 4, 28, math.inf),
                                           ("C2", 2, 14, 0.1)])
def test_strips_config_vs_oracle(rds, orc, name, G, seg, dr):
    """Row strips on a BASELINE config at full size and its stated K, compared directly with
    the whole-image fp64 oracle (not only with the GPU whole-image solve): every strip's owned
    rows within the north_star tolerances, labels bit-exact."""
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    delta = wl.band_delta(dr, orc.absmax(f))
    lam, K = cfg.lambdas[0], cfg.iters
    plan = strips.partition(cfg.H, G, seg)
    engines = []
    for st in plan:
        e = rds.Solver(st.rows, cfg.W)
        e.set_image(z[st.r0:st.r0 + st.rows])
        e.set_fitting(cfg.c1, cfg.c2, cfg.gamma,
                      None if P is None else np.ascontiguousarray(P[st.r0:st.r0 + st.rows]))
        engines.append(e)
    strips.solve_local(engines, plan, lam, cfg.theta, cfg.tau, delta, K, seg)
    o = orc.solve(f, delta, lam, np.float32(cfg.theta), cfg.tau, K)
    for st, e in zip(plan, engines):
        got = _state(e)
        got["labels"] = e.labels()
        rows = slice(st.lo, st.hi)
        for k in ("u", "v", "p1", "p2"):
            err = np.abs(got[k][st.owned].astype(np.float64) - o[k][rows]).max()
            assert err <= 5e-4, (st.rank, k, err)
        assert np.array_equal(got["labels"][st.owned], o["labels"][rows])
        assert np.mean(got["mask"][st.owned] != (o["u"][rows] > 0.5)) <= 5e-4
        e.close()


def test_torch_default_stream(rds):
    """stream=0 (torch's default stream) is the legacy default stream, not the private one:
    work is ordered with torch's (temporary device inputs are safe) and CUDA events on it
    time the solve."""
    import torch

    H, W = 512, 512
    z = _image(H, W, 9)
    ref = rds.Solver(H, W)
    ref.set_image(z)
    ref.set_fitting(0.8, 0.2)
    ref.solve(*PAR, math.inf, 200)
    s = rds.Solver(H, W, stream=torch.cuda.default_stream().cuda_stream)
    with torch.cuda.stream(torch.cuda.default_stream()):
        s.set_image(torch.from_numpy(z).cuda() * 1.0)   # a temporary freed right after
        s.set_fitting(0.8, 0.2)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.solve(*PAR, math.inf, 200)
        b.record()
        torch.cuda.synchronize()
    assert a.elapsed_time(b) > 0.05
    assert np.array_equal(s.u(), ref.u())


@pytest.mark.parametrize("G,s,m,tol,norm", [(3, 7, 10, 2e-2, "l2"), (4, 5, 7, 3e-4, "rms"),
                                            (2, 14, 14, 5e-2, "l2")])
def test_strips_global_q_and_stop(rds, orc, G, s, m, tol, norm):
    """The paper's q -> q^ knob and stopping rule on a strip-decomposed image (PAPER.md:74-84,
    234-238): summed radix histograms of the strips' owned rows give the whole image's q^
    bit for bit, and the tolerance solve over strips (owned-row sums of rds_continue_check,
    added over strips) stops at the iteration of the whole-image fp64 oracle, with the
    whole-image GPU state on every owned row."""
    cfg = wl.CONFIGS["C1"]
    z, P = wl.make_image(cfg)
    z = z[:300, :257].copy()
    H, W = z.shape
    f = orc.fitting(z, cfg.c1, cfg.c2)
    plan = strips.partition(H, G, s)
    engines = []
    for st in plan:
        e = rds.Solver(st.rows, W)
        e.set_image(z[st.r0:st.r0 + st.rows])
        e.set_fitting(cfg.c1, cfg.c2)
        engines.append(e)
    for q in (0.0, 0.02, 0.3, 1.0):
        assert strips.band_for_fraction_local(engines, plan, q, H, W) == \
            orc.band_for_fraction(f, q), q
    delta = orc.band_for_fraction(f, 0.3)
    st = strips.solve_tol_local(engines, plan, 5.0, cfg.theta, cfg.tau, delta, 600, tol, m, s,
                                norm)
    ref = orc.solve_tol(f, delta, 5.0, np.float32(cfg.theta), cfg.tau, 600, tol, m, norm)
    assert st["iters"] == ref["iters"], (st, ref["iters"])
    assert st["converged"] == int(ref["residual"] <= tol)
    assert abs(st["residual"] - ref["residual"]) <= 2e-2 * ref["residual"]
    whole = rds.Solver(H, W, resident=0)
    whole.set_image(z)
    whole.set_fitting(cfg.c1, cfg.c2)
    whole.solve(5.0, cfg.theta, cfg.tau, delta, st["iters"])
    want = _state(whole)
    for stp, e in zip(plan, engines):
        got = _state(e)
        for k in ("u", "v", "p1", "p2"):
            assert np.array_equal(got[k][stp.owned], want[k][stp.lo:stp.hi]), (stp.rank, k)
        e.close()


def test_abs_histogram_and_continue_check(rds, orc):
    """rds_abs_histogram over a row range equals numpy's count of the |f| bit bytes, and
    rds_continue_check's sums equal (u^l - u^(l-1))^2, (v^l - v^(l-1))^2 summed over the rows
    (from two fixed-K solves of the same handle shape)."""
    H, W = 90, 70
    z = _image(H, W, 4)
    s = rds.Solver(H, W, resident=0)
    s.set_image(z)
    s.set_fitting(0.8, 0.2)
    f = orc.fitting(z, 0.8, 0.2)
    b = np.abs(f).view(np.uint32)
    for r0, r1, prefix, mask, shift in ((0, H, 0, 0, 24), (13, 57, 0x3e000000, 0xff000000, 16),
                                        (40, 41, 0, 0, 0), (5, 5, 0, 0, 8)):
        h = s.abs_histogram(r0, r1, prefix, mask, shift)
        sel = b[r0:r1].ravel()
        sel = sel[(sel & np.uint32(mask)) == np.uint32(prefix)]
        want = np.bincount((sel >> np.uint32(shift)) & np.uint32(255), minlength=256)
        assert np.array_equal(h, want), (r0, r1, prefix, mask, shift)
    delta = np.float32(0.4 * float(orc.absmax(f)))
    s.solve(5.0, 0.1, 0.125, delta, 11)
    ua, va = s.u().astype(np.float64), s.v().astype(np.float64)
    su, sv = s.continue_check(1, 20, 71)
    ub, vb = s.u().astype(np.float64), s.v().astype(np.float64)
    assert su == pytest.approx(((ub - ua)[20:71] ** 2).sum(), rel=1e-6)
    assert sv == pytest.approx(((vb - va)[20:71] ** 2).sum(), rel=1e-6)
    ref = rds.Solver(H, W, resident=0)
    ref.set_image(z)
    ref.set_fitting(0.8, 0.2)
    ref.solve(5.0, 0.1, 0.125, delta, 12)
    assert np.array_equal(ref.u(), s.u()) and np.array_equal(ref.v(), s.v())
    s.continue_check(9, 0, H)   # a multi-launch block
    ref.solve_continue(9)
    assert np.array_equal(ref.u(), s.u()) and np.array_equal(ref.v(), s.v())
    with pytest.raises(rds.RdsError):
        s.continue_check(0, 0, H)
    with pytest.raises(rds.RdsError):
        s.abs_histogram(0, H + 1, 0, 0, 24)
    s.close()
    ref.close()


def test_strips_weighted_cuts_bitwise(rds):
    """Balanced cuts from the GPU's own band labels (a K = 0 solve, strips.row_weights):
    uneven strips, still bit-identical to the whole-image solve."""
    H, W, G, s, K = 300, 160, 3, 5, 27
    z = _image(H, W, 77)
    z[: H // 2] = 0.8                          # flat upper half: no RD pixels there
    ref = rds.Solver(H, W)
    ref.set_image(z)
    ref.set_fitting(0.8, 0.2)
    delta = wl.band_delta(0.3, ref.absmax())
    ref.solve(*PAR, delta, 0)
    w = strips.row_weights(ref.labels())
    plan = strips.partition(H, G, s, w)
    assert plan[0].hi - plan[0].lo > plan[-1].hi - plan[-1].lo
    ref.solve(*PAR, delta, K)
    want = _state(ref)
    engines = []
    for st in plan:
        e = rds.Solver(st.rows, W)
        e.set_image(z[st.r0:st.r0 + st.rows])
        e.set_fitting(0.8, 0.2)
        engines.append(e)
    strips.solve_local(engines, plan, *PAR, delta, K, s)
    for st, e in zip(plan, engines):
        got = _state(e)
        for k in got:
            assert np.array_equal(got[k][st.owned], want[k][st.lo:st.hi]), (st.rank, k)
