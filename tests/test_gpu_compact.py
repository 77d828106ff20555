"""f3: the compacted RD iteration (RDS_OPT_COMPACT) runs the same float
operations per pixel as the dense stencil, so both paths must give the same u, v, rho and
mask value for value (signed zeros aside) on every shape, band and iteration count; the
dense path itself is pinned to the oracle by tests/test_gpu_parity.py, and one case here
checks the compact path against the oracle directly."""
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


def _run(rds, z, delta, K, compact, batch=None, kf=0, lam=5.0, warm=None, P=None, gamma=0.0,
         resident=None, grid=None, rdc_split=None):
    H, W = z.shape[-2:] if batch else z.shape
    kw = dict(compact=compact, k_fuse=kf, resident=resident, grid=grid, rdc_split=rdc_split)
    s = rds.BatchSolver(batch, H, W, **kw) if batch else rds.Solver(H, W, **kw)
    s.set_image(z)
    s.set_fitting(0.8, 0.2, gamma, P)
    if warm is not None:
        s.set_state(*warm)
    s.solve(lam, 0.1, 0.125, delta, K)
    p1, p2 = s.p()
    out = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask(), labels=s.labels())
    return s, out


def _same(a, b):
    for k in a:
        assert np.array_equal(a[k], b[k]), k   # == on floats: -0.0 equals +0.0


@pytest.mark.parametrize("H,W,delta_rel,K", [(1, 1, 0.5, 3), (7, 5, math.inf, 9),
                                             (64, 64, 0.2, 1), (64, 64, 0.2, 2),
                                             (130, 97, 0.1, 50), (257, 300, 0.3, 37),
                                             (200, 131, math.inf, 20), (96, 128, 0.0, 10),
                                             (333, 45, 0.05, 64)])
def test_compact_equals_dense(rds, orc, H, W, delta_rel, K):
    z = wl.gen_voronoi(N=max(H, W), seed=H + W, n_sites=9)[:H, :W].copy()
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(delta_rel, orc.absmax(f)) if delta_rel else np.float32(0.0)
    s_d, d = _run(rds, z, delta, K, 0)
    s_c, c = _run(rds, z, delta, K, 1)
    assert s_c.stats()["compact"] == 1 and s_d.stats()["compact"] == 0
    _same(d, c)
    assert s_c.energy() == s_d.energy()
    assert s_c.check_frame() == 0


def test_compact_oracle(rds, orc):
    z, _ = wl.make_image("C1")
    z = z[:300, :260].copy()
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(0.1, orc.absmax(f))
    s, g = _run(rds, z, delta, 120, 1)
    o = orc.solve(f, delta, *PAR, 120)
    for k in ("u", "v", "p1", "p2"):
        assert np.abs(g[k].astype(np.float64) - o[k]).max() <= 5e-4, k
    assert np.mean(g["mask"] != (o["u"] > 0.5)) <= 5e-4
    assert np.array_equal(g["labels"], o["labels"])


def test_compact_variants(rds):
    """Batch handles (per-image Neumann columns, widths not multiples of 4), the selection
    term, warm starts, every k_fuse of the dense twin, and the auto switch."""
    rng = np.random.default_rng(4)
    zb = rng.uniform(0, 1, (3, 40, 30)).astype(np.float32)
    _, d = _run(rds, zb, np.float32(0.3), 25, 0, batch=3)
    _, c = _run(rds, zb, np.float32(0.3), 25, 1, batch=3)
    _same(d, c)
    z = wl.gen_voronoi(N=150, seed=8, n_sites=12)[:150, :150].copy()
    P = rng.uniform(0, 1, z.shape).astype(np.float32)
    for kf in (1, 4, 7):
        _, d = _run(rds, z, np.float32(0.25), 30, 0, kf=kf, P=P, gamma=1.5)
        _, c = _run(rds, z, np.float32(0.25), 30, 1, kf=kf, P=P, gamma=1.5)
        _same(d, c)
    warm = wl.random_state(150, 150, 3)
    _, d = _run(rds, z, np.float32(0.2), 15, 0, warm=warm)
    _, c = _run(rds, z, np.float32(0.2), 15, 1, warm=warm)
    _same(d, c)
    for d in (np.float32(math.inf), np.float32(0.01)):  # small image: dense is launch bound
        s, _ = _run(rds, z, d, 5, 2, resident=0, grid=0)
        assert s.stats()["compact"] == 1
        s, _ = _run(rds, z, d, 5, 2)               # ... and the resident cluster beats both
        assert s.stats()["compact"] == 0 and s.stats()["resident"] == 1
    z3, _ = wl.make_image("C3")                        # thin scattered band on 4096^2: compact
    s3 = rds.Solver(*z3.shape, compact=2)
    s3.set_image(z3)
    s3.set_fitting(0.8, 0.2)
    am = s3.absmax()
    s3.solve(*PAR, wl.band_delta(0.02, am), 5)
    assert s3.stats()["compact"] == 1
    s3.solve(*PAR, wl.band_delta(0.2, am), 5)
    assert s3.stats()["compact"] == 0


def _decoupled_count(lab, img_w):
    """RD pixels none of whose six stencil neighbours (up, up-right, left, down, down-left,
    right) is RD and which are not on an image's last column (the split's rule, RDS_OPT_RDC_SPLIT;
    the neighbour relation of PAPER.md Eq. 7-9's forward differences / divergence)"""
    rd = lab == 2
    H, W = rd.shape
    pad = np.zeros((H + 2, W + 2), bool)
    pad[1:-1, 1:-1] = rd
    nb = np.zeros_like(rd)
    for di, dj in ((-1, 0), (-1, 1), (0, -1), (1, 0), (1, -1), (0, 1)):
        nb |= pad[1 + di:H + 1 + di, 1 + dj:W + 1 + dj]
    last = (np.arange(W) % img_w) == img_w - 1
    return int((rd & ~nb & ~last[None, :]).sum())


def _component_sizes(lab, img_w):
    """Sizes of the connected components of the RD pixels under the six-neighbour relation of
    the stencil (scipy.ndimage.label with the hexagonal structuring element), seams of a batch
    included as edges (the library's superset)"""
    from scipy import ndimage
    st = np.array([[0, 1, 1], [1, 1, 1], [1, 1, 0]])  # up, up-right, left, right, down-left, down
    cl, n = ndimage.label(lab == 2, structure=st)
    return np.bincount(cl.ravel())[1:]


@pytest.mark.parametrize("case", ["voronoi", "noise", "batch", "warm", "K1", "K2", "P"])
def test_compact_split_equals_unsplit(rds, orc, case):
    """The coupled / decoupled split (RDS_OPT_RDC_SPLIT) gives the unsplit compact path's
    values bit for bit, and its decoupled count equals the host count of RD pixels without an
    RD neighbour."""
    rng = np.random.default_rng(11)
    batch, warm, P, gamma, K, dr = None, None, None, 0.0, 40, 0.1
    if case == "noise":  # C3's recipe (cells 0.2 / 0.8, noise 0.15): a scattered band
        z = wl.gen_voronoi(N=336, seed=9, n_sites=30)[:300, :333].copy()
    elif case == "batch":  # image seams: the last column's right neighbour is EDGE
        z = np.stack([wl.gen_voronoi(N=200, seed=20 + b, n_sites=8)[:, :150] for b in range(3)])
        batch = 3
    else:
        z = wl.gen_voronoi(N=320, seed=5, n_sites=40)[:257, :301].copy()
        z = (z + 0.05 * rng.standard_normal(z.shape)).astype(np.float32)
    if case == "warm":
        warm = wl.random_state(*z.shape, 7)
    if case in ("K1", "K2"):
        K = int(case[1])
    if case == "P":
        P = rng.uniform(0, 1, z.shape).astype(np.float32)
        gamma, dr = 1.0, 0.2
    zf = z.reshape(-1, z.shape[-1])
    f = orc.fitting(zf, 0.8, 0.2, gamma, P)
    delta = wl.band_delta(dr, orc.absmax(f))
    s0, a = _run(rds, z, delta, K, 1, batch=batch, warm=warm, P=P, gamma=gamma, rdc_split=0)
    s1, b = _run(rds, z, delta, K, 1, batch=batch, warm=warm, P=P, gamma=gamma, rdc_split=1)
    st0, st1 = s0.stats(), s1.stats()
    assert st0["compact"] == 1 and st1["compact"] == 1
    assert st0["rdc_decoupled"] == 0
    n_rd = int((b["labels"] == 2).sum())
    # a batch is solved as one H x (B W) frame, the images side by side (rds.h, rds_create_batch)
    frame = np.concatenate(list(b["labels"]), axis=1) if batch else b["labels"]
    want = _decoupled_count(frame, z.shape[-1]) if n_rd >= 4096 else 0
    assert st1["rdc_decoupled"] == want, (st1["rdc_decoupled"], want, n_rd)
    if case in ("noise", "batch"):
        assert want > 0.2 * n_rd
    _same(a, b)
    assert s1.energy() == s0.energy()
    assert s1.check_frame() == 0
    assert st1["rdc_grouped"] == 0
    # split = 2: small connected components of the coupled pixels inside one warp / CTA each
    s2, c = _run(rds, z, delta, K, 1, batch=batch, warm=warm, P=P, gamma=gamma, rdc_split=2)
    st2 = s2.stats()
    assert st2["compact"] == 1 and st2["rdc_decoupled"] == want
    if n_rd >= 4096:
        coupled = n_rd - want
        if batch is None:  # grouped pixels lie in components of <= 1024 pixels and are coupled
            sizes = _component_sizes(b["labels"], z.shape[-1])
            assert sizes.sum() == n_rd
            small = int(sizes[sizes <= 1024].sum()) - want
            assert 0 <= st2["rdc_grouped"] <= small, (st2["rdc_grouped"], small)
        if case in ("noise", "batch"):
            assert st2["rdc_grouped"] > 0.9 * coupled, (st2["rdc_grouped"], coupled)
    else:
        assert st2["rdc_grouped"] == 0
    _same(a, c)
    assert s2.energy() == s0.energy()
    assert s2.check_frame() == 0


def test_compact_grouped_block_sizes(rds, orc):
    """Components of every slot class (2 ... 1024 records) so that the warp, 256-thread and
    1024-thread forms of k_rdc_grp all run: rectangles of RD pixels (z = 0.5, f ~ 0) on a
    pinned ground (z = 0.2 / 0.8), two pixels apart.  All of them are grouped, the result is
    the barrier kernel's bit for bit, and it matches the fp64 oracle."""
    rng = np.random.default_rng(5)
    H, W = 330, 420
    z = np.where(rng.uniform(size=(H, W)) < 0.5, 0.2, 0.8).astype(np.float32)
    shapes = [(1, 2), (2, 3), (3, 5), (5, 8), (7, 9), (10, 20), (12, 21), (20, 30), (25, 40),
              (32, 32), (1, 40), (60, 1), (2, 200)]
    i0 = 2
    n_blob = 0
    while i0 < H - 62:
        j0, hmax = 2, 0
        while True:
            h, w = shapes[n_blob % len(shapes)]
            if j0 + w + 2 > W or i0 + h + 2 > H:
                break
            z[i0:i0 + h, j0:j0 + w] = 0.5 + 0.005 * rng.standard_normal((h, w))
            j0 += w + 2
            hmax = max(hmax, h)
            n_blob += 1
        i0 += hmax + 2
    # isolated RD pixels below the rectangles: the grouping is only tried where at least 15%
    # of the RD pixels are decoupled (the library's scattered-band gate)
    z = np.concatenate([z, np.full((70, W), 0.2, np.float32)])
    z[H + 4:H + 66:2, 2:W - 2:3] = 0.5
    H = z.shape[0]
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(0.1, orc.absmax(f))
    K = 60
    s0, a = _run(rds, z, delta, K, 1, rdc_split=0)
    s2, c = _run(rds, z, delta, K, 1, rdc_split=2)
    st = s2.stats()
    sizes = _component_sizes(c["labels"], W)
    n_rd = int((c["labels"] == 2).sum())
    assert n_rd >= 4096 and sizes.max() <= 1024
    assert st["rdc_decoupled"] >= 0.15 * n_rd
    assert {int(2 ** math.ceil(math.log2(max(2, x)))) for x in sizes if x > 1} >= {2, 8, 64, 256, 1024}
    assert st["rdc_decoupled"] + st["rdc_grouped"] == n_rd, (st, n_rd)
    assert st["rdc_grouped"] == int(sizes[sizes > 1].sum())
    assert 4 <= st["rdc_label_rounds"] <= 16 and st["rdc_label_rounds"] % 4 == 0
    _same(a, c)
    o = orc.solve(f, delta, 5.0, np.float32(0.1), 0.125, K)
    assert np.array_equal(c["labels"], o["labels"])
    for k in ("u", "v", "p1", "p2"):
        assert np.abs(c[k].astype(np.float64) - o[k]).max() <= 5e-4, k


def test_compact_auto_second_chance(rds):
    """Auto mode (RDS_OPT_COMPACT = 2): a scattered band the barrier kernel's cost model leaves
    dense (C1 at delta = 0.2 max|f|, 17% RD, every tile active) is taken by the grouped compact
    path -- every RD pixel decoupled or grouped -- with the dense path's values; with the
    grouping off (split = 1) the same solve stays dense."""
    cfg = wl.CONFIGS["C1"]
    z, P = wl.make_image(cfg)
    out = {}
    for name, kw in (("dense", dict(compact=0)), ("auto", dict(compact=2)),
                     ("auto_nogroup", dict(compact=2, rdc_split=1))):
        s = rds.Solver(cfg.H, cfg.W, **kw)
        s.set_image(z)
        s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
        s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, wl.band_delta(0.2, s.absmax()), 60)
        p1, p2 = s.p()
        out[name] = (s.stats(), dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask()))
        s.close()
    st = out["auto"][0]
    assert out["dense"][0]["compact"] == 0 and out["auto_nogroup"][0]["compact"] == 0
    assert st["compact"] == 1
    assert st["rdc_decoupled"] + st["rdc_grouped"] == st["n_rd"]
    _same(out["dense"][1], out["auto"][1])
    _same(out["dense"][1], out["auto_nogroup"][1])


@pytest.mark.parametrize("split", [1, 2])
def test_compact_split_oracle(rds, orc, split):
    """The split path against the fp64 oracle at the north_star tolerances (a C3-like noise
    band, about half of it decoupled)."""
    z = wl.gen_voronoi(N=320, seed=3, n_sites=20)[:256, :320].copy()
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(0.1, orc.absmax(f))
    s, g = _run(rds, z, delta, 300, 1, rdc_split=split)
    assert s.stats()["rdc_decoupled"] > 0
    assert (s.stats()["rdc_grouped"] > 0) == (split == 2)
    o = orc.solve(f, delta, 5.0, np.float32(0.1), 0.125, 300)
    assert np.array_equal(g["labels"], o["labels"])
    for k in ("u", "v", "p1", "p2"):  # north_star: u, rho within 5e-4, mask <= 0.05%
        err = np.abs(g[k].astype(np.float64) - o[k]).max()
        assert err <= 5e-4, (k, err)
    assert np.mean(g["mask"] != (o["u"] > 0.5)) <= 5e-4


def test_compact_then_continue(rds):
    z = wl.gen_voronoi(N=120, seed=2, n_sites=10)[:120, :120].copy()
    s1, _ = _run(rds, z, np.float32(0.3), 20, 1)
    s1.solve_continue(13)
    s2, _ = _run(rds, z, np.float32(0.3), 33, 0)
    p1a, p2a = s1.p()
    p1b, p2b = s2.p()
    for a, b in ((s1.u(), s2.u()), (s1.v(), s2.v()), (p1a, p1b), (p2a, p2b)):
        assert np.array_equal(a, b)


@pytest.mark.slow
@pytest.mark.parametrize("delta_rel", [0.05, 0.1])
def test_compact_c3_full(rds, delta_rel):
    """Full C3 (4096^2, K = 1000) at the low-band deltas where the compact path pays."""
    z, _ = wl.make_image("C3")
    s_d = rds.Solver(*z.shape)
    s_d.set_image(z)
    s_d.set_fitting(0.8, 0.2)
    delta = wl.band_delta(delta_rel, s_d.absmax())
    s_d.solve(*PAR, delta, 1000)
    s_c = rds.Solver(*z.shape, compact=1)
    s_c.set_image(z)
    s_c.set_fitting(0.8, 0.2)
    s_c.solve(*PAR, delta, 1000)
    assert np.array_equal(s_c.u(), s_d.u())
    assert np.array_equal(s_c.v(), s_d.v())


@pytest.mark.slow
@pytest.mark.parametrize("delta_rel", [0.02, 0.05])
def test_compact_c3_full_oracle(rds, orc, cache, delta_rel):
    """The compact path at full C3 (4096^2) and the config's K = 1000, at the thin bands where
    the bench takes it (restricted_compact), element-wise against the fp64 oracle at the
    north_star tolerances, labels bit-exact."""
    cfg = wl.CONFIGS["C3"]
    z, P = cache.get_or(("C3", "image"), lambda: wl.make_image(cfg))
    f = orc.fitting(z, cfg.c1, cfg.c2)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    s, g = _run(rds, z, delta, cfg.iters, 1)
    assert s.stats()["compact"] == 1
    o = orc.solve(f, delta, *PAR, cfg.iters)
    assert np.array_equal(g["labels"], o["labels"])
    for k in ("u", "v", "p1", "p2"):
        err = np.abs(g[k].astype(np.float64) - o[k]).max()
        assert err <= 5e-4, (k, err)
    assert np.mean(g["mask"] != (o["u"] > 0.5)) <= 5e-4
    s.close()


def _resid(a, b):
    return max(float(np.sqrt(np.sum((a[0].astype(np.float64) - b[0]) ** 2))),
               float(np.sqrt(np.sum((a[1].astype(np.float64) - b[1]) ** 2))))


@pytest.mark.parametrize("img,delta_rel,tol,m", [("C0", math.inf, 1e-2, 10),
                                                 ("C3crop", 0.1, 5e-2, 7),
                                                 ("C3crop", 0.05, 2e-2, 1)])
def test_compact_tolerance(rds, img, delta_rel, tol, m):
    """The stopping rule inside the persistent kernel: it stops at the first check l with
    max(||u^l - u^(l-1)||, ||v^l - v^(l-1)||) <= tol (reading R-F2), leaving
    exactly the fixed-K state of l iterations, at the same l as the dense tolerance solve."""
    if img == "C0":
        z, _ = wl.make_image("C0")
    else:
        z = wl.make_image("C3")[0][:384, :448].copy()
    H, W = z.shape

    def solver(compact):
        s = rds.Solver(H, W, compact=compact)
        s.set_image(z)
        s.set_fitting(0.8, 0.2)
        return s

    s = solver(1)
    d = wl.band_delta(delta_rel, s.absmax())
    st = s.solve_tol(*PAR, d, 2000, tol, m)
    assert st["compact"] == 1
    l = st["iters"]
    assert st["converged"] == 1 and 0 < l < 2000 and (l % m == 0)
    f = solver(1)
    f.solve(*PAR, d, l)
    p1a, p2a = s.p()
    p1b, p2b = f.p()
    for a, b in ((s.u(), f.u()), (s.v(), f.v()), (p1a, p1b), (p2a, p2b), (s.mask(), f.mask())):
        assert np.array_equal(a, b)
    uv = {}
    for k in sorted({l, l - 1, l - m, l - m - 1} - {0, -1} if l > m else {l, l - 1}):
        f.solve(*PAR, d, k)
        uv[k] = (f.u(), f.v())
    r_l = _resid(uv[l], uv[l - 1])
    assert r_l <= tol and abs(r_l - st["residual"]) <= 1e-4 * max(r_l, 1e-12) + 1e-7
    if l > m:
        assert _resid(uv[l - m], uv[l - m - 1]) > tol
    sd = solver(0).solve_tol(*PAR, d, 2000, tol, m)     # the dense twin stops at the same l
    assert sd["compact"] == 0 and sd["iters"] == l


def test_compact_tolerance_batch(rds):
    """A batch handle on the compact path with the stopping rule: same stop and state as the
    dense twin (per-image Neumann columns, widths not multiples of 4)."""
    rng = np.random.default_rng(11)
    zb = np.clip(rng.normal(0.5, 0.3, (4, 36, 22)), 0, 1).astype(np.float32)
    out = []
    for compact in (0, 1):
        s = rds.BatchSolver(4, 36, 22, compact=compact)
        s.set_image(zb)
        s.set_fitting(0.8, 0.2)
        st = s.solve_tol(*PAR, np.float32(0.3), 3000, 1e-3, 5)
        p1, p2 = s.p()
        out.append((st, s.u(), s.v(), p1, p2))
    (sd, *a), (sc, *b) = out
    assert sc["compact"] == 1 and sd["iters"] == sc["iters"] and sc["converged"] == 1
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_compact_tolerance_empty_band(rds):
    """RD empty (q = 0): both paths report the first check (residual 0, converged) and u0."""
    z, _ = wl.make_image("C0")
    out = []
    for compact in (0, 1):
        s = rds.Solver(*z.shape, compact=compact)
        s.set_image(z)
        s.set_fitting(0.8, 0.2)
        st = s.solve_tol(*PAR, np.float32(0.0), 500, 1e-2, 10)
        out.append((st["iters"], st["converged"], st["residual"], s.u()))
    assert out[0][:3] == out[1][:3] == (10, 1, 0.0)
    assert np.array_equal(out[0][3], out[1][3])
