"""GPU parity of librds (through the C ABI) against the CPU oracle on seeded inputs.

Bars (BASELINE.json north_star): labels / active tiles / f bit-exact; u and rho within 5e-4
max-abs after the stated iteration count; thresholded mask disagreeing on <= 0.05% of pixels.
"""
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

pytestmark = pytest.mark.gpu

TOL = 5e-4          # u, rho max-abs (north_star)
MASK_FRAC = 5e-4    # <= 0.05% mask disagreement


@pytest.fixture(scope="module")
def rds():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1807_11534_b200 import _build

    _build.build()
    from paper_1807_11534_b200 import rds as _rds

    return _rds


def gpu_solve(rds, z, P, c1, c2, gamma, lam, theta, tau, delta, iters, init=None, **opt):
    H, W = z.shape
    s = rds.Solver(H, W, **opt)
    s.set_image(z)
    s.set_fitting(c1, c2, gamma, P)
    if init is not None:
        s.set_state(*init)
    s.solve(lam, theta, tau, delta, iters)
    p1, p2 = s.p()
    out = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask(), labels=s.labels(),
               f=s.fitting(), tiles=s.active_tiles(), stats=s.stats(), solver=s)
    return out


def compare(g, o, lab=None, tol=TOL, mask_frac=MASK_FRAC, ctx=""):
    for k in ("u", "v", "p1", "p2"):
        err = np.abs(g[k].astype(np.float64) - o[k]).max() if g[k].size else 0.0
        assert err <= tol, f"{ctx} {k} max-abs {err:.3g} > {tol}"
    dis = np.mean(g["mask"] != (o["u"] > 0.5)) if g["mask"].size else 0.0
    assert dis <= mask_frac, f"{ctx} mask disagreement {dis:.3g}"


def _params(cfg):
    return dict(c1=cfg.c1, c2=cfg.c2, gamma=cfg.gamma, theta=cfg.theta, tau=cfg.tau)


# ------------------------------------------------------------------------------------------
# K1 / K2: fitting, labels, tiles bit-exact (all configs at full size, C4 included)
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["C0", "C1", "C2", "C3"])
def test_setup_bitexact(rds, orc, name):
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    f_o = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    am = orc.absmax(f_o)
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    assert s.absmax() == am
    for dr in cfg.delta_rels:
        delta = wl.band_delta(dr, am)
        s.solve(cfg.lambdas[0], cfg.theta, cfg.tau, delta, 0)
        assert np.array_equal(s.fitting(), f_o)
        lab_o = orc.labels(f_o, delta)
        assert np.array_equal(s.labels(), lab_o)
        assert np.array_equal(s.active_tiles(), orc.tiles(lab_o, 32, 32))
        st = s.stats()
        assert st["n_rd"] == int((lab_o == 2).sum())
        h = (f_o <= 0)
        assert np.array_equal(s.u(), h.astype(np.float32))          # K = 0 -> u = H(-f)
        assert np.array_equal(s.mask(), h.astype(np.uint8))
    s.close()


@pytest.fixture(scope="module")
def c4(orc, cache):
    cfg = wl.CONFIGS["C4"]

    def build():
        z, P = wl.make_image(cfg)
        f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
        return z, P, f, orc.absmax(f)

    return cfg, cache.get_or(("C4", "image"), build)


@pytest.mark.slow
def test_setup_bitexact_c4(rds, orc, c4):
    cfg, (z, P, f_o, am) = c4
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    assert s.absmax() == am
    delta = wl.band_delta(0.2, am)
    s.solve(5.0, cfg.theta, cfg.tau, delta, 0)
    assert np.array_equal(s.fitting(), f_o)
    lab_o = orc.labels(f_o, delta)
    assert np.array_equal(s.labels(), lab_o)
    assert np.array_equal(s.active_tiles(), orc.tiles(lab_o, 32, 32))
    s.close()


def _window_oracle(orc, f, delta, lam, cfg, K, r0, c0, h, w):
    """Oracle u, v, rho on the block [r0, r0+h) x [c0, c0+w) of a full-size solve, computed
    on a window with a margin of K+1 rows / columns on every side: the error a window cut
    introduces advances at most one row / column per iteration in each direction, so the
    block's values after K iterations equal the full-image iteration's bit for bit (proof in
    DESIGN.md §2 "window margin"; pinned by test_oracle_pins.py::test_cone_margin_k_plus_1,
    which also shows a margin of K-1 is not enough)."""
    H, W = f.shape
    m = K + 1
    R0, R1 = max(0, r0 - m), min(H, r0 + h + m)
    C0, C1 = max(0, c0 - m), min(W, c0 + w + m)
    o = orc.solve(np.ascontiguousarray(f[R0:R1, C0:C1]), delta, lam, np.float32(cfg.theta),
                  cfg.tau, K)
    sl = (slice(r0 - R0, r0 - R0 + h), slice(c0 - C0, c0 - C0 + w))
    return {k: o[k][sl] for k in ("u", "v", "p1", "p2", "labels")}


# |rho| <= 1 is algebraic (|rho + tau g| / (1 + tau |g|) <= 1 when |rho| <= 1).
# In the fp32 kernel the update is rho' = fma(g, tau, rho) * rcp.approx(fma(sqrt.approx(s), tau,
# 1)) with s = fma(g1, g1, fma(g2, g2, |c'|)); with relative errors e_r, e_s of the two MUFU ops
# and u = 2^-24 per rounding, |rho'| <= max(1, |rho|) (1 + e_r + e_s + 4u) to first order
# (reading R-G1), so after K steps |rho| <= (1 + RHO_STEP_EXCESS)^K.  e_r, e_s are
# the exhaustively measured maxima over every float input (scripts/micro/mufu_err.cu,
# profiles/micro_mufu_err.txt: sqrt 2^-23.25, rcp 2^-23.28 on B200), rounded up to 2^-23.
MUFU_SQRT_REL_ERR = 2.0 ** -23
MUFU_RCP_REL_ERR = 2.0 ** -23
RHO_STEP_EXCESS = MUFU_SQRT_REL_ERR + MUFU_RCP_REL_ERR + 4 * 2.0 ** -24


def rho_bound(K):
    return (1.0 + RHO_STEP_EXCESS) ** K


@pytest.mark.slow
@pytest.mark.parametrize("dr", [0.2, math.inf])
def test_c4_full_size(rds, orc, c4, dr):
    """C4 (16384^2, 64 blocks of the selection-term generator) at full size, in the bench's
    launch configuration and at the config's stated K = 1000: (i) sampled 48x48 blocks
    (image corners, block seams, interior) against the oracle on K+1-margin windows, at the
    north_star tolerances; (ii) properties that hold at any size on the whole image."""
    cfg, (z, P, f, am) = c4
    delta = wl.band_delta(dr, am)
    lam, K = cfg.lambdas[0], cfg.iters
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    s.solve(lam, cfg.theta, cfg.tau, delta, K)
    g = {"u": s.u(), "v": s.v()}
    g["p1"], g["p2"] = s.p()
    mask = s.mask()
    lab = s.labels()
    assert np.array_equal(lab, orc.labels(f, delta))
    H, W, b = cfg.H, cfg.W, 48
    blocks = [(0, 0), (H - b, W - b), (2048 - b // 2, 2048 - b // 2),
              (8192 - b // 2, 6144 - b // 2), (11000, 3000)]
    for r0, c0 in blocks:
        o = _window_oracle(orc, f, delta, lam, cfg, K, r0, c0, b, b)
        gb = {k: g[k][r0:r0 + b, c0:c0 + b] for k in g}
        gb["mask"] = mask[r0:r0 + b, c0:c0 + b]
        assert np.array_equal(lab[r0:r0 + b, c0:c0 + b], o["labels"])
        compare(gb, o, ctx=f"C4 d={dr} block ({r0},{c0}) K={K}")
    v, p1, p2 = g["v"], g["p1"], g["p2"]
    assert v.min() >= 0 and v.max() <= 1
    off = lab != 2
    u0 = (f <= 0).astype(np.float32)
    assert np.array_equal(g["u"][off], u0[off]) and np.array_equal(v[off], u0[off])
    assert not p1[off].any() and not p2[off].any()
    assert not p1[-1].any() and not p2[:, -1].any()
    pn = np.hypot(p1.astype(np.float64), p2.astype(np.float64)).max()
    assert pn <= rho_bound(K), pn
    print(f"C4 d={dr}: max|rho| - 1 = {pn - 1:.3g} (derived bound {rho_bound(K) - 1:.3g})")
    del g, v, p1, p2, mask
    e = s.energy()
    assert e["gap"] >= -1e-6 * abs(e["E_v"])
    s.close()


# ------------------------------------------------------------------------------------------
# K3: the iteration on small and ragged shapes, every fusion depth, warm starts
# ------------------------------------------------------------------------------------------

SHAPES = [(1, 1), (1, 7), (9, 1), (5, 3), (33, 129), (100, 77), (130, 250), (257, 131)]


@pytest.mark.parametrize("path", ["stencil", "grid", "default"])
@pytest.mark.parametrize("shape", SHAPES)
def test_ragged_shapes(rds, orc, shape, path):
    """(stencil: the tiled stencil; grid: resident on the whole GPU, k_grid; default: the
    library's choice, the resident cluster where the shape fits one)"""
    opt = {"stencil": dict(resident=0, grid=0, compact=0), "grid": dict(resident=0, grid=1),
           "default": {}}[path]
    H, W = shape
    z = wl.random_image(H, W, seed=H * 1000 + W)
    for dr in (0.0, 0.3, math.inf):
        f = orc.fitting(z, 0.8, 0.2)
        delta = wl.band_delta(dr, orc.absmax(f))
        for iters in (1, 8, 23):
            g = gpu_solve(rds, z, None, 0.8, 0.2, 0.0, 5.0, 0.1, 0.125, delta, iters, **opt)
            o = orc.solve(f, delta, 5.0, np.float32(0.1), 0.125, iters)
            assert np.array_equal(g["labels"], o["labels"])
            if path == "grid":
                assert g["stats"]["resident"] == 2
            compare(g, o, tol=1e-5, mask_frac=0.0 if H * W < 2000 else MASK_FRAC,
                    ctx=f"{shape} d={dr} K={iters}")


@pytest.mark.parametrize("persist", [0, 1])
@pytest.mark.parametrize("kf", [1, 2, 3, 4, 5, 6, 7, 8])
def test_every_fusion_depth(rds, orc, kf, persist):
    """Each KF (iterations per HBM round trip) and each remainder stage count matches the
    oracle; item rows small so many chunk seams are crossed."""
    H, W = 150, 300
    z = wl.random_image(H, W, seed=kf)
    f = orc.fitting(z, 0.75, 0.25)
    delta = wl.band_delta(0.4, orc.absmax(f))
    for iters in (kf, 2 * kf + 1, 3 * kf + kf - 1):
        g = gpu_solve(rds, z, None, 0.75, 0.25, 0.0, 2.0, 0.1, 0.125, delta, iters, k_fuse=kf,
                      item_rows=40, resident=0, grid=0, persist=persist, compact=0)
        o = orc.solve(f, delta, 2.0, np.float32(0.1), 0.125, iters)
        compare(g, o, tol=1e-5, ctx=f"kf={kf} K={iters}")


def test_warm_start_random_state(rds, orc):
    """One and several iterations from a random (v, rho) state: exercises every term of the
    update with O(1) values, not just the smooth evolution from H(-f)."""
    H, W = 96, 200
    z = wl.random_image(H, W, seed=77)
    f = orc.fitting(z, 0.8, 0.2)
    v, p1, p2 = wl.random_state(H, W, 78)
    for dr in (0.5, math.inf):
        delta = wl.band_delta(dr, orc.absmax(f))
        for iters in (1, 2, 9):
            g = gpu_solve(rds, z, None, 0.8, 0.2, 0.0, 5.0, 0.1, 0.125, delta, iters,
                          init=(v, p1, p2), resident=0, grid=0)
            o = orc.solve(f, delta, 5.0, np.float32(0.1), 0.125, iters,
                          init=(v.astype(np.float64), p1.astype(np.float64),
                                p2.astype(np.float64)))
            compare(g, o, tol=2e-5, mask_frac=1e-3, ctx=f"warm d={dr} K={iters}")


def test_fusion_depth_equivalence(rds):
    """k=1 and k=KF run the same per-pixel arithmetic (every operation an explicit rounded
    intrinsic, so no instantiation may contract differently): results are bit-identical."""
    cfg = wl.CONFIGS["C1"]
    z, P = wl.make_image(cfg)
    res = []
    for kf in (1, 3, 7):
        g = gpu_solve(rds, z, P, cfg.c1, cfg.c2, cfg.gamma, 5.0, cfg.theta, cfg.tau,
                      np.float32(0.2), 23, k_fuse=kf, compact=0, grid=0)
        res.append(g)
    for g in res[1:]:
        for k in ("u", "v", "p1", "p2", "mask"):
            assert np.array_equal(g[k], res[0][k]), k


def test_skip_equivalence_and_determinism(rds):
    """Tile skipping never changes the result (pinned pixels are fixed points), and repeated
    solves are bit-identical."""
    cfg = wl.CONFIGS["C2"]
    z, P = wl.make_image(cfg)
    am = np.float32(0)
    s = rds.Solver(cfg.H, cfg.W, compact=0)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    am = s.absmax()
    delta = wl.band_delta(0.2, am)
    outs = []
    for skip in (1, 1, 0):
        s.set_option(rds.RDS_OPT_SKIP, skip)
        s.solve(5.0, cfg.theta, cfg.tau, delta, 40)
        p1, p2 = s.p()
        outs.append((s.u(), s.v(), p1, p2))
    st = s.stats()
    assert st["n_active_cells"] == st["n_items"]  # last run: skip off -> every cell
    for a, b in zip(outs[0], outs[1]):      # identical configuration: bit-identical
        assert a.tobytes() == b.tobytes()
    for a, b in zip(outs[0], outs[2]):      # skip on vs off: same values (a processed pinned
        assert np.array_equal(a, b)         # pixel may hold -0.0 where a skipped one holds +0.0)
    s.close()


# ------------------------------------------------------------------------------------------
# configs at their stated sizes / iteration counts
# ------------------------------------------------------------------------------------------

def _run_cfg(rds, orc, name, lam, dr, iters=None, **opt):
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    delta = wl.band_delta(dr, orc.absmax(f))
    K = cfg.iters if iters is None else iters
    g = gpu_solve(rds, z, P, cfg.c1, cfg.c2, cfg.gamma, lam, cfg.theta, cfg.tau, delta, K,
                  **opt)
    o = orc.solve(f, delta, lam, np.float32(cfg.theta), cfg.tau, K)
    assert np.array_equal(g["labels"], o["labels"])
    assert np.array_equal(g["tiles"], orc.tiles(o["labels"], 32, 32))
    compare(g, o, ctx=f"{name} lam={lam} d={dr} K={K}")
    return g, o


@pytest.mark.parametrize("resident", [0, 2])
@pytest.mark.parametrize("dr", [0.2, math.inf])
def test_c0(rds, orc, dr, resident):
    g, o = _run_cfg(rds, orc, "C0", 5.0, dr, resident=resident, grid=0)
    assert g["stats"]["resident"] == (1 if resident else 0)


@pytest.mark.parametrize("grid", [0, 1])
@pytest.mark.parametrize("lam,dr", [(5.0, 0.05), (5.0, 0.1), (5.0, 0.2), (5.0, 0.4),
                                    (2.0, 0.2), (10.0, 0.2), (5.0, math.inf)])
def test_c1(rds, orc, lam, dr, grid):
    """(grid 0: the default, the stencil or the compact path; 1: resident on the GPU)"""
    g, _ = _run_cfg(rds, orc, "C1", lam, dr, grid=grid)
    if grid:
        assert g["stats"]["resident"] == 2


@pytest.mark.parametrize("dr", [0.05, 0.1, 0.2, 0.4, math.inf])
def test_c2(rds, orc, dr):
    _run_cfg(rds, orc, "C2", 5.0, dr)


@pytest.mark.parametrize("dr", [0.1, math.inf])
def test_c3_reduced_iters(rds, orc, dr):
    """C3 at full size in the bench's launch configuration, K=60 (oracle cost bound)."""
    _run_cfg(rds, orc, "C3", 5.0, dr, iters=60)


@pytest.mark.slow
@pytest.mark.parametrize("dr", [0.1, 0.2, 0.4, math.inf])
def test_c3_full(rds, orc, cache, dr):
    """C3 (the headline) at full size and its stated K = 1000, every delta of the bench sweep,
    element-wise against the fp64 oracle at the north_star tolerances."""
    cfg = wl.CONFIGS["C3"]
    z, P = cache.get_or(("C3", "image"), lambda: wl.make_image(cfg))
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    delta = wl.band_delta(dr, orc.absmax(f))
    K = cfg.iters
    g = gpu_solve(rds, z, P, cfg.c1, cfg.c2, cfg.gamma, 5.0, cfg.theta, cfg.tau, delta, K)
    o = orc.solve(f, delta, 5.0, np.float32(cfg.theta), cfg.tau, K)
    assert np.array_equal(g["labels"], o["labels"])
    assert np.array_equal(g["tiles"], orc.tiles(o["labels"], 32, 32))
    compare(g, o, ctx=f"C3 d={dr} K={K}")
    errs = {k: float(np.abs(g[k].astype(np.float64) - o[k]).max()) for k in ("u", "p1", "p2")}
    print(f"C3 d={dr} K={K}: max-abs {errs}, mask disagreement "
          f"{np.mean(g['mask'] != (o['u'] > 0.5)):.3g}")
    g["solver"].close()


def test_c3_full_properties(rds, orc, cache):
    """Headline config, full K: properties that hold at any size -- |rho| <= 1, v in [0,1],
    exact pinning, Neumann zeros, weak-duality gap >= 0 (GPU energy), labels bit-exact."""
    cfg = wl.CONFIGS["C3"]
    z, P = cache.get_or(("C3", "image"), lambda: wl.make_image(cfg))
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    am = orc.absmax(f)
    for dr in (0.1, math.inf):
        delta = wl.band_delta(dr, am)
        g = gpu_solve(rds, z, P, cfg.c1, cfg.c2, cfg.gamma, 5.0, cfg.theta, cfg.tau, delta,
                      cfg.iters)
        lab = orc.labels(f, delta)
        assert np.array_equal(g["labels"], lab)
        pn = np.sqrt(g["p1"].astype(np.float64) ** 2 + g["p2"].astype(np.float64) ** 2)
        # |rho| <= 1 is algebraic; the fp32 kernel's excess is bounded per step by the MUFU
        # and rounding errors (rho_bound, derived above); the measured excess is reported
        assert pn.max() <= rho_bound(cfg.iters), pn.max()
        print(f"C3 d={dr}: max|rho| - 1 = {pn.max() - 1:.3g} "
              f"(derived bound {rho_bound(cfg.iters) - 1:.3g})")
        assert g["v"].min() >= 0 and g["v"].max() <= 1
        off = lab != 2
        u0 = (f <= 0).astype(np.float32)
        assert np.array_equal(g["u"][off], u0[off]) and np.array_equal(g["v"][off], u0[off])
        assert not g["p1"][off].any() and not g["p2"][off].any()
        assert not g["p1"][-1].any() and not g["p2"][:, -1].any()
        e = g["solver"].energy()
        assert e["gap"] >= -1e-6 * abs(e["E_v"])
        g["solver"].close()


# ------------------------------------------------------------------------------------------
# K5 energy, API behaviour
# ------------------------------------------------------------------------------------------

def test_energy_matches_oracle(rds, orc):
    """GPU energies equal the oracle's energies evaluated on the GPU's own state."""
    cfg = wl.CONFIGS["C1"]
    z, P = wl.make_image(cfg)
    for dr in (0.2, math.inf):
        g = gpu_solve(rds, z, P, cfg.c1, cfg.c2, cfg.gamma, 5.0, cfg.theta, cfg.tau,
                      wl.band_delta(dr, np.float32(0.7637)), 50)
        e_g = g["solver"].energy()
        e_o = orc.energy(g["f"], 5.0, g["u"], g["v"], g["p1"], g["p2"])
        for k in ("E_v", "E_u", "D_p", "TV_v", "fit_v"):
            assert abs(e_g[k] - e_o[k]) <= 1e-5 * max(1.0, abs(e_o[k])), (k, e_g[k], e_o[k])
        assert e_g["gap"] >= 0
        assert abs(e_g["gap"] - e_o["gap"]) <= 1e-5 * abs(e_o["E_v"])
        g["solver"].close()


def test_errors(rds):
    s = rds.Solver(16, 16)
    with pytest.raises(rds.RdsError) as ei:
        s.u()
    assert ei.value.code == rds.RDS_ESTATE
    with pytest.raises(rds.RdsError) as ei:
        s.solve(5.0, 0.1, 0.125, 0.1, 10)
    assert ei.value.code == rds.RDS_ESTATE
    z = np.zeros((16, 16), np.float32)
    s.set_image(z)
    with pytest.raises(rds.RdsError):
        s.set_fitting(0.5, 0.5)
    with pytest.raises(rds.RdsError):
        s.set_fitting(0.8, 0.2, 1.0, None)
    s.set_fitting(0.8, 0.2)
    for bad in [(0.0, 0.1, 0.125, 0.1, 1), (5.0, 0.0, 0.125, 0.1, 1), (5.0, 0.1, 0.2, 0.1, 1),
                (5.0, 0.1, 0.125, -1.0, 1), (5.0, 0.1, 0.125, float("nan"), 1),
                (5.0, 0.1, 0.125, 0.1, -1)]:
        with pytest.raises(rds.RdsError) as ei:
            s.solve(*bad)
        assert ei.value.code == rds.RDS_EINVAL
    zn = z.copy()
    zn[3, 3] = np.nan
    with pytest.raises(rds.RdsError):
        s.set_image(zn)
    with pytest.raises(rds.RdsError):
        s.solve(5.0, 0.1, 0.125, 0.1, 1)
    s.set_image(z)
    s.solve(5.0, 0.1, 0.125, 0.1, 1)
    s.close()


def test_device_buffers_and_stream(rds, orc):
    """torch CUDA tensors in/out (on_device=1) on a user stream give the same bytes as the
    host path."""
    import torch

    cfg = wl.CONFIGS["C0"]
    z, _ = wl.make_image(cfg)
    host = gpu_solve(rds, z, None, cfg.c1, cfg.c2, 0.0, 5.0, cfg.theta, cfg.tau, np.inf, 200)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        zt = torch.from_numpy(z).cuda()
        s = rds.Solver(*z.shape, stream=st.cuda_stream)
        s.set_image(zt)
        s.set_fitting(cfg.c1, cfg.c2)
        s.solve(5.0, cfg.theta, cfg.tau, np.inf, 200)
        ut = torch.empty(z.shape, dtype=torch.float32, device="cuda")
        mt = torch.empty(z.shape, dtype=torch.uint8, device="cuda")
        s.u(ut)
        s.mask(mt)
    st.synchronize()
    assert ut.cpu().numpy().tobytes() == host["u"].tobytes()
    assert mt.cpu().numpy().tobytes() == host["mask"].tobytes()
    s.close()


# ------------------------------------------------------------------------------------------
# q -> q^, NEXT item f1
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["C0", "C2", "C3"])
def test_band_for_fraction_exact(rds, orc, name):
    """GPU radix select of the q -> q^ threshold equals the oracle's sort, bit for bit, and
    rds_solve_q labels the requested fraction (ties join RD)."""
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    N = cfg.H * cfg.W
    for q in ((0.0, 1e-6, 0.1, 0.25, 0.5, 0.9, 1.0) if N < 10**7 else (0.0, 0.1, 0.5, 1.0)):
        qh = s.band_for_fraction(q)
        assert qh == orc.band_for_fraction(f, q), q
        s.solve_q(cfg.lambdas[0], cfg.theta, cfg.tau, q, 0)
        lab = s.labels()
        assert np.array_equal(lab, orc.labels(f, qh))
        assert (lab == 2).sum() >= np.ceil(q * N)
    s.close()


# ------------------------------------------------------------------------------------------
# f2: tolerance solves -- stopping rule fused into the stencil
# ------------------------------------------------------------------------------------------

def _tol_case(rds, orc, z, P, cfg, lam, delta, max_iters, tol, m, ctx, norm="l2", **opt):
    s = rds.Solver(*z.shape, **opt)
    s.set_option(rds.RDS_OPT_STOP_NORM, {"l2": 0, "rms": 1}[norm])
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    st = s.solve_tol(lam, cfg.theta, cfg.tau, delta, max_iters, tol, m)
    me = st["check_every"]
    assert me == (m or 5 * st["k_fuse"])
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    o = orc.solve_tol(f, delta, lam, np.float32(cfg.theta), cfg.tau, max_iters, tol, me, norm)
    if st["iters"] != o["iters"]:
        # only a check whose residual sits within rounding of tol may decide differently
        lo = min(st["iters"], o["iters"])
        r_lo = orc.solve_tol(f, delta, lam, np.float32(cfg.theta), cfg.tau, lo, np.inf,
                             lo, norm)["residual"]
        assert abs(st["iters"] - o["iters"]) == me and abs(r_lo - tol) <= 2e-2 * tol, \
            (ctx, st["iters"], o["iters"], r_lo)
        o = orc.solve_tol(f, delta, lam, np.float32(cfg.theta), cfg.tau, st["iters"], np.inf,
                          st["iters"], norm)
    assert st["converged"] == int(o["residual"] <= tol or st["iters"] < max_iters), ctx
    assert abs(st["residual"] - o["residual"]) <= 2e-2 * max(o["residual"], 1e-6), \
        (ctx, st["residual"], o["residual"])
    p1, p2 = s.p()
    g = dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask())
    compare(g, o, ctx=ctx)
    return s, st


@pytest.mark.parametrize("name,lam,dr,tol,m,norm", [
    ("C0", 5.0, 0.2, 1e-2, 0, "l2"),      # empty band: fires at the first check, residual 0
    ("C0", 5.0, math.inf, 1e-2, 0, "l2"),  # the paper's delta_stop on the paper's image size
    ("C0", 5.0, math.inf, 1e-3, 0, "rms"),
    ("C1", 5.0, 0.2, 0.5, 0, "l2"),
    ("C1", 2.0, math.inf, 2e-3, 10, "rms"),  # blocks of 10 = two launches of 5 at k_fuse 7
    ("C2", 5.0, 0.2, 1.0, 8, "l2"),
])
def test_solve_tol_configs(rds, orc, name, lam, dr, tol, m, norm):
    cfg = wl.CONFIGS[name]
    z, P = wl.make_image(cfg)
    delta = wl.band_delta(dr, orc.absmax(orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)))
    s, st = _tol_case(rds, orc, z, P, cfg, lam, delta, cfg.iters, tol, m,
                      f"{name} lam={lam} d={dr} tol={tol} m={m} {norm}", norm=norm)
    if dr == 0.2 and name == "C0":
        assert st["iters"] == st["check_every"] and st["residual"] == 0.0
    s.close()


@pytest.mark.parametrize("m,kf,max_iters,tol", [(1, 7, 23, 0.1), (3, 2, 31, 0.0),
                                               (9, 4, 50, 0.2), (7, 7, 45, 0.0),
                                               (7, 7, 3000, 0.05), (2, 5, 4001, 0.05),
                                               (10, 7, 7, 0.0)])
def test_solve_tol_schedules(rds, orc, m, kf, max_iters, tol):
    """Single-stage CHECK launches (u^(l-1) from the u plane), blocks split across launches,
    max_iters off the check grid, tol = 0 (runs to max_iters, converged = 0), ragged shape."""
    cfg = wl.CONFIGS["C1"]
    rng = np.random.default_rng(m * 100 + kf)
    z = rng.uniform(0, 1, (75, 133)).astype(np.float32)
    s, st = _tol_case(rds, orc, z, None, cfg, 5.0, np.float32(0.3), max_iters, tol, m,
                      f"m={m} kf={kf} K={max_iters} tol={tol}", k_fuse=kf, compact=0)
    if tol == 0.0:
        assert st["iters"] == max_iters and st["converged"] == 0
    # graph replay and a fixed-K solve on the same handle afterwards
    u1 = s.u().copy()
    st2 = s.solve_tol(5.0, cfg.theta, cfg.tau, np.float32(0.3), max_iters, tol, m)
    assert st2["iters"] == st["iters"] and np.array_equal(s.u(), u1)
    s.solve(5.0, cfg.theta, cfg.tau, np.float32(0.3), st["iters"])
    assert np.array_equal(s.u(), u1)
    s.close()


# ------------------------------------------------------------------------------------------
# float64 mode: the paper's ground truth u^GT and E1 / E2
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["C0-original", "random-restricted"])
def test_solve_gt_fp64(rds, orc, case):
    """rds_solve_gt evaluates every formula in float64 in the order written, with correctly
    rounded sqrt/division and no contraction -- like the fp64 oracle -- so the stopping
    iteration agrees and the state is expected to be bit-identical."""
    if case == "C0-original":
        cfg = wl.CONFIGS["C0"]
        z, P = wl.make_image(cfg)
        delta, tol, m, K = math.inf, 1e-6, 10, 40000
    else:
        cfg = wl.CONFIGS["C1"]
        z = np.random.default_rng(9).uniform(0, 1, (64, 70)).astype(np.float32)
        P = None
        delta, tol, m, K = np.float32(0.3), 1e-7, 7, 40000
    f = orc.fitting(z, cfg.c1, cfg.c2, cfg.gamma, P)
    s = rds.Solver(*z.shape)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2, cfg.gamma, P)
    g = s.solve_gt(5.0, cfg.theta, cfg.tau, delta, K, tol, m)
    o = orc.solve_tol(f, delta, 5.0, np.float32(cfg.theta), cfg.tau, K, tol, m)
    assert g["converged"] == 1 and g["iters"] == o["iters"], (g, o["iters"])
    assert abs(g["residual"] - o["residual"]) <= 1e-9 * o["residual"]
    ug = s.u_gt()
    assert np.abs(ug - o["u"]).max() <= 1e-12
    assert np.array_equal(ug, o["u"]), "fp64 mode not bit-identical to the fp64 oracle"
    s.close()


def test_compare_gt_e1_e2(rds, orc):
    """E1 / E2 on the GPU equal the oracle's definitions applied to the GPU's own arrays;
    at q = 1 (delta = inf) the float solve to the paper's 1e-2 reproduces the thresholded
    ground truth exactly (Table 1's q = 1 row: E1 = 1.000)."""
    cfg = wl.CONFIGS["C0"]
    z, P = wl.make_image(cfg)
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2)
    s.solve_gt(5.0, cfg.theta, cfg.tau, math.inf, 100000, 1e-8, 10)
    ug = s.u_gt()
    for q in (1.0, 0.3, 0.0):
        st = s.solve_tol(5.0, cfg.theta, cfg.tau, s.band_for_fraction(q), 20000, 1e-2)
        u = s.u()
        e1, e2 = s.compare_gt(0.5)
        assert e1 == orc.tanimoto(u > 0.5, ug > 0.5), (q, e1)
        assert abs(e2 - orc.l2_error(u, ug)) <= 1e-9 * max(1.0, e2), (q, e2)
        if q == 1.0:
            assert e1 == 1.0
    s.close()


def test_solve_tol_c3_full_size(rds, orc):
    """The tolerance path (graph while loop, CHECK launches, per-item sums) at the headline
    size in the bench's launch configuration: tol = 0 runs all 63 iterations (9 checks)."""
    cfg = wl.CONFIGS["C3"]
    z, P = wl.make_image(cfg)
    f = orc.fitting(z, cfg.c1, cfg.c2)
    delta = wl.band_delta(0.2, orc.absmax(f))
    s = rds.Solver(cfg.H, cfg.W)
    s.set_image(z)
    s.set_fitting(cfg.c1, cfg.c2)
    st = s.solve_tol(5.0, cfg.theta, cfg.tau, delta, 63, 0.0, 7)
    assert st["iters"] == 63 and st["converged"] == 0 and st["check_every"] == 7
    o = orc.solve_tol(f, delta, 5.0, np.float32(cfg.theta), cfg.tau, 63, 0.0, 7)
    assert abs(st["residual"] - o["residual"]) <= 2e-2 * o["residual"]
    p1, p2 = s.p()
    compare(dict(u=s.u(), v=s.v(), p1=p1, p2=p2, mask=s.mask()), o, ctx="C3 tol")
    s.close()


@pytest.mark.parametrize("grid", [0, 1])
@pytest.mark.parametrize("shape,kf", [((37, 61), 0), ((64, 128), 7), ((5, 3), 2),
                                      ((130, 250), 5), ((33, 129), 8)])
def test_frame_untouched(rds, shape, kf, grid):
    """Memory safety without a sanitizer (compute-sanitizer is closed on this pool): after
    solves in every launch mode, warm starts, tolerance and fp64 solves, no element of the
    padded frame around the image has changed (rds_check_frame)."""
    H, W = shape
    z = np.random.default_rng(H * W).uniform(0, 1, shape).astype(np.float32)
    s = rds.Solver(H, W, k_fuse=kf, compact=0, resident=0, grid=grid)
    s.set_image(z)
    s.set_fitting(0.75, 0.25, 1.5, np.random.default_rng(1).uniform(0, 1, shape).astype(np.float32))
    d = 0.3 * s.absmax()
    s.solve(4.0, 0.1, 0.125, d, 23)
    assert s.check_frame() == 0
    s.solve_tol(4.0, 0.1, 0.125, d, 40, 1e-3, 3)
    assert s.check_frame() == 0
    s.set_state(s.v(), *s.p())
    s.solve(4.0, 0.1, 0.125, math.inf, 9)
    s.solve_gt(4.0, 0.1, 0.125, math.inf, 30, 1e-6, 7)
    s.energy()
    assert s.check_frame() == 0
    s.close()



@pytest.mark.parametrize("delta_rel,K", [(0.3, 1), (0.3, 60), (math.inf, 40), (0.15, 25)])
def test_energy_f_rd(rds, orc, delta_rel, K):
    """F_rd of rds_energy is the oracle's F^RD(u', v) (reading R-C12; u' = v^(K-1) - theta
    div rho^K on the full grid) at the last iteration, to float32 accuracy."""
    z = wl.random_image(57, 83, 21)
    f = orc.fitting(z, 0.75, 0.25)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    s = rds.Solver(57, 83)
    s.set_image(z)
    s.set_fitting(0.75, 0.25)
    s.solve(4.0, 0.1, 0.125, delta, K)
    e = s.energy()
    o = orc.solve(f, delta, 4.0, np.float32(0.1), 0.125, K, trace=True)
    F = o["trace"][K - 1][3]
    assert abs(e["F_rd"] - F) <= 1e-4 * max(1.0, abs(F)), (e["F_rd"], F)
    s.close()
