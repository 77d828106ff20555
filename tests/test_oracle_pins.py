"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and mathematics fix.

None of these re-derive the oracle's own formula: each checks a closed form, a textbook
identity, a brute-force enumeration, an invariant the paper states or implies, or a worked
value (fixtures under tests/golden/, each with its citation).  CPU only.
"""
import itertools
import math

import numpy as np
import pytest

from paper_1807_11534_b200 import workloads as wl

THETA, TAU = 0.1, 0.125


def _golden(name):
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", name)
    rows = []
    with open(path) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append([float(x) for x in line.split()])
    return rows


# ------------------------------------------------------------------------------------------
# A1 fitting term (Eq. 2-3)
# ------------------------------------------------------------------------------------------

def test_fitting_worked_values(orc):
    """SPEC.md:128-130 plug-in values (tests/golden/fitting_values.txt)."""
    for z, c1, c2, gamma, P, f_expect in _golden("fitting_values.txt"):
        f = orc.fitting(np.array([[z]], np.float32), c1, c2, gamma,
                        np.array([[P]], np.float32))
        assert f[0, 0] == np.float32(f_expect), (z, c1, c2, gamma, P, f[0, 0])


def test_fitting_algebraic_identity(orc):
    """f = (c2-c1)(2z-c1-c2) exactly in reals; float32 A1 order is within 4 ulp(max(a^2,b^2))."""
    rng = np.random.default_rng(7)
    z = rng.uniform(-0.5, 1.5, size=(64, 64)).astype(np.float32)
    for c1, c2 in [(0.8, 0.2), (0.75, 0.25), (0.1, 0.9), (0.3, 0.31)]:
        c1f, c2f = np.float32(c1), np.float32(c2)
        f = orc.fitting(z, c1, c2).astype(np.float64)
        zd = z.astype(np.float64)
        exact = (float(c2f) - float(c1f)) * (2 * zd - float(c1f) - float(c2f))
        scale = np.maximum((zd - float(c1f)) ** 2, (zd - float(c2f)) ** 2)
        ulp = np.spacing(scale.astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(f - exact) <= 4 * ulp + 1e-30)
        # antisymmetry in (c1, c2) is exact in IEEE round-to-nearest
        assert np.array_equal(orc.fitting(z, c2, c1), -orc.fitting(z, c1, c2))


def test_fitting_selective_reduces(orc):
    """gamma=0 or P=0 gives the Chan-Vese term exactly."""
    rng = np.random.default_rng(8)
    z = rng.uniform(0, 1, size=(33, 17)).astype(np.float32)
    P = rng.uniform(0, 1, size=z.shape).astype(np.float32)
    cv = orc.fitting(z, 0.75, 0.25)
    assert np.array_equal(orc.fitting(z, 0.75, 0.25, 0.0, P), cv)
    assert np.array_equal(orc.fitting(z, 0.75, 0.25, 2.0, np.zeros_like(P)), cv)
    # selective term is monotone in gamma*P
    f2 = orc.fitting(z, 0.75, 0.25, 2.0, P)
    assert np.all(f2 >= cv)


def test_absmax_exact(orc):
    rng = np.random.default_rng(9)
    f = rng.normal(size=(100, 37)).astype(np.float32)
    assert orc.absmax(f) == np.abs(f).max()
    assert orc.absmax(np.zeros((3, 3), np.float32)) == 0.0


# ------------------------------------------------------------------------------------------
# A2 partition + tiles
# ------------------------------------------------------------------------------------------

def _labels_by_sets(f, delta):
    """The paper's set display: Fg = {f <= -q^}, Bg = {f >= q^}, RD = rest; overlap at
    f = 0, q^ = 0 resolved to Fg (reading R-C7)."""
    lab = np.full(f.shape, 2, dtype=np.uint8)
    fg = f <= -delta
    bg = (f >= delta) & ~fg
    lab[bg] = 0
    lab[fg] = 1
    return lab


def test_labels_bruteforce_enumeration(orc):
    """All 3x3 grids over f in {-1,-.5,0,.5,1} (5^9 grids, batched as one image) for
    delta in {0, .5, 1, inf}: labels equal the set definition."""
    vals = np.array([-1.0, -0.5, 0.0, 0.5, 1.0], np.float32)
    grids = np.array(list(itertools.product(range(5), repeat=9)), dtype=np.int64)
    f = vals[grids].reshape(-1, 9)  # each row one 3x3 grid
    for delta in (0.0, 0.5, 1.0, np.inf):
        lab = orc.labels(f, delta)
        assert np.array_equal(lab, _labels_by_sets(f, np.float32(delta)))


def test_labels_edge_semantics(orc):
    f = np.array([[-1.0, -0.5, 0.0, 0.5, 1.0, -0.0]], np.float32)
    assert orc.labels(f, np.inf).tolist() == [[2] * 6]            # q=1: RD = Omega
    assert orc.labels(f, 0.0).tolist() == [[1, 1, 1, 0, 0, 1]]      # q=0: sign rule, H(0)=1
    assert orc.labels(f, 0.5).tolist() == [[1, 1, 2, 0, 0, 2]]      # |f| = delta is pinned
    assert orc.labels(f, 0.5000001).tolist() == [[1, 2, 2, 2, 0, 2]]


def test_labels_monotone_and_consistent(orc):
    rng = np.random.default_rng(10)
    f = rng.normal(size=(50, 60)).astype(np.float32)
    prev = None
    u0 = (f <= 0)
    for delta in (0.0, 0.01, 0.1, 0.5, 1.0, 3.0, np.inf):
        lab = orc.labels(f, delta)
        rd = lab == 2
        if prev is not None:
            assert np.all(rd[prev])  # RD(delta) grows with delta
        prev = rd
        assert np.all(u0[lab == 1]) and not np.any(u0[lab == 0])


def test_tiles_bruteforce(orc):
    rng = np.random.default_rng(11)
    for (H, W, th, tw) in [(1, 1, 32, 32), (70, 45, 32, 32), (64, 64, 32, 32), (33, 97, 8, 16),
                           (5, 200, 4, 4)]:
        for p in (0.0, 0.001, 0.05, 1.0):
            lab = np.where(rng.random((H, W)) < p, 2, 1).astype(np.uint8)
            got = orc.tiles(lab, th, tw)
            ntj = -(-W // tw)
            expect = [ti * ntj + tj for ti in range(-(-H // th)) for tj in range(ntj)
                      if np.any(lab[ti * th:(ti + 1) * th, tj * tw:(tj + 1) * tw] == 2)]
            assert got.tolist() == expect


# ------------------------------------------------------------------------------------------
# Discrete operators (PAPER.md:70 -> reading R-C6)
# ------------------------------------------------------------------------------------------

def test_grad_small_examples(orc):
    g1, g2 = orc.grad(np.full((5, 5), 3.7))
    assert not g1.any() and not g2.any()
    g1, g2 = orc.grad(np.array([[0.0, 1.0]]))
    assert g2.tolist() == [[1.0, 0.0]] and g1.tolist() == [[0.0, 0.0]]


def test_grad_div_dense_matrix(orc):
    """Build the forward-difference gradient as a dense matrix from its definition; div must
    act as -G^T (negative adjoint) on random fields."""
    H, W = 4, 5
    n = H * W
    G = np.zeros((2 * n, n))
    for i in range(H):
        for j in range(W):
            k = i * W + j
            if i < H - 1:
                G[k, k] -= 1
                G[k, k + W] += 1
            if j < W - 1:
                G[n + k, k] -= 1
                G[n + k, k + 1] += 1
    rng = np.random.default_rng(12)
    u = rng.normal(size=(H, W))
    g1, g2 = orc.grad(u)
    assert np.allclose(np.concatenate([g1.ravel(), g2.ravel()]), G @ u.ravel(), atol=1e-15)
    p = rng.normal(size=2 * n)
    # only components the gradient can produce are meaningful for the adjoint
    mask = np.abs(G).sum(axis=1) > 0
    p[~mask] = 0
    d = orc.div(p[:n].reshape(H, W), p[n:].reshape(H, W))
    assert np.allclose(d.ravel(), -(G.T @ p), atol=1e-14)


def test_adjointness_random(orc):
    """<grad u, p> + <u, div p> = 0 with p1 last row / p2 last col zero."""
    rng = np.random.default_rng(13)
    for _ in range(40):
        H, W = rng.integers(1, 40, size=2)
        u = rng.normal(size=(H, W))
        p1 = rng.normal(size=(H, W))
        p2 = rng.normal(size=(H, W))
        p1[-1, :] = 0
        p2[:, -1] = 0
        g1, g2 = orc.grad(u)
        lhs = (g1 * p1).sum() + (g2 * p2).sum()
        rhs = (u * orc.div(p1, p2)).sum()
        scale = np.abs(g1 * p1).sum() + np.abs(g2 * p2).sum() + 1e-300
        assert abs(lhs + rhs) <= 1e-12 * scale


def test_div_grad_delta_is_neumann_laplacian(orc):
    """div grad of a delta = 5-point Laplacian with Neumann boundary."""
    for (H, W, ci, cj) in [(3, 3, 1, 1), (4, 4, 0, 0), (5, 3, 4, 2), (1, 4, 0, 1)]:
        e = np.zeros((H, W))
        e[ci, cj] = 1.0
        lap = orc.div(*orc.grad(e))
        expect = np.zeros((H, W))
        for di, dj in [(-1, 0), (1, 0), (0, -1), (0, 1)]:
            i, j = ci + di, cj + dj
            if 0 <= i < H and 0 <= j < W:
                expect[i, j] += 1.0
                expect[ci, cj] -= 1.0
        assert np.array_equal(lap, expect)


def test_tv_closed_forms(orc):
    N = 16
    u = np.zeros((N, N))
    u[:, : N // 2] = 1.0
    assert orc.tv(u) == N
    assert orc.tv(np.full((7, 9), 0.3)) == 0.0
    rng = np.random.default_rng(14)
    r = rng.normal(size=(20, 30))
    assert math.isclose(orc.tv(-2.5 * r), 2.5 * orc.tv(r), rel_tol=1e-13)
    # single interior pixel = 1: |grad| = sqrt(2) at the pixel, 1 above and 1 left
    e = np.zeros((5, 5))
    e[2, 2] = 1
    assert math.isclose(orc.tv(e), 2 + math.sqrt(2), rel_tol=1e-15)


def test_energy_closed_forms(orc):
    N = 12
    f = np.full((N, N), -1.0, np.float32)
    z = np.zeros((N, N))
    one = np.ones((N, N))
    half = np.zeros((N, N))
    half[:, : N // 2] = 1
    e0 = orc.energy(f, 2.0, z, z, z, z)
    assert e0["E_v"] == 0.0 and e0["E_u"] == 0.0
    assert e0["D_p"] == -2.0 * N * N                               # sum min(0, lambda f)
    e1 = orc.energy(f, 2.0, one, one, z, z)
    assert e1["E_v"] == 2.0 * f.sum()
    eh = orc.energy(f, 2.0, half, half, z, z)
    assert eh["E_v"] == N - N * N
    # u outside [0,1] is clamped for E_u
    e2 = orc.energy(f, 2.0, 3 * one, one, z, z)
    assert e2["E_u"] == e1["E_v"]


# ------------------------------------------------------------------------------------------
# A3 the iteration
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(1, 1), (1, 9), (9, 1), (7, 5), (32, 48)])
def test_unrestricted_equals_plain_twin(orc, shape):
    """delta = inf is bit-identical to the separately written plain solver (PAPER.md:84
    "For q=1 ... conventional manner")."""
    rng = np.random.default_rng(hash(shape) % 2**32)
    f = rng.uniform(-1, 1, size=shape).astype(np.float32)
    for lam in (0.5, 5.0):
        a = orc.solve(f, np.inf, lam, THETA, TAU, 60)
        b = orc.solve_plain(f, lam, THETA, TAU, 60)
        for k in ("u", "v", "p1", "p2"):
            assert np.array_equal(a[k], b[k]), k


def test_empty_band_is_heaviside(orc):
    """q=0 (RD = empty): the solution is the zero-thresholding H(-f)."""
    rng = np.random.default_rng(15)
    f = rng.uniform(-1, 1, size=(40, 30)).astype(np.float32)
    g = f.copy()
    g[3, 4] = 0.0
    for f, delta in ((g, 0.0), (f, float(np.abs(f).min()))):
        h = (f <= 0).astype(np.float64)
        r = orc.solve(f, delta, 5.0, THETA, TAU, 50)
        assert np.array_equal(r["u"], h) and np.array_equal(r["v"], h)
        assert not r["p1"].any() and not r["p2"].any()


def test_all_foreground(orc):
    """f < 0 everywhere gives u* = 1."""
    rng = np.random.default_rng(16)
    f = -rng.uniform(0.1, 1, size=(20, 20)).astype(np.float32)
    for delta in (np.inf, 0.5):
        r = orc.solve(f, delta, 5.0, THETA, TAU, 100)
        assert np.all(r["u"] == 1.0) and np.all(r["v"] == 1.0)


def test_v_update_worked_example(orc):
    """u=0.4, theta=0.1, lambda=5, f=-0.6 gives v = 0.7: 1x1 grid, warm start
    v=0.4, rho=0 (div rho = 0 on a 1x1 grid, so u = v)."""
    f = np.array([[-0.6]], np.float32)
    r = orc.solve(f, np.inf, 5.0, 0.1, TAU, 1, init=(np.array([[0.4]]), np.zeros((1, 1)),
                                                      np.zeros((1, 1))))
    assert abs(r["u"][0, 0] - 0.4) < 1e-15
    assert abs(r["v"][0, 0] - 0.7) < 1e-7


def test_rho_zero_for_constant_v(orc):
    """rho=0 with constant v stays 0."""
    f = np.full((9, 11), 0.01, np.float32)
    p1, p2, obj = orc.inner(f, np.inf, THETA, TAU, 5, np.full((9, 11), 0.3))
    assert not p1.any() and not p2.any()


def _disk_f(N, R):
    ii, jj = np.mgrid[0:N, 0:N]
    d2 = (ii - (N - 1) / 2.0) ** 2 + (jj - (N - 1) / 2.0) ** 2
    inside = d2 <= R * R
    return np.where(inside, -1.0, 1.0).astype(np.float32), inside


def test_disk_cheeger(orc):
    """f = -1 in a disk of radius R, +1 outside, unrestricted: E(r) = 2 pi r - lambda pi r^2
    is concave, so the minimiser is the disk for lambda R > 2 and empty for lambda R < 2
    (tests/golden/disk_cheeger.txt)."""
    for R, lamR, expect in _golden("disk_cheeger.txt"):
        f, inside = _disk_f(96, R)
        r = orc.solve(f, np.inf, lamR / R, THETA, TAU, 1000)
        m = orc.mask(r["u"]).astype(bool)
        if expect == 0:
            assert not m.any()
        else:
            assert not np.any(m & ~inside)
            assert m.sum() >= 0.98 * inside.sum()
        # restricted with delta <= 1: RD = empty, the "large lambda" answer
        r = orc.solve(f, 1.0, lamR / R, THETA, TAU, 50)
        assert np.array_equal(orc.mask(r["u"]).astype(bool), inside)


def _tv_binary(u):
    g1 = np.zeros_like(u)
    g2 = np.zeros_like(u)
    g1[:-1] = u[1:] - u[:-1]
    g2[:, :-1] = u[:, 1:] - u[:, :-1]
    return np.sqrt(g1 ** 2 + g2 ** 2).sum()


@pytest.mark.parametrize("H,W", [(2, 2), (3, 2)])
def test_bruteforce_binary_minimiser(orc, H, W):
    """Thresholded converged u* matches the exhaustive minimiser of Eq. 1
    over all 2^N labelings, for >= 95% of non-tied instances."""
    lam = 2.0
    N = H * W
    labs = np.array(list(itertools.product([0.0, 1.0], repeat=N)))
    tvs = np.array([_tv_binary(l.reshape(H, W)) for l in labs])
    old = orc.get_threads()
    orc.set_threads(1)
    try:
        ok = tot = 0
        for fv in itertools.product([-1.0, -0.5, 0.0, 0.5, 1.0], repeat=N):
            f = np.array(fv, np.float32).reshape(H, W)
            E = tvs + lam * labs @ f.ravel().astype(np.float64)
            best = np.flatnonzero(E <= E.min() + 1e-9)
            if len(best) > 1:
                continue
            r = orc.solve(f, np.inf, lam, THETA, TAU, 300)
            tot += 1
            ok += np.array_equal(orc.mask(r["u"]).ravel(), labs[best[0]].astype(np.uint8))
    finally:
        orc.set_threads(old)
    assert tot > 0 and ok >= 0.95 * tot


@pytest.mark.parametrize("delta_rel", [0.05, 0.2, 0.4, np.inf])
def test_invariants_every_iteration(orc, delta_rel):
    """|rho| <= 1, v in [0,1], weak-duality gap >= 0 at every iteration; exact pinning and
    Neumann zeros at the end (Eq. 7-9)."""
    z, _ = wl.make_image("C0")
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    r = orc.solve(f, delta, 5.0, THETA, TAU, 200, trace=True)
    tr = r["trace"]
    assert tr[:, 0].max() <= 1 + 1e-12
    assert tr[:, 1].min() >= 0 and tr[:, 2].max() <= 1
    assert tr[:, 4].min() >= -1e-9 * np.abs(tr[:, 3]).max()
    lab = r["labels"]
    u0 = (f <= 0).astype(np.float64)
    off = lab != 2
    assert np.array_equal(r["u"][off], u0[off]) and np.array_equal(r["v"][off], u0[off])
    assert not r["p1"][off].any() and not r["p2"][off].any()
    assert not r["p1"][-1, :].any() and not r["p2"][:, -1].any()


@pytest.mark.parametrize("delta_rel", [0.05, 0.2, 0.4, np.inf])
def test_energy_nonincreasing(orc, delta_rel):
    """F^RD(u', v) is non-increasing with 5 inner rho-steps (reading R-C12); with the
    default single step it may rise transiently (reported, not pinned)."""
    rng = np.random.default_rng(17)
    z = wl.gen_disk(64, 64, seed=3, R=15.0, sigma=0.15)
    f = orc.fitting(z, 0.8, 0.2)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    r = orc.solve(f, delta, 5.0, THETA, TAU, 150, inner_steps=5, trace=True)
    F = r["trace"][:, 3]
    assert np.all(np.diff(F) <= 1e-12 * np.abs(F[1:]))


@pytest.mark.parametrize("delta", [0.3, 0.7, np.inf])
def test_chambolle_inner_descent(orc, delta):
    """With v fixed and tau <= 1/8 the rho fixed point decreases
    || div rho - v/theta ||^2 at every step (Chambolle 2004)."""
    rng = np.random.default_rng(18)
    v = rng.uniform(0, 1, size=(48, 40))
    f = rng.uniform(-1, 1, size=(48, 40)).astype(np.float32)
    _, _, obj = orc.inner(f, delta, THETA, TAU, 150, v)
    assert np.all(np.diff(obj) <= 1e-12 * obj[1:])


def test_duality_gap_closes(orc):
    """Near convergence the iterate is close to the global minimiser of Eq. 4: the weak-
    duality gap E(v) - D(rho) is tiny relative to |E| (a dropped or mis-signed term would
    leave a large gap)."""
    z, _ = wl.make_image("C0")
    f = orc.fitting(z, 0.8, 0.2)
    r = orc.solve(f, np.inf, 5.0, THETA, TAU, 1000)
    e = orc.energy(f, 5.0, r["u"], r["v"], r["p1"], r["p2"])
    assert 0 <= e["gap"] <= 1e-3 * abs(e["E_v"])


def test_deterministic_across_threads(orc):
    z, _ = wl.make_image("C0")
    f = orc.fitting(z, 0.8, 0.2)
    old = orc.get_threads()
    try:
        orc.set_threads(1)
        a = orc.solve(f, np.float32(0.5), 5.0, THETA, TAU, 40)
        orc.set_threads(max(2, old))
        b = orc.solve(f, np.float32(0.5), 5.0, THETA, TAU, 40)
    finally:
        orc.set_threads(old)
    for k in ("u", "v", "p1", "p2"):
        assert a[k].tobytes() == b[k].tobytes()


def test_warm_start_respects_pinning(orc):
    rng = np.random.default_rng(19)
    f = rng.uniform(-1, 1, size=(17, 13)).astype(np.float32)
    v, p1, p2 = wl.random_state(17, 13, 3)
    r = orc.solve(f, np.float32(0.5), 5.0, THETA, TAU, 0, init=(v, p1, p2))
    lab = r["labels"]
    rd = lab == 2
    assert np.array_equal(r["v"][rd], v.astype(np.float64)[rd])
    assert np.array_equal(r["v"][~rd], (f <= 0).astype(np.float64)[~rd])
    assert not r["p1"][~rd].any() and not r["p1"][-1].any() and not r["p2"][:, -1].any()


# ------------------------------------------------------------------------------------------
# q -> q^
# ------------------------------------------------------------------------------------------

def test_band_for_fraction_spec_example(orc):
    """f = {-3..5} (3x3), q = 1/3 -> RD = {-1, 0, 1}, rd_fraction 3/9."""
    f = np.arange(-3, 6, dtype=np.float32).reshape(3, 3)
    qh = orc.band_for_fraction(f, 1.0 / 3.0)
    lab = orc.labels(f, qh)
    assert sorted(f[lab == 2].tolist()) == [-1.0, 0.0, 1.0]


def test_band_for_fraction_definition(orc):
    """Brute force against the definition: q^ is the smallest float32 with
    #{|f| < q^} >= ceil(q N); q = 0 -> RD empty, q = 1 -> RD = Omega; RD grows with q."""
    rng = np.random.default_rng(21)
    for n in (1, 2, 7, 100, 1000):
        f = rng.normal(size=n).astype(np.float32)
        f[: n // 3] = np.round(f[: n // 3], 1)   # ties
        prev = -1
        for q in (0.0, 1e-9, 0.1, 1 / 3, 0.5, 0.9, 1.0):
            qh = orc.band_for_fraction(f, q)
            k = int(np.ceil(q * n))
            cnt = int((np.abs(f) < qh).sum())
            assert cnt >= k
            below = np.nextafter(qh, np.float32(-np.inf), dtype=np.float32)
            if k > 0:
                assert int((np.abs(f) < below).sum()) < k       # minimality
            else:
                assert qh == 0.0 and cnt == 0
            assert cnt >= prev
            prev = cnt
        assert int((np.abs(f) < orc.band_for_fraction(f, 1.0)).sum()) == n


@pytest.mark.parametrize("delta_rel", [0.3, math.inf])
def test_dependency_cone_window(orc, delta_rel):
    """The premise of the full-size windowed parity tests (test_c4_full_size): after K
    iterations a block's u, v, rho depend only on inputs within 2K+2 rows/columns, so the
    oracle on a window with that margin reproduces the full-image iteration exactly -- and a
    margin that is too small does not (the cone really reaches that far)."""
    rng = np.random.default_rng(11)
    H, W, K = 90, 84, 9
    f = rng.uniform(-1, 1, (H, W)).astype(np.float32)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    full = orc.solve(f, delta, 4.0, np.float32(0.1), 0.125, K)
    r0, c0, b = 40, 38, 8
    for m, exact in ((2 * K + 2, True), (K // 2, False)):
        win = orc.solve(np.ascontiguousarray(f[r0 - m:r0 + b + m, c0 - m:c0 + b + m]), delta,
                        4.0, np.float32(0.1), 0.125, K)
        same = all(np.array_equal(win[k][m:m + b, m:m + b], full[k][r0:r0 + b, c0:c0 + b])
                   for k in ("u", "v", "p1", "p2"))
        assert same == exact, (m, same)


def _window_exact(orc, f, delta, K, r0, c0, b, top, bot, left, right):
    full = orc.solve(f, delta, 4.0, np.float32(0.1), 0.125, K)
    win = orc.solve(np.ascontiguousarray(f[r0 - top:r0 + b + bot, c0 - left:c0 + b + right]),
                    delta, 4.0, np.float32(0.1), 0.125, K)
    return all(np.array_equal(win[k][top:top + b, left:left + b], full[k][r0:r0 + b, c0:c0 + b])
               for k in ("u", "v", "p1", "p2"))


@pytest.mark.parametrize("K", [1, 2, 3, 9, 20])
@pytest.mark.parametrize("delta_rel", [0.3, math.inf])
def test_cone_margin_k_plus_1(orc, K, delta_rel):
    """The tight margin the stated-K window tests use ("window margin"): the
    window solve differs from the full one only through its cut rows / columns (rho1 of the
    row above the top cut and rho2 of the column left of the left cut read as 0; the Neumann
    conditions forced on the last window row / column).  By induction on the iteration, after
    k iterations the wrong rho reaches at most k-1 rows (columns) in from the top (left) cut
    and v at most k, and from the bottom (right) cut at most k-1: so a margin of K+1 on EVERY
    side reproduces the full-image iterates bit for bit, and (at delta = inf, where no pinned
    pixel stops the front) a margin of K-1 on the top or the bottom side does not."""
    rng = np.random.default_rng(11)
    H, W = 160, 150
    f = rng.uniform(-1, 1, (H, W)).astype(np.float32)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    r0, c0, b, m = 70, 68, 8, K + 1
    assert _window_exact(orc, f, delta, K, r0, c0, b, m, m, m, m)
    if math.isinf(delta_rel) and 2 <= K <= 9:
        assert not _window_exact(orc, f, delta, K, r0, c0, b, K - 1, m, m, m)
        assert not _window_exact(orc, f, delta, K, r0, c0, b, m, K - 1, m, m)
        assert not _window_exact(orc, f, delta, K, r0, c0, b, m, m, K - 1, m)


# ------------------------------------------------------------------------------------------
# f2: the stopping rule, RMS norm (reading R-F2)
# ------------------------------------------------------------------------------------------

def _rule_residual(orc, f, delta, lam, ell, norm):
    """max(||u^l - u^(l-1)||, ||v^l - v^(l-1)||) from two plain fixed-K solves, with the
    Euclidean norm over pixels (norm="l2") or the RMS."""
    a = orc.solve(f, delta, lam, np.float32(0.1), 0.125, ell)
    b = orc.solve(f, delta, lam, np.float32(0.1), 0.125, ell - 1)
    n = f.size if norm == "rms" else 1
    return max(math.sqrt(((a["u"] - b["u"]) ** 2).sum() / n),
               math.sqrt(((a["v"] - b["v"]) ** 2).sum() / n))


@pytest.mark.parametrize("m,tol,delta_rel,norm", [(7, 3e-3, 0.4, "rms"), (1, 1e-2, math.inf, "rms"),
                                                  (5, 1e-3, math.inf, "rms"), (4, 0.0, 0.3, "rms"),
                                                  (7, 3e-2, 0.4, "l2"), (3, 1e-2, math.inf, "l2")])
def test_stopping_rule_definition(orc, m, tol, delta_rel, norm):
    """orc_solve_tol stops at the FIRST check (multiples of m, and max_iters) whose residual,
    recomputed here from two independent fixed-K solves, is <= tol; its state is the fixed-K
    state at that iteration, bit for bit."""
    rng = np.random.default_rng(5)
    f = rng.uniform(-1, 1, (24, 30)).astype(np.float32)
    delta = wl.band_delta(delta_rel, orc.absmax(f))
    K = 40
    o = orc.solve_tol(f, delta, 4.0, np.float32(0.1), 0.125, K, tol, m, norm)
    checks = list(range(m, K, m)) + [K]
    want, r_want = None, None
    for c in checks:
        r = _rule_residual(orc, f, delta, 4.0, c, norm)
        if r <= tol or c == K:
            want, r_want = c, r
            break
    assert o["iters"] == want
    assert abs(o["residual"] - r_want) <= 1e-12 * max(1.0, r_want)
    ref = orc.solve(f, delta, 4.0, np.float32(0.1), 0.125, want)
    for k in ("u", "v", "p1", "p2"):
        assert np.array_equal(o[k], ref[k])


def test_stopping_rule_special_cases(orc):
    rng = np.random.default_rng(6)
    f = rng.uniform(-1, 1, (20, 20)).astype(np.float32)
    # empty band: nothing moves, the first check fires with residual exactly 0
    o = orc.solve_tol(f, np.float32(0.0), 4.0, np.float32(0.1), 0.125, 50, 0.0, 6)
    assert o["iters"] == 6 and o["residual"] == 0.0
    assert np.array_equal(o["u"], (f <= 0).astype(np.float64))
    # tol = inf stops at the first check; max_iters shorter than check_every -> max_iters
    o = orc.solve_tol(f, np.float32(np.inf), 4.0, np.float32(0.1), 0.125, 50, np.inf, 6)
    assert o["iters"] == 6
    o = orc.solve_tol(f, np.float32(np.inf), 4.0, np.float32(0.1), 0.125, 4, np.inf, 6)
    assert o["iters"] == 4
    # larger tolerances never stop later (the first index with r <= tol is monotone)
    its = [orc.solve_tol(f, np.float32(np.inf), 4.0, np.float32(0.1), 0.125, 200, t, 3)["iters"]
           for t in (1e-1, 1e-2, 1e-3, 1e-4)]
    assert its == sorted(its)


# ------------------------------------------------------------------------------------------
# E1 / E2 of the paper's evaluation protocol
# ------------------------------------------------------------------------------------------

def test_tanimoto_and_l2(orc):
    a = np.zeros((4, 5), bool)
    b = np.zeros((4, 5), bool)
    assert orc.tanimoto(a, b) == 1.0                       # empty/empty (R-C15)
    a.flat[[0, 1, 2]] = True
    b.flat[[1, 2, 3]] = True
    assert orc.tanimoto(a, b) == 0.5                       # |{1,2}| / |{0,1,2,3}|
    assert orc.tanimoto(a, a) == 1.0
    assert orc.tanimoto(a, ~a) == 0.0
    assert orc.tanimoto(a, b) == orc.tanimoto(b, a)
    rng = np.random.default_rng(3)
    u = rng.uniform(0, 1, (6, 7))
    assert orc.l2_error(u, u) == 0.0
    assert orc.l2_error(u + 0.25, u) == pytest.approx(42 * 0.0625, rel=1e-12)
