"""Seeded synthetic inputs for the restricted-domain solver (shared by tests, bench and smoke).

This module holds the *input recipe only*: it draws images z and selection maps P (and random
solver states for warm-start tests).  It contains none of the method's arithmetic -- no fitting
term, no band test, no iteration -- so that the CUDA path and the oracle can both consume its
arrays without sharing any computation (task rule: "only the seeded input generators serve
both").

The recipes follow SURVEY.md §8(d) (configs C0-C4 = BASELINE.json ``configs[0..4]``):

* C0  128^2 disk on a flat background, sigma=0.05     -- the paper's own image size
      (§4 "the size of all images tested here are 128x128").
* C1  1024^2, 12 random ellipses + ramp, sigma=0.1    -- Chan-Vese fitting (Eq. 2).
* C2  2048^2, 30 ellipses, selection map P from a polygon through 5 markers in ellipse 0
      -- distance-selective fitting (Eq. 3; P is not defined there, reading C13).
* C3  4096^2 Voronoi of 200 sites, sigma=0.15          -- the "strong noise" case.
* C4  16384^2 = 8x8 tiles of the C2 generator, seeds 100..163.
* V1  256^3 volume, 12 random ellipsoids + ramp, sigma=0.1 -- the 3-D extension (f4,
      PAPER.md:310; not a BASELINE config: the C1 recipe lifted to a volume).

Everything is drawn in float64 with ``numpy.random.default_rng(seed)`` (PCG64) and cast to
float32 last; z is not clipped (reading C14).  Pixel (i, j) has its centre at integer
coordinates, i is the row.  The paper's own images are not distributed (PAPER.md:160-195 are
[FIGURE] placeholders), so these synthetic inputs stand in for them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

INF = float("inf")


@dataclass(frozen=True)
class Config:
    name: str
    H: int
    W: int
    seed: int
    c1: float
    c2: float
    gamma: float
    lambdas: tuple
    theta: float
    tau: float
    iters: int
    delta_rels: tuple  # band thresholds as fractions of max|f|; inf = unrestricted
    desc: str = ""


CONFIGS = {
    "C0": Config("C0", 128, 128, 0, 0.8, 0.2, 0.0, (5.0,), 0.1, 0.125, 200, (0.2, INF),
                 "128x128 disk R=30, bg 0.2 / fg 0.8, sigma 0.05 (BASELINE configs[0])"),
    "C1": Config("C1", 1024, 1024, 1, 0.75, 0.25, 0.0, (2.0, 5.0, 10.0), 0.1, 0.125, 500,
                 (0.05, 0.1, 0.2, 0.4, INF),
                 "1024x1024, 12 ellipses + ramp, sigma 0.1 (BASELINE configs[1])"),
    "C2": Config("C2", 2048, 2048, 2, 0.75, 0.25, 2.0, (5.0,), 0.1, 0.125, 500,
                 (0.05, 0.1, 0.2, 0.4, INF),
                 "2048x2048, 30 ellipses, selective P, gamma 2 (BASELINE configs[2])"),
    "C3": Config("C3", 4096, 4096, 3, 0.8, 0.2, 0.0, (5.0,), 0.1, 0.125, 1000,
                 (0.1, 0.2, 0.4, INF),
                 "4096x4096 Voronoi of 200 cells, sigma 0.15 (BASELINE configs[3], headline)"),
    "C4": Config("C4", 16384, 16384, 100, 0.75, 0.25, 1.0, (5.0,), 0.1, 0.125, 1000,
                 (0.2, INF),
                 "16384x16384, 8x8 blocks of the C2 generator, seeds 100..163, gamma 1 "
                 "(BASELINE configs[4])"),
}


# --------------------------------------------------------------------------------------------
# primitive shapes
# --------------------------------------------------------------------------------------------

def _grid(H, W):
    ii = np.arange(H, dtype=np.float64)[:, None]
    jj = np.arange(W, dtype=np.float64)[None, :]
    return ii, jj


def _paint_ellipse(img, cy, cx, a, b, ang, value):
    """Overwrite pixels with centre inside the rotated ellipse (semi-axes a, b, major axis at
    angle ``ang`` from the column axis) with ``value``."""
    H, W = img.shape
    r = max(a, b)
    i0, i1 = max(0, int(math.floor(cy - r)) - 1), min(H, int(math.ceil(cy + r)) + 2)
    j0, j1 = max(0, int(math.floor(cx - r)) - 1), min(W, int(math.ceil(cx + r)) + 2)
    if i0 >= i1 or j0 >= j1:
        return
    ii = np.arange(i0, i1, dtype=np.float64)[:, None] - cy
    jj = np.arange(j0, j1, dtype=np.float64)[None, :] - cx
    ca, sa = math.cos(ang), math.sin(ang)
    u = jj * ca + ii * sa
    w = -jj * sa + ii * ca
    inside = (u / a) ** 2 + (w / b) ** 2 <= 1.0
    img[i0:i1, j0:j1][inside] = value


def _polygon_distance(H, W, poly):
    """Euclidean distance from each pixel centre to the filled polygon ``poly`` (K x 2 array of
    (row, col) vertices in order); 0 inside (crossing-number test)."""
    ii, jj = _grid(H, W)
    ii = np.broadcast_to(ii, (H, W))
    jj = np.broadcast_to(jj, (H, W))
    n = len(poly)
    inside = np.zeros((H, W), dtype=bool)
    dist2 = np.full((H, W), np.inf)
    for k in range(n):
        ay, ax = poly[k]
        by, bx = poly[(k + 1) % n]
        # crossing test along +col ray
        cond = (ay > ii) != (by > ii)
        with np.errstate(divide="ignore", invalid="ignore"):
            xint = ax + (ii - ay) * (bx - ax) / (by - ay)
        inside ^= cond & (jj < xint)
        # point-segment distance
        dy, dx = by - ay, bx - ax
        L2 = dy * dy + dx * dx
        t = np.clip(((ii - ay) * dy + (jj - ax) * dx) / L2, 0.0, 1.0)
        py = ay + t * dy
        px = ax + t * dx
        dist2 = np.minimum(dist2, (ii - py) ** 2 + (jj - px) ** 2)
    d = np.sqrt(dist2)
    d[inside] = 0.0
    return d


# --------------------------------------------------------------------------------------------
# generators
# --------------------------------------------------------------------------------------------

def gen_disk(H=128, W=128, seed=0, R=30.0, bg=0.2, fg=0.8, sigma=0.05):
    """C0: disk of radius R centred at ((H-1)/2, (W-1)/2), inside iff d^2 <= R^2."""
    rng = np.random.default_rng(seed)
    ii, jj = _grid(H, W)
    d2 = (ii - (H - 1) / 2.0) ** 2 + (jj - (W - 1) / 2.0) ** 2
    z = np.where(d2 <= R * R, fg, bg).astype(np.float64)
    z = z + rng.normal(0.0, sigma, size=(H, W))
    return z.astype(np.float32)


def gen_ellipses(N, seed, n_ell, bg=0.25, fg=0.75, ramp=0.05, sigma=0.1, selective=False):
    """C1 / C2 generator.  Draw order: per ellipse (a, b, cy, cx, angle); for C2 the target
    ellipse 0 has its centre in [N/4, 3N/4)^2; then (C2) 5 markers uniform in the target scaled
    by 0.8; then the noise field.  Returns (z float32, P float32 or None, markers)."""
    rng = np.random.default_rng(seed)
    z = np.full((N, N), bg, dtype=np.float64)
    ells = []
    for e in range(n_ell):
        a = rng.uniform(20.0, 150.0)
        b = rng.uniform(20.0, 150.0)
        if selective and e == 0:
            cy, cx = rng.uniform(N / 4.0, 3.0 * N / 4.0, size=2)
        else:
            cy, cx = rng.uniform(0.0, N, size=2)
        ang = rng.uniform(0.0, math.pi)
        ells.append((cy, cx, a, b, ang))
        _paint_ellipse(z, cy, cx, a, b, ang, fg)
    _, jj = _grid(1, N)
    z = z + ramp * (2.0 * jj / (N - 1) - 1.0)
    markers = None
    P = None
    if selective:
        cy, cx, a, b, ang = ells[0]
        r = np.sqrt(rng.uniform(0.0, 1.0, size=5))
        phi = rng.uniform(0.0, 2.0 * math.pi, size=5)
        u = 0.8 * a * r * np.cos(phi)
        w = 0.8 * b * r * np.sin(phi)
        ca, sa = math.cos(ang), math.sin(ang)
        mx = cx + u * ca - w * sa
        my = cy + u * sa + w * ca
        markers = np.stack([my, mx], axis=1)
    z = z + rng.normal(0.0, sigma, size=(N, N))
    if selective:
        cen = markers.mean(axis=0)
        order = np.argsort(np.arctan2(markers[:, 0] - cen[0], markers[:, 1] - cen[1]),
                           kind="stable")
        poly = markers[order]
        d = _polygon_distance(N, N, poly)
        P = (d / d.max()).astype(np.float32)
    return z.astype(np.float32), P, markers


def gen_voronoi(N=4096, seed=3, n_sites=200, lo=0.2, hi=0.8, sigma=0.15):
    """C3: Voronoi partition of ``n_sites`` sites ~ U[0,N)^2 (nearest site, ties -> lower
    index), cell value lo or hi with probability 1/2, plus N(0, sigma^2) noise."""
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    sites = rng.uniform(0.0, N, size=(n_sites, 2))
    vals = np.where(rng.random(n_sites) < 0.5, lo, hi)
    tree = cKDTree(sites)
    z = np.empty((N, N), dtype=np.float64)
    jj = np.arange(N, dtype=np.float64)
    for i0 in range(0, N, 256):
        i1 = min(N, i0 + 256)
        pts = np.stack(np.broadcast_arrays(np.arange(i0, i1, dtype=np.float64)[:, None],
                                           jj[None, :]), axis=-1).reshape(-1, 2)
        d, idx = tree.query(pts, k=2)
        tie = d[:, 0] == d[:, 1]
        nearest = np.where(tie, np.minimum(idx[:, 0], idx[:, 1]), idx[:, 0])
        z[i0:i1] = vals[nearest].reshape(i1 - i0, N)
    z = z + rng.normal(0.0, sigma, size=(N, N))
    return z.astype(np.float32)


def make_image(cfg: Config | str):
    """Return (z, P) for a config; P is None when the config has no selection term."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.name == "C0":
        return gen_disk(cfg.H, cfg.W, cfg.seed), None
    if cfg.name == "C1":
        z, _, _ = gen_ellipses(cfg.H, cfg.seed, 12)
        return z, None
    if cfg.name == "C2":
        z, P, _ = gen_ellipses(cfg.H, cfg.seed, 30, selective=True)
        return z, P
    if cfg.name == "C3":
        return gen_voronoi(cfg.H, cfg.seed), None
    if cfg.name == "C4":
        B = 2048
        nb = cfg.H // B
        z = np.empty((cfg.H, cfg.W), dtype=np.float32)
        P = np.empty((cfg.H, cfg.W), dtype=np.float32)
        for b in range(nb * nb):
            bi, bj = divmod(b, nb)
            zb, Pb, _ = gen_ellipses(B, 100 + b, 30, selective=True)
            z[bi * B:(bi + 1) * B, bj * B:(bj + 1) * B] = zb
            P[bi * B:(bi + 1) * B, bj * B:(bj + 1) * B] = Pb
        return z, P
    raise KeyError(cfg.name)


@dataclass(frozen=True)
class VolConfig:
    name: str
    D: int
    H: int
    W: int
    seed: int
    c1: float
    c2: float
    lam: float
    theta: float
    tau: float
    iters: int
    delta_rels: tuple
    desc: str = ""


VOL_CONFIGS = {
    "V1": VolConfig("V1", 256, 256, 256, 11, 0.75, 0.25, 5.0, 0.1, 1.0 / 12.0, 200,
                    (0.2, INF), "256^3, 12 ellipsoids + ramp, sigma 0.1 (3-D extension, f4)"),
}


def gen_ellipsoids(D, H, W, seed, n_ell=12, bg=0.25, fg=0.75, ramp=0.05, sigma=0.1,
                   amin=8.0, amax=60.0):
    """Volume recipe (V1): per ellipsoid semi-axes (a, b, c) ~ U[amin, amax], centre ~
    U[0,D) x U[0,H) x U[0,W), a random rotation (three angles ~ U[0, pi)), value fg
    (overwrite) on bg; a ramp +-ramp along j; N(0, sigma^2) noise.  float32 (D, H, W)."""
    rng = np.random.default_rng(seed)
    z = np.full((D, H, W), bg, dtype=np.float64)
    kk = np.arange(D, dtype=np.float64)[:, None, None]
    ii = np.arange(H, dtype=np.float64)[None, :, None]
    jj = np.arange(W, dtype=np.float64)[None, None, :]
    for _ in range(n_ell):
        a, b, c = rng.uniform(amin, amax, size=3)
        ck, ci, cj = rng.uniform(0, D), rng.uniform(0, H), rng.uniform(0, W)
        al, be, ga = rng.uniform(0.0, math.pi, size=3)
        ca, sa, cb, sb, cg, sg = (math.cos(al), math.sin(al), math.cos(be), math.sin(be),
                                  math.cos(ga), math.sin(ga))
        R = np.array([[ca, -sa, 0], [sa, ca, 0], [0, 0, 1]]) @ \
            np.array([[cb, 0, sb], [0, 1, 0], [-sb, 0, cb]]) @ \
            np.array([[1, 0, 0], [0, cg, -sg], [0, sg, cg]])
        dk, di, dj = kk - ck, ii - ci, jj - cj
        x = R[0, 0] * dk + R[1, 0] * di + R[2, 0] * dj
        y = R[0, 1] * dk + R[1, 1] * di + R[2, 1] * dj
        w = R[0, 2] * dk + R[1, 2] * di + R[2, 2] * dj
        z[(x / a) ** 2 + (y / b) ** 2 + (w / c) ** 2 <= 1.0] = fg
    z = z + ramp * (2.0 * jj / max(W - 1, 1) - 1.0)
    z = z + rng.normal(0.0, sigma, size=(D, H, W))
    return z.astype(np.float32)


def make_volume(cfg: VolConfig | str):
    if isinstance(cfg, str):
        cfg = VOL_CONFIGS[cfg]
    return gen_ellipsoids(cfg.D, cfg.H, cfg.W, cfg.seed)


def band_delta(delta_rel: float, absmax_f: float) -> np.float32:
    """Absolute band threshold: delta_rel * max|f| formed in float64 and rounded once to
    float32.  inf stays inf (unrestricted solve)."""
    if math.isinf(delta_rel):
        return np.float32(np.inf)
    return np.float32(np.float64(delta_rel) * np.float64(absmax_f))


def random_image(H, W, seed, lo=0.0, hi=1.0):
    """Uniform random image for small parity cases."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(H, W)).astype(np.float32)


def random_state(H, W, seed):
    """Random warm-start state: v ~ U[0,1], p uniform in the unit disk (|p| <= 1)."""
    rng = np.random.default_rng(seed)
    v = rng.uniform(0.0, 1.0, size=(H, W))
    r = np.sqrt(rng.uniform(0.0, 1.0, size=(H, W))) * 0.999
    phi = rng.uniform(0.0, 2.0 * math.pi, size=(H, W))
    return (v.astype(np.float32), (r * np.cos(phi)).astype(np.float32),
            (r * np.sin(phi)).astype(np.float32))
