"""Seeded input recipe (paper_1807_11534_b200/workloads.py): determinism and structure."""
import numpy as np

from paper_1807_11534_b200 import workloads as wl


def test_deterministic_and_float32():
    a = wl.make_image("C0")[0]
    b = wl.make_image("C0")[0]
    assert a.dtype == np.float32 and a.shape == (128, 128)
    assert a.tobytes() == b.tobytes()


def test_disk_structure():
    z = wl.gen_disk(128, 128, seed=0, sigma=0.0)
    ii, jj = np.mgrid[0:128, 0:128]
    inside = (ii - 63.5) ** 2 + (jj - 63.5) ** 2 <= 900
    assert np.all(z[inside] == np.float32(0.8)) and np.all(z[~inside] == np.float32(0.2))


def test_selective_map():
    z, P, markers = wl.gen_ellipses(256, 5, 6, selective=True)
    assert P.dtype == np.float32 and P.min() == 0.0 and P.max() == 1.0
    for (mi, mj) in markers:  # markers lie in the filled polygon -> P = 0 at nearest pixel
        i, j = int(round(mi)), int(round(mj))
        assert P[i, j] <= 2.0 / 256


def test_voronoi_levels():
    z = wl.gen_voronoi(256, seed=1, n_sites=20, sigma=0.0)
    assert set(np.unique(z).tolist()) <= {np.float32(0.2), np.float32(0.8)}


def test_band_delta():
    assert wl.band_delta(float("inf"), 1.0) == np.float32(np.inf)
    assert wl.band_delta(0.2, np.float32(1.3707132)) == np.float32(0.2 * float(np.float32(1.3707132)))
